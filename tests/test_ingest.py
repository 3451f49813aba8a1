"""Host document loader (csrc/host_ingest.cpp), no GPU.

NFC: checked against CPython's unicodedata (an independent UAX #15
implementation over the same UCD version) on every code point and on random
text dense in combining sequences, Hangul and ill-formed bytes.  Loader:
checked against the reference's own build_manifest / surviving_documents /
RejectLog (oracle/_ref; its ICU-free text shim is exact for NFC input, so the
reference comparison uses NFC-stable text and the non-NFC cases are checked
against unicodedata)."""
import json
import unicodedata

import numpy as np
import pytest

from paper_2501_01046_b200 import corpus, pipeline
from paper_2501_01046_b200.minhash import ShingleUnit


def _nfc(b: bytes) -> bytes:
    return unicodedata.normalize("NFC", b.decode("utf-8", errors="replace")).encode()


def test_nfc_every_code_point():
    # each scalar isolated by '\n' (a starter that composes with nothing)
    cps = [c for c in range(0x110000) if not 0xD800 <= c < 0xE000]
    for i in range(0, len(cps), 200_000):
        s = "\n".join(chr(c) for c in cps[i:i + 200_000]).encode("utf-8")
        assert corpus.nfc_normalize(s) == _nfc(s)


def test_nfc_random_sequences():
    rng = np.random.default_rng(8)
    pool = ([chr(c) for c in range(0x41, 0x5B)] + [chr(c) for c in range(0x300, 0x370)]
            + [chr(c) for c in range(0x1100, 0x1113)] + [chr(c) for c in range(0x1161, 0x1176)]
            + [chr(c) for c in range(0x11A8, 0x11C3)] + [chr(c) for c in range(0xAC00, 0xAC40)]
            + ["Å", "Ω", "क़", "େ", "ା", "ୗ", "ཱི", "̈́",
               "Ḋ", "̣", "ೆ", "ೂ", "ೕ", "ָ", "ַ", "ཱ",
               "ི", "ᴕE", "\U0001D165", "\U0001D16E", "゙", "か", "Å",
               "e", "́", "̧", "̛", "ͅ"])
    for _ in range(3000):
        n = int(rng.integers(0, 12))
        s = "".join(pool[int(k)] for k in rng.integers(0, len(pool), size=n)).encode()
        if rng.random() < 0.2:  # ill-formed bytes -> U+FFFD first (text.cpp:49-66)
            pos = int(rng.integers(0, len(s) + 1))
            s = s[:pos] + bytes(rng.integers(0x80, 0x100, size=2, dtype=np.uint8)) + s[pos:]
        assert corpus.nfc_normalize(s) == _nfc(s), s


def test_codepoint_count_and_parse():
    assert corpus.codepoint_count("héllo") == 5
    assert corpus.codepoint_count(b"a\xe1\x80b\xff") == 4  # maximal subparts count once
    ok, text, why = corpus.parse_jsonl_line('{"text": "x\\u00e9\\ud83d\\ude00"}', "text")
    assert ok and text == "xé😀".encode()
    for line, why in [("not json", "invalid_json"), ("[1]", "not_an_object"),
                      ('{"a": 1}', "missing_text_field"), ('{"text": null}', "text_field_not_string"),
                      ('{"text": "\\ud800"}', "invalid_json"), (b'{"text": "\xff"}', "invalid_json"),
                      ('{"text": "a"} x', "invalid_json"), ("  ", "invalid_json")]:
        assert corpus.parse_jsonl_line(line, "text") == (False, None, why), line
    assert corpus.parse_jsonl_line('{"text": "a", "text": "b"}', "text") == (True, b"b", None)


def _tricky_lines(rng):
    word = lambda n: "".join(rng.choice(list("abcdefghij     klmnop"), size=n))  # noqa: E731
    lines = []
    for i in range(3000):
        k = i % 17
        if k == 0:
            lines.append("not json")
        elif k == 1:
            lines.append("")
        elif k == 2:
            lines.append(json.dumps({"text": word(50)}))  # below min_chars
        elif k == 3:
            lines.append(json.dumps({"meta": {"text": word(300)}}))
        elif k == 4:
            lines.append(json.dumps({"text": word(300), "id": i}) + "\r")
        elif k == 5:
            lines.append(json.dumps({"text": "Ωμέγα " + word(250)}, ensure_ascii=False))
        elif k == 6:
            lines.append(json.dumps({"text": "ж" * 199 + "a"}))
        elif k == 7:
            lines.append('{"text": 12}')
        elif k == 8:
            lines.append("   ")
        else:
            lines.append(json.dumps({"text": word(int(rng.integers(200, 900)))}))
    return lines


@pytest.mark.parametrize("unit,L,min_chars", [(0, 5, 200), (1, 5, 200), (0, 400, 10)])
def test_loader_matches_reference(ref, tmp_path, unit, L, min_chars):
    rng = np.random.default_rng(unit + L)
    d = tmp_path / "c"
    d.mkdir()
    lines = _tricky_lines(rng)
    (d / "b.jsonl").write_bytes(("\n".join(lines[:1500]) + "\n").encode())
    (d / "a.jsonl").write_bytes("\n".join(lines[1500:]).encode())  # no final newline
    rej_path = str(tmp_path / "rejects.jsonl")
    r_rec, r_surv, r_data, r_offs, r_ids, r_ch = ref.load_corpus(str(d), rej_path, min_chars=min_chars,
                                                                 L=L, unit=unit)
    cfg = pipeline.RunConfig(shingle_len=L, unit=ShingleUnit(unit), min_chars=min_chars)
    m, rejects = corpus.build_manifest([str(d)], cfg)
    assert (m.total_records, m.total_surviving) == (r_rec, r_surv)
    ours = str(tmp_path / "ours.jsonl")
    pipeline._write_rejects(ours, rejects)
    assert open(ours, "rb").read() == open(rej_path, "rb").read()
    parts = [corpus.surviving_packed(m, i, cfg) for i in range(len(m.files))]
    data = np.concatenate([p[0] for p in parts])
    ids = np.concatenate([p[2] for p in parts])
    chars = np.concatenate([p[3] for p in parts])
    lens = np.concatenate([np.diff(p[1]) for p in parts])
    np.testing.assert_array_equal(data, r_data)
    np.testing.assert_array_equal(ids, r_ids)
    np.testing.assert_array_equal(chars, r_ch)
    np.testing.assert_array_equal(lens, np.diff(r_offs))
    # the stages' single-parse variant: cached files pack identically, the cap
    # keeps a prefix of the files and the manifest does not change
    for cap in (1 << 40, len(parts[0][0]), 0):
        m2, rej2, cache = corpus.build_manifest_cached([str(d)], cfg, cap)
        assert (m2, rej2) == (m, rejects)
        assert sorted(cache) == list(range(len(cache)))
        assert len(cache) == (2 if cap == 1 << 40 else 1 if cap else 0)
        for i, packed in cache.items():
            for a, b in zip(packed, parts[i]):
                np.testing.assert_array_equal(a, b)


def test_loader_normalises_and_is_thread_invariant(tmp_path):
    # non-NFC input: decomposed sequences, singletons, Hangul jamo, ill-formed
    # bytes inside otherwise valid lines are rejected by the JSON parser
    texts = ["é" * 120 + "x" * 100, "Å" * 210, "각" * 80,
             "ạ̇" * 90 + "q" * 20, "plain " * 50]
    p = tmp_path / "n.jsonl"
    p.write_text("\n".join(json.dumps({"text": t}) for t in texts * 200) + "\n", encoding="utf-8")
    cfg = pipeline.RunConfig()
    outs = []
    for threads in (1, 3, 16):
        f = corpus.JsonlFile(str(p), cfg, keep_text=True, threads=threads)
        outs.append((f.records, f.surviving, f.rejects(), [a.tobytes() for a in f.packed(7)]))
    assert outs[0] == outs[1] == outs[2]
    data, offs, ids, chars = corpus.JsonlFile(str(p), cfg, keep_text=True).packed(7)
    want = [unicodedata.normalize("NFC", t) for t in texts * 200]
    want = [w for w in want if len(w) >= 200]
    got = [bytes(data[int(offs[i]):int(offs[i + 1])]).decode() for i in range(len(ids))]
    assert got == want
    assert chars.tolist() == [len(w) for w in want]
    assert ids[0] == 7


def _parse(line: bytes, mode: int, field=b"text"):
    import ctypes as C

    from paper_2501_01046_b200 import _lib

    lib = _lib.load()
    reason, n = C.c_uint32(), C.c_uint64()
    out = (C.c_uint8 * (len(line) + 8))()
    assert lib.nd_parse_jsonl_line_mode(line, len(line), field, mode, C.byref(reason), out,
                                        len(out), C.byref(n)) == 0
    return reason.value, bytes(out[:n.value]) if reason.value == 0 else None


def test_fast_scanner_agrees_with_nlohmann():
    # differential fuzz: the fast scanner either defers (255) or gives exactly
    # nlohmann's verdict and text, on valid lines and on byte-level mutations
    rng = np.random.default_rng(13)
    atoms = [b'"x"', b'""', b'"a\\"b\\\\c\\/d\\n\\t"', b'"\\u00e9"', b'"\\ud83d\\ude00"', b'"\\ud800"',
             b'"caf\xc3\xa9"', b'"\xe2\x82"', b'"\xff"', b'0', b'-0', b'12', b'-7', b'01', b'1.5',
             b'1e3', b'123456789012345678', b'1234567890123456789', b'true', b'false', b'null',
             b'tru', b'[]', b'{}', b'[1, 2]', b'{"a": [1, {"text": 2}]}', b'"\x7f"', b'"\x01"']

    def value(d):
        k = rng.integers(0, 10)
        if d < 3 and k == 0:
            return b"[" + b", ".join(value(d + 1) for _ in range(rng.integers(0, 3))) + b"]"
        if d < 3 and k == 1:
            return obj(d + 1)
        return atoms[int(rng.integers(len(atoms)))]

    def obj(d):
        keys = [b'"text"', b'"id"', b'"t"', b'"text "', b'"te\\u0078t"']
        items = [keys[int(rng.integers(len(keys)))] + b": " + value(d) for _ in range(rng.integers(0, 4))]
        return b"{" + b", ".join(items) + b"}"

    decided = 0
    for _ in range(20000):
        line = obj(0) if rng.random() < 0.85 else value(0)
        if rng.random() < 0.5:  # mutate
            b = bytearray(line)
            for _ in range(int(rng.integers(1, 4))):
                op, pos = rng.integers(0, 3), int(rng.integers(0, len(b) + 1))
                if op == 0 and pos < len(b):
                    del b[pos]
                elif op == 1:
                    b.insert(pos, int(rng.choice(list(b' {}[]",:\\\x00\x80\xc3ae0-'))))
                elif pos < len(b):
                    b[pos] = int(rng.integers(0, 256))
            line = bytes(b)
        if rng.random() < 0.1:
            line = b" \t" + line + b" \r"
        fast = _parse(line, 2)
        ref = _parse(line, 1)
        assert _parse(line, 0) == ref, line
        if fast[0] != 255:
            decided += 1
            assert fast == ref, line
    assert decided > 5000
