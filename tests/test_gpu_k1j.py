"""K1j -- the family-specialised signature kernel compiled by NVRTC at family
upload (csrc/k1_jit.cpp) -- against the register-constant K1 and the oracle.

K1j walks each item per lane in aligned 32-bit words with single steps at
both ends, so the shapes that matter are: every shingle length 1..16 (the
ring of words above the current one), documents of exactly L .. L+8 bytes,
every byte alignment of the text (4-byte words at absolute addresses), H not
a multiple of the pass width, documents split into 8192-window items, and
text ending at the very end of its buffer.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2501_01046_b200 import _lib, minhash

pytestmark = pytest.mark.gpu


def _kernel(ctx):
    return ctx.lib.nd_k1_kernel(ctx.h).decode()


def _both(ctx, monkeypatch, data, offs, fam, bands=0, rows=0, K=0):
    out = {}
    for jit in ("1", "0"):
        monkeypatch.setenv("ND_K1_JIT", jit)
        ctx._family_key = None
        sig, band = minhash.signatures_packed(data, offs, fam, bands, rows, K, ctx=ctx,
                                              want_bands=bool(bands))
        out[jit] = (sig, band, _kernel(ctx))
    monkeypatch.delenv("ND_K1_JIT")
    ctx._family_key = None
    assert out["1"][2] == "k1j", out["1"][2]
    assert out["0"][2] == "k1"
    return out


def _docs(rng, lens, alphabet=256):
    texts = [bytes(rng.integers(0, alphabet, size=int(n), dtype=np.uint8)) for n in lens]
    offs = np.zeros(len(texts) + 1, np.uint64)
    offs[1:] = np.cumsum([len(t) for t in texts])
    return np.frombuffer(b"".join(texts), np.uint8).copy(), offs


@pytest.mark.parametrize("L", list(range(1, 17)))
def test_k1j_every_shingle_length(ctx, oracle, monkeypatch, L):
    rng = np.random.default_rng(100 + L)
    lens = [L + k for k in range(9)] + list(rng.integers(L, 3000, size=40)) + [20000]
    data, offs = _docs(rng, lens)
    fam = minhash.derive_family(5, 64, L)
    out = _both(ctx, monkeypatch, data, offs, fam)
    assert np.array_equal(out["1"][0], out["0"][0])
    assert np.array_equal(out["1"][0], oracle.signatures(data, offs, oracle.derive_family(5, 64, L), L=L))


@pytest.mark.parametrize("H,bands,rows", [(100, 10, 10), (128, 16, 8), (256, 32, 8), (40, 5, 8),
                                          (512, 64, 8), (8, 2, 4)])
def test_k1j_hash_counts_and_band_keys(ctx, oracle, monkeypatch, H, bands, rows):
    rng = np.random.default_rng(H)
    lens = list(rng.integers(5, 5000, size=300)) + [9000, 17000, 8196, 8197]
    data, offs = _docs(rng, lens, alphabet=37)
    fam = minhash.derive_family(5, H, 5)
    out = _both(ctx, monkeypatch, data, offs, fam, bands, rows, 977)
    assert np.array_equal(out["1"][0], out["0"][0])
    assert np.array_equal(out["1"][1], out["0"][1])
    want = oracle.signatures(data, offs, oracle.derive_family(5, H))
    assert np.array_equal(out["1"][0], want)
    assert np.array_equal(out["1"][1], oracle.band_ids(want, bands, rows, 977))


@pytest.mark.parametrize("shift", [0, 1, 2, 3, 5, 7])
def test_k1j_text_alignment_and_buffer_end(ctx, oracle, monkeypatch, shift):
    # device text starting `shift` bytes into an allocation whose last byte is
    # the last document byte (no slack for whole-word reads past the end)
    import torch

    rng = np.random.default_rng(shift)
    data, offs = _docs(rng, list(rng.integers(5, 700, size=257)) + [5, 6, 7])
    n = len(offs) - 1
    fam = minhash.derive_family(5, 128, 5)
    buf = torch.zeros(len(data) + shift, dtype=torch.uint8, device="cuda")
    buf[shift:] = torch.from_numpy(data).cuda()
    d_offs = torch.from_numpy(offs.view(np.int64)).cuda()
    res = {}
    for jit in ("1", "0"):
        monkeypatch.setenv("ND_K1_JIT", jit)
        ctx._family_key = None
        sig = torch.empty((n, 128), dtype=torch.int32, device="cuda")
        band = torch.empty((n, 16), dtype=torch.int32, device="cuda")
        minhash.signatures_device(buf.data_ptr() + shift, d_offs.data_ptr(), n, fam, sig.data_ptr(),
                                  band.data_ptr(), 16, 8, 0, ctx=ctx)
        torch.cuda.synchronize()
        res[jit] = (sig.cpu().numpy().view(np.uint32), band.cpu().numpy().view(np.uint32))
    monkeypatch.delenv("ND_K1_JIT")
    ctx._family_key = None
    assert np.array_equal(res["1"][0], res["0"][0]) and np.array_equal(res["1"][1], res["0"][1])
    assert np.array_equal(res["1"][0], oracle.signatures(data, offs, oracle.derive_family(5, 128)))


def test_k1j_skewed_lengths_many_items(ctx, oracle, monkeypatch):
    # lognormal lengths up to 60 KB: multi-item documents (atomicMin across
    # items) mixed with short ones in one length-sorted work order
    spec = _lib.NdSynthSpec(doc_count=3000, group_count=200, group_size_min=2, group_size_max=4,
                            edit_num=1, edit_den=100, len_min=800, len_max=60000, seed=9, mode=1,
                            len_law=1, sigma_milli=1400)
    lib = _lib.load()
    nb = C.c_uint64()
    _lib.check(lib.nd_synth_generate(C.byref(spec), None, None, C.byref(nb)))
    data = np.empty(nb.value, np.uint8)
    offs = np.empty(spec.doc_count + 1, np.uint64)
    _lib.check(lib.nd_synth_generate(C.byref(spec), data.ctypes.data_as(_lib.u8p),
                                     offs.ctypes.data_as(_lib.u64p), C.byref(nb)))
    assert np.diff(offs).max() > 3 * 8196
    fam = minhash.derive_family(5, 128, 5)
    out = _both(ctx, monkeypatch, data, offs, fam, 16, 8, 1500)
    assert np.array_equal(out["1"][0], out["0"][0]) and np.array_equal(out["1"][1], out["0"][1])
    sample = np.random.default_rng(0).choice(spec.doc_count, 200, replace=False)
    for i in sample[:50]:
        o = np.array([0, offs[i + 1] - offs[i]], np.uint64)
        d = data[int(offs[i]):int(offs[i + 1])].copy()
        assert np.array_equal(out["1"][0][i], oracle.signatures(d, o, oracle.derive_family(5, 128))[0])


def test_k1j_not_used_outside_its_domain(ctx, monkeypatch):
    # codepoint units: K1j for the documents below U+0100, K1j over 16-bit
    # units for those below U+10000, K1w for the rest; L > 16: the
    # register-constant kernel
    fam = minhash.derive_family(5, 32, 5, minhash.ShingleUnit.CODEPOINT)
    ctx.upload_family(fam)
    assert _kernel(ctx) == "k1j+k1j16+k1w"
    ctx._family_key = None
    monkeypatch.setenv("ND_K1J_U16", "0")
    ctx.upload_family(fam)
    assert _kernel(ctx) == "k1j+k1w"
    monkeypatch.delenv("ND_K1J_U16")
    ctx._family_key = None
    fam = minhash.derive_family(5, 32, 20)  # L > 16
    ctx.upload_family(fam)
    assert _kernel(ctx) == "k1"
    ctx._family_key = None


@pytest.mark.parametrize("mix", ["ascii", "latin1", "mixed"])
def test_codepoint_narrow_documents_take_the_byte_kernels(ctx, oracle, monkeypatch, mix):
    # codepoint units < 256 (ASCII, and Latin-1 whose UTF-8 is two bytes)
    # hash exactly like bytes: those documents run K1j over narrowed units,
    # the rest K1w; every row must equal K1w-only and the oracle
    rng = np.random.default_rng({"ascii": 1, "latin1": 2, "mixed": 3}[mix])
    latin = [chr(c) for c in range(0xA0, 0x100)] + list("abcdefgh ")
    wide = [chr(c) for c in range(0x400, 0x450)] + [chr(c) for c in range(0x4E00, 0x4E40)]
    texts = []
    for i in range(400):
        k = int(rng.integers(5, 3000)) if i % 50 else 12000  # some multi-item documents
        if mix == "ascii" or (mix == "mixed" and i % 3 == 0):
            texts.append("".join(rng.choice(list("abcdefghijklmnop qrstuvwxyz"), size=k)))
        elif mix == "latin1" or (mix == "mixed" and i % 3 == 1):
            texts.append("".join(rng.choice(latin, size=k)))
        else:
            texts.append("".join(rng.choice(latin + wide, size=k)))
    raw = [t.encode() for t in texts]
    offs = np.zeros(len(raw) + 1, np.uint64)
    offs[1:] = np.cumsum([len(b) for b in raw])
    data = np.frombuffer(b"".join(raw), np.uint8).copy()
    fam = minhash.derive_family(5, 128, 5, minhash.ShingleUnit.CODEPOINT)
    res = {}
    for narrow in ("1", "0"):
        monkeypatch.setenv("ND_K1_NARROW", narrow)
        res[narrow] = minhash.signatures_packed(data, offs, fam, 16, 8, 1000, ctx=ctx)
    monkeypatch.delenv("ND_K1_NARROW")
    assert np.array_equal(res["1"][0], res["0"][0]) and np.array_equal(res["1"][1], res["0"][1])
    want = oracle.signatures(data, offs, oracle.derive_family(5, 128), unit=1)
    assert np.array_equal(res["1"][0], want)


@pytest.mark.parametrize("L", [1, 4, 5, 9, 16])
def test_k1j_two_words_per_iteration(ctx, oracle, monkeypatch, L):
    # ND_K1J_UNROLL=2 (pairs of words, the odd last word on single steps):
    # not the default, but a compiled shape must still be exact
    monkeypatch.setenv("ND_K1J_UNROLL", "2")
    rng = np.random.default_rng(700 + L)
    lens = [L + k for k in range(12)] + list(rng.integers(L, 3000, size=60)) + [20000]
    data, offs = _docs(rng, lens)
    fam = minhash.derive_family(5, 64, L)
    out = _both(ctx, monkeypatch, data, offs, fam)
    assert np.array_equal(out["1"][0], out["0"][0])
    assert np.array_equal(out["1"][0], oracle.signatures(data, offs, oracle.derive_family(5, 64, L), L=L))


def test_chunk_gate_host_pipelines(ctx, oracle, monkeypatch):
    # ~150 MB of text: several chunks through nd_signatures (gated K1j
    # launches on two streams, ramp down at the end) and through nd_dedup's
    # ring (gated on request); every configuration gives the same rows
    from paper_2501_01046_b200 import pipeline

    rng = np.random.default_rng(77)
    n = 70000
    lens = rng.integers(1200, 3000, size=n)
    offs = np.zeros(n + 1, np.uint64)
    offs[1:] = np.cumsum(lens)
    data = rng.integers(97, 123, size=int(offs[-1]), dtype=np.uint8)
    fam = minhash.derive_family(5, 128, 5)
    res = {}
    for name, env in {"gate": {}, "nogate": {"ND_K1J_GATE": "0"},
                      "notail": {"ND_H2D_TAIL_DIV": "0"}}.items():
        for k in ("ND_K1J_GATE", "ND_H2D_TAIL_DIV"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        res[name] = minhash.signatures_packed(data, offs, fam, 16, 8, 1000, ctx=ctx)
    for k in ("ND_K1J_GATE", "ND_H2D_TAIL_DIV"):
        monkeypatch.delenv(k, raising=False)
    for name in ("nogate", "notail"):
        assert np.array_equal(res[name][0], res["gate"][0]) and np.array_equal(res[name][1], res["gate"][1])
    idx = rng.choice(n, 300, replace=False)
    for i in idx[:40]:
        o = np.array([0, offs[i + 1] - offs[i]], np.uint64)
        assert np.array_equal(res["gate"][0][i], oracle.signatures(
            data[int(offs[i]):int(offs[i + 1])].copy(), o, oracle.derive_family(5, 128))[0])
    got = {}
    for name, env in {"ring": {}, "ring_gate": {"ND_K1J_RING_GATE": "1"}}.items():
        monkeypatch.delenv("ND_K1J_RING_GATE", raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        rep = pipeline.dedup_packed(data, offs, pipeline.RunConfig(), bucket_count=1000, ctx=ctx)
        sig = np.empty((n, 128), np.uint32)
        ctx.check(ctx.lib.nd_dedup_fetch_signatures(ctx.h, sig.ctypes.data_as(_lib.u32p), None))
        got[name] = (rep.stats["candidate_pairs"], sig)
    monkeypatch.delenv("ND_K1J_RING_GATE", raising=False)
    assert got["ring"][0] == got["ring_gate"][0]
    assert np.array_equal(got["ring"][1], res["gate"][0]) and np.array_equal(got["ring_gate"][1], res["gate"][0])


@pytest.mark.parametrize("seed,H,L", [(35, 128, 5), (8, 64, 3)])
@pytest.mark.parametrize("shape", [
    {},                                                        # dn, F=32, 4 CTAs, prefetch 2
    {"ND_K1J_ARITH": "fq"},                                    # fq, F=16, 6 CTAs
    {"ND_K1J_F": "16", "ND_K1J_MINB": "6", "ND_K1J_PREFETCH": "1"},  # round-2 dn shape
    {"ND_K1J_CLASSES": "1", "ND_K1J_F": "20"},                 # one w class, partial passes
    {"ND_K1J_SRING": "1"},                                     # text via a shared-memory ring
    {"ND_K1J_GPTR": "1", "ND_K1J_PFW": "40"},                  # __ldg words + L1 prefetch
])
def test_k1j_shapes_and_dn_misfits(ctx, oracle, monkeypatch, seed, H, L, shape):
    """families whose dn plan leaves one function to an fq pass of the same
    kernel (nd_k1j_plan: seed 35 at H=128/L=5, seed 8 at H=64/L=3), under the
    shipped shape and the knobs' other settings: identical to the oracle"""
    fam = minhash.derive_family(seed, H, L)
    plan = np.zeros((H, 12), np.uint32)
    assert ctx.lib.nd_k1j_plan(fam.functions, H, L, plan.ctypes.data_as(C.POINTER(C.c_uint32)),
                               H) == H
    if not shape:
        assert (plan[:, 2] == 0).sum() == 1  # one fq function
    rng = np.random.default_rng(seed)
    data, offs = _docs(rng, list(rng.integers(L, 5000, size=300)) + [L, L + 1, 30000])
    for k, v in shape.items():
        monkeypatch.setenv(k, v)
    ctx._family_key = None
    sig, _ = minhash.signatures_packed(data, offs, fam, 0, 0, 0, ctx=ctx, want_bands=False)
    assert _kernel(ctx) == "k1j"
    for k in shape:
        monkeypatch.delenv(k)
    ctx._family_key = None
    assert np.array_equal(sig, oracle.signatures(data, offs, oracle.derive_family(seed, H, L), L=L))


_ASCII = list("abcdefghijklmnop qrstuvwxyz")
_LATIN = [chr(c) for c in range(0xA0, 0x100)]
_BMP = ([chr(c) for c in range(0x400, 0x450)] + [chr(c) for c in range(0x4E00, 0x4E40)] +
        [chr(c) for c in range(0xAC00, 0xAC20)] + [chr(0xFFFD), chr(0xFFEE), chr(0x100)])
_ASTRAL = [chr(c) for c in range(0x1F600, 0x1F610)] + [chr(0x10FFFD), chr(0x10000)]


def _cp_corpus(rng, n, L, kinds):
    texts = []
    for i in range(n):
        k = int(rng.integers(L, 3000)) if i % 40 else 20000  # some multi-item documents
        if i % 97 == 5:
            k = L + i % 3  # documents of exactly L .. L+2 code points
        kind = kinds[i % len(kinds)]
        pool = {"ascii": _ASCII, "latin": _LATIN + _ASCII[:5], "bmp": _BMP + _ASCII[:8],
                "cjk": _BMP[80:144], "astral": _BMP + _ASTRAL}[kind]
        texts.append("".join(rng.choice(pool, size=k)))
    raw = [t.encode() for t in texts]
    offs = np.zeros(len(raw) + 1, np.uint64)
    offs[1:] = np.cumsum([len(b) for b in raw])
    return np.frombuffer(b"".join(raw), np.uint8).copy(), offs


@pytest.mark.parametrize("L,H,kinds", [
    (5, 128, ("bmp",)), (5, 128, ("cjk", "ascii", "bmp", "astral", "latin")),
    (1, 40, ("bmp", "astral")), (2, 64, ("cjk",)), (9, 128, ("bmp", "ascii")),
    (16, 100, ("cjk", "astral")),
])
def test_codepoint_bmp_documents_take_k1j16(ctx, oracle, monkeypatch, L, H, kinds):
    """documents whose code points are all < 2^16 (Cyrillic, CJK, Hangul,
    U+FFFD ...) run K1j over 16-bit units (fq arithmetic, c5 = 2^-3): every
    row equals the oracle and the K1w-only path, next to ASCII / Latin-1
    documents (byte K1j) and documents with supplementary code points (K1w)"""
    rng = np.random.default_rng(1000 * L + H)
    data, offs = _cp_corpus(rng, 240, L, kinds)
    fam = minhash.derive_family(7, H, L, minhash.ShingleUnit.CODEPOINT)
    bands = next(b for b in (16, 10, 8, 5, 4, 2, 1) if H % b == 0)
    res = {}
    for u16 in ("1", "0"):
        monkeypatch.setenv("ND_K1J_U16", u16)
        ctx._family_key = None
        res[u16] = minhash.signatures_packed(data, offs, fam, bands, H // bands, 997, ctx=ctx)
        assert _kernel(ctx) == ("k1j+k1j16+k1w" if u16 == "1" else "k1j+k1w")
    monkeypatch.delenv("ND_K1J_U16")
    ctx._family_key = None
    want = oracle.signatures(data, offs, oracle.derive_family(7, H, L), L=L, unit=1)
    assert np.array_equal(res["1"][0], want)
    assert np.array_equal(res["1"][0], res["0"][0]) and np.array_equal(res["1"][1], res["0"][1])


@pytest.mark.parametrize("layout", ["ascii", "ascii_short", "one_high_byte", "small_batch"])
def test_codepoint_pure_ascii_batch_runs_the_byte_path(ctx, oracle, monkeypatch, layout):
    """a codepoint batch without a byte >= 0x80 has units == bytes: it runs
    the byte path on the text as it is (no decode); one byte >= 0x80 anywhere
    sends the batch through the decode.  Both equal the oracle and the
    all-K1w path; documents shorter than L still raise ShortDocumentError"""
    rng = np.random.default_rng(7)
    texts = ["".join(rng.choice(_ASCII, size=int(k))) for k in rng.integers(5, 4000, size=300)]
    texts.append("x" * 20000)  # multi-item
    if layout == "one_high_byte":
        texts[150] = texts[150][:40] + "\u00e9" + texts[150][40:]
    if layout == "small_batch":
        texts = texts[:3]
    raw = [t.encode() for t in texts]
    if layout == "ascii_short":
        raw[7] = b"abc"
    offs = np.zeros(len(raw) + 1, np.uint64)
    offs[1:] = np.cumsum([len(b) for b in raw])
    data = np.frombuffer(b"".join(raw), np.uint8).copy()
    fam = minhash.derive_family(5, 128, 5, minhash.ShingleUnit.CODEPOINT)
    if layout == "ascii_short":
        with pytest.raises(minhash.ShortDocumentError):
            minhash.signatures_packed(data, offs, fam, 16, 8, 1000, ctx=ctx)
        return
    got = minhash.signatures_packed(data, offs, fam, 16, 8, 1000, ctx=ctx)
    monkeypatch.setenv("ND_K1_NARROW", "0")
    wide = minhash.signatures_packed(data, offs, fam, 16, 8, 1000, ctx=ctx)
    monkeypatch.delenv("ND_K1_NARROW")
    assert np.array_equal(got[0], wide[0]) and np.array_equal(got[1], wide[1])
    assert np.array_equal(got[0], oracle.signatures(data, offs, oracle.derive_family(5, 128), unit=1))
