"""Document loader -- mirror of the reference's corpus.hpp / text.hpp, backed by
the multi-threaded C++ loader of libneardup_b200 (csrc/host_ingest.cpp):

  parse_jsonl_line       corpus.cpp:31-54 (the reference's parser, nlohmann::json)
  for_each_raw_document  corpus.cpp:56-82 (record ordinals count valid records)
  nfc_normalize          text.cpp:70-86 (U+FFFD for ill-formed UTF-8, then UAX #15 NFC)
  codepoint_count        text.cpp:88-99
  preprocess             corpus.cpp:93-101 (NFC, code point count, min_chars)
  can_shingle            corpus.cpp:103-107
  build_manifest         corpus.cpp:109-141 (sorted paths, record offsets, reject log)
  build_manifest_cached  the same scan keeping the packed text of the files that
                         fit a host-memory cap (no second parse for those)
  surviving_documents    corpus.cpp:143-163
  surviving_packed       the same documents as one packed batch (text + offsets +
                         doc ids), the input the GPU stages take
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import u8p, u32p, u64p
from .minhash import CleanDocument, ShingleUnit

REASONS = {1: "invalid_json", 2: "not_an_object", 3: "missing_text_field",
           4: "text_field_not_string", 5: "below_min_chars", 6: "too_short_to_shingle"}


@dataclass
class RawDocument:
    file_ordinal: int
    record_ordinal: int
    line: int
    text: str


@dataclass
class FileStats:
    path: str
    records: int = 0
    surviving: int = 0
    record_offset: int = 0


@dataclass
class CorpusManifest:
    files: list[FileStats] = field(default_factory=list)
    total_records: int = 0
    total_surviving: int = 0


def _check(rc: int) -> None:
    if rc != _lib.ND_OK:
        lib = _lib.load()
        raise _lib.ERRORS.get(rc, _lib.NdError)(rc, lib.nd_ingest_last_error().decode(errors="replace"))


def _b(t: bytes | str) -> bytes:
    return t.encode("utf-8", errors="surrogatepass") if isinstance(t, str) else bytes(t)


def parse_jsonl_line(line: bytes | str, text_field: str):
    """-> (ok, text bytes or None, reason or None)."""
    lib = _lib.load()
    raw = _b(line)
    reason, n = C.c_uint32(), C.c_uint64()
    _check(lib.nd_parse_jsonl_line(raw, len(raw), text_field.encode(), C.byref(reason), None, 0,
                                   C.byref(n)))
    if reason.value:
        return False, None, REASONS[reason.value]
    out = (C.c_uint8 * max(1, n.value))()
    _check(lib.nd_parse_jsonl_line(raw, len(raw), text_field.encode(), C.byref(reason), out,
                                   n.value, C.byref(n)))
    return True, bytes(out[:n.value]), None


def for_each_raw_document(path: str, file_ordinal: int, text_field: str, rejects, fn) -> int:
    """corpus.cpp:56-82: valid records in order (record ordinals count valid
    records), malformed lines to `rejects` as (path, line, reason); returns the
    record count.  The bulk loader is JsonlFile; this is the per-record API."""
    try:
        fh = open(path, "rb")
    except OSError as e:
        raise _lib.IoError(_lib.ND_ERR_IO, f"cannot open '{path}': {e.strerror}")
    ordinal = 0
    with fh:
        for line_no, raw in enumerate(fh, start=1):
            line = raw[:-1] if raw.endswith(b"\n") else raw
            if line.endswith(b"\r"):
                line = line[:-1]
            if not line:
                continue
            ok, text, reason = parse_jsonl_line(line, text_field)
            if not ok:
                if rejects is not None:
                    rejects.append((path, line_no, reason))
                continue
            fn(RawDocument(file_ordinal, ordinal, line_no, text))
            ordinal += 1
    return ordinal


def load_jsonl_file(path: str, file_ordinal: int, text_field: str, rejects=None) -> list[RawDocument]:
    """corpus.cpp:84-91."""
    docs = []
    for_each_raw_document(path, file_ordinal, text_field, rejects, docs.append)
    return docs


def nfc_normalize(text: bytes | str) -> bytes:
    lib = _lib.load()
    raw = _b(text)
    src = (C.c_uint8 * max(1, len(raw))).from_buffer_copy(raw or b"\0")
    n = C.c_uint64()
    _check(lib.nd_nfc_normalize(src, len(raw), None, 0, C.byref(n)))
    out = (C.c_uint8 * max(1, n.value))()
    _check(lib.nd_nfc_normalize(src, len(raw), out, n.value, C.byref(n)))
    return bytes(out[:n.value])


def codepoint_count(text: bytes | str) -> int:
    raw = _b(text)
    src = (C.c_uint8 * max(1, len(raw))).from_buffer_copy(raw or b"\0")
    return int(_lib.load().nd_codepoint_count(src, len(raw)))


def preprocess(raw: RawDocument, min_chars: int, record_offset: int):
    text = nfc_normalize(raw.text)
    count = codepoint_count(text)
    if count < min_chars:
        return None
    return CleanDocument(record_offset + raw.record_ordinal, text, count)


def can_shingle(doc: CleanDocument, shingle_len: int, unit: ShingleUnit) -> bool:
    if shingle_len == 0:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "shingle length must be positive")
    units = len(_b(doc.text)) if unit == ShingleUnit.BYTE else doc.char_count
    return units >= shingle_len


class JsonlFile:
    """One parsed + preprocessed JSONL file (nd_jsonl_load)."""

    def __init__(self, path: str, config, keep_text: bool, threads: int = 0):
        lib = self.lib = _lib.load()
        h = C.c_void_p()
        _check(lib.nd_jsonl_load(path.encode(), config.text_field.encode(), config.min_chars,
                                 config.shingle_len, int(config.unit), threads, int(keep_text),
                                 C.byref(h)))
        self.h = h
        r, s, nb, nr = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        lib.nd_jsonl_counts(h, C.byref(r), C.byref(s), C.byref(nb), C.byref(nr))
        self.records, self.surviving, self.text_bytes, self.nrejects = r.value, s.value, nb.value, nr.value

    def rejects(self):
        lines = np.empty(self.nrejects, np.uint64)
        reasons = np.empty(self.nrejects, np.uint32)
        if self.nrejects:
            _check(self.lib.nd_jsonl_rejects(self.h, lines.ctypes.data_as(u64p),
                                             reasons.ctypes.data_as(u32p)))
        return [(int(a), REASONS[int(b)]) for a, b in zip(lines, reasons)]

    def packed(self, record_offset: int):
        n = self.surviving
        data = np.empty(self.text_bytes, np.uint8)
        offsets = np.empty(n + 1, np.uint64)
        ids = np.empty(n, np.uint64)
        chars = np.empty(n, np.uint64)
        _check(self.lib.nd_jsonl_documents(self.h, record_offset,
                                           data.ctypes.data_as(u8p) if data.size else None,
                                           offsets.ctypes.data_as(u64p), ids.ctypes.data_as(u64p),
                                           chars.ctypes.data_as(u64p)))
        return data, offsets, ids, chars

    def close(self):
        if self.h:
            self.lib.nd_jsonl_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


def expand_inputs(inputs) -> list[str]:
    """pipeline.cpp:79-99: files as given, directories -> sorted *.jsonl."""
    paths = []
    for entry in inputs:
        if os.path.isdir(entry):
            found = sorted(os.path.join(entry, f) for f in os.listdir(entry)
                           if f.endswith(".jsonl") and os.path.isfile(os.path.join(entry, f)))
            paths.extend(found)
        elif os.path.isfile(entry):
            paths.append(entry)
        else:
            raise _lib.IoError(_lib.ND_ERR_IO, f"input '{entry}' does not exist")
    return paths


def build_manifest(inputs, config):
    """-> (CorpusManifest, rejects [(path, line, reason)] in file and line order)."""
    manifest, rejects, _ = build_manifest_cached(inputs, config, 0)
    return manifest, rejects


def _host_memory_bytes() -> int:
    try:
        return os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        return 0


def default_text_cache_bytes() -> int:
    """How much preprocessed text the stages keep between the manifest scan and
    hashing: a quarter of the free host memory, at most 32 GiB."""
    return min(_host_memory_bytes() // 4, 32 << 30)


def build_manifest_cached(inputs, config, keep_text_bytes: int):
    """build_manifest that keeps the parsed, NFC-normalised text of the first
    files whose texts fit in `keep_text_bytes`, so the stages pack them without
    the reference's second parse of every file (corpus.cpp:143-163 re-reads
    what corpus.cpp:109-141 already read).  -> (manifest, rejects,
    {file index: packed (text, offsets, doc ids, char counts)})."""
    paths = sorted(expand_inputs(inputs))
    if not paths:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "no input files given")
    for a, b in zip(paths, paths[1:]):
        if a == b:
            raise _lib.ConfigError(_lib.ND_ERR_CONFIG, f"duplicate input file '{b}'")
    manifest = CorpusManifest()
    rejects = []
    offset = 0
    cache = {}
    for i, p in enumerate(paths):
        keep = keep_text_bytes > 0 and len(cache) == i
        f = JsonlFile(p, config, keep_text=keep)
        st = FileStats(p, f.records, f.surviving, offset)
        rejects.extend((p, line, why) for line, why in f.rejects())
        if keep and f.text_bytes <= keep_text_bytes:
            cache[i] = f.packed(offset)
            keep_text_bytes -= f.text_bytes
        f.close()
        manifest.total_records += st.records
        manifest.total_surviving += st.surviving
        offset += st.records
        manifest.files.append(st)
    return manifest, rejects, cache


def surviving_packed(manifest: CorpusManifest, index: int, config):
    """File `index`'s surviving documents as (text u8, offsets[n+1] u64, doc_ids u64,
    char_counts u64), doc_id = record_offset + record ordinal."""
    if index >= len(manifest.files):
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "manifest file index out of range")
    st = manifest.files[index]
    f = JsonlFile(st.path, config, keep_text=True)
    if f.records != st.records:
        raise _lib.PrerequisiteError(_lib.ND_ERR_PREREQ,
                                     f"'{st.path}' changed since the manifest was built "
                                     f"({f.records} records, manifest says {st.records})")
    out = f.packed(st.record_offset)
    f.close()
    return out


def surviving_documents(manifest: CorpusManifest, index: int, config) -> list[CleanDocument]:
    data, offsets, ids, chars = surviving_packed(manifest, index, config)
    return [CleanDocument(int(ids[i]), bytes(data[int(offsets[i]):int(offsets[i + 1])]), int(chars[i]))
            for i in range(len(ids))]
