"""Document loader -- mirror of the reference's corpus.hpp / text.hpp (host side).

  parse_jsonl_line       corpus.cpp:31-54 (reject reasons verbatim)
  for_each_raw_document  corpus.cpp:56-82 (record ordinals count valid records)
  preprocess             corpus.cpp:93-101 (NFC, code point count, min_chars)
  can_shingle            corpus.cpp:103-107
  build_manifest         corpus.cpp:109-141 (sorted paths, record offsets)
  surviving_documents    corpus.cpp:143-163
NFC uses Python's unicodedata (the reference uses ICU); ill-formed UTF-8 is
replaced by U+FFFD first, as text.cpp:49-66 does.  This is host preprocessing
ahead of the GPU path, outside the hot path.
"""
from __future__ import annotations

import json
import os
import unicodedata
from dataclasses import dataclass, field

from . import _lib
from .minhash import CleanDocument, ShingleUnit


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


def parse_jsonl_line(line: str, text_field: str):
    try:
        j = json.loads(line)
    except ValueError:
        return False, None, "invalid_json"
    if not isinstance(j, dict):
        return False, None, "not_an_object"
    if text_field not in j:
        return False, None, "missing_text_field"
    if not isinstance(j[text_field], str):
        return False, None, "text_field_not_string"
    return True, j[text_field], None


def for_each_raw_document(path: str, file_ordinal: int, text_field: str, rejects, fn) -> int:
    try:
        fh = open(path, "rb")
    except OSError as e:
        raise _lib.IoError(_lib.ND_ERR_IO, f"cannot open '{path}': {e.strerror}")
    ordinal = 0
    with fh:
        for line_no, raw in enumerate(fh, start=1):
            line = raw.rstrip(b"\n")
            if line.endswith(b"\r"):
                line = line[:-1]
            if not line:
                continue
            ok, text, reason = parse_jsonl_line(line.decode("utf-8", errors="replace"), text_field)
            if not ok:
                if rejects is not None:
                    rejects.append((path, line_no, reason))
                continue
            fn(RawDocument(file_ordinal, ordinal, line_no, text))
            ordinal += 1
    return ordinal


def nfc_normalize(text: str) -> str:
    return unicodedata.normalize("NFC", text)


def preprocess(raw: RawDocument, min_chars: int, record_offset: int):
    text = nfc_normalize(raw.text)
    count = len(text)  # code points
    if count < min_chars:
        return None
    return CleanDocument(record_offset + raw.record_ordinal, text.encode("utf-8"), count)


def can_shingle(doc: CleanDocument, shingle_len: int, unit: ShingleUnit) -> bool:
    if shingle_len == 0:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "shingle length must be positive")
    units = len(doc.text) if unit == ShingleUnit.BYTE else doc.char_count
    return units >= shingle_len


def expand_inputs(inputs) -> list[str]:
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
    paths = sorted(expand_inputs(inputs))
    if not paths:
        raise _lib.ConfigError(_lib.ND_ERR_CONFIG, "no input files given")
    for a, b in zip(paths, paths[1:]):
        if a == b:
            raise _lib.ConfigError(_lib.ND_ERR_CONFIG, f"duplicate input file '{b}'")
    manifest = CorpusManifest()
    rejects = []
    offset = 0
    for i, p in enumerate(paths):
        st = FileStats(p, record_offset=offset)

        def visit(raw, st=st):
            doc = preprocess(raw, config.min_chars, st.record_offset)
            if doc is None:
                rejects.append((p, raw.line, "below_min_chars"))
            elif not can_shingle(doc, config.shingle_len, config.unit):
                rejects.append((p, raw.line, "too_short_to_shingle"))
            else:
                st.surviving += 1

        st.records = for_each_raw_document(p, i, config.text_field, rejects, visit)
        manifest.total_records += st.records
        manifest.total_surviving += st.surviving
        offset += st.records
        manifest.files.append(st)
    return manifest, rejects


def surviving_documents(manifest: CorpusManifest, index: int, config) -> list[CleanDocument]:
    st = manifest.files[index]
    docs = []

    def visit(raw):
        doc = preprocess(raw, config.min_chars, st.record_offset)
        if doc is not None and can_shingle(doc, config.shingle_len, config.unit):
            docs.append(doc)

    records = for_each_raw_document(st.path, index, config.text_field, None, visit)
    if records != st.records:
        raise _lib.PrerequisiteError(_lib.ND_ERR_PREREQ,
                                     f"'{st.path}' changed since the manifest was built")
    return docs
