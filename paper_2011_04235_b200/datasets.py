"""Dataset text format (datasets.py:1-186 of the reference): ``load_dataset``
through the library's native parser (`fpi_dataset_parse`, csrc/dataset_io.cpp),
``save_dataset`` and ``from_matrix`` on the host.

Format: first line ``m n L``; each of the m following lines is
``l1,l2,... f1:v1 f2:v2 ...`` (0-based label list, possibly empty, then
``index:value`` features with strictly increasing indices).

The parser accepts and rejects exactly what the reference loader does (the same
Python grammars for lines, whitespace, ``int()`` and ``float()``, the same check
order), and rejections raise ``ParseError`` with the reference's message and
1-based line number, rendered here from the token span the parser reports.
Deviation: the reference's ``save_dataset`` formats numpy scalars with ``repr``,
which under numpy >= 2 writes ``np.float64(1.5)`` -- text its own loader
rejects.  ``save_dataset`` here writes the value's Python-float ``repr``
(``1.5``), the form the format specifies and both loaders accept.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np
import scipy.sparse as sp

from . import _lib
from .regression import MultiLabelDataset
from .validation import ParseError, as_csr


DatasetInfo = _lib.DatasetInfo

(DS_OK, DS_EMPTY, DS_HEADER_SHAPE, DS_HEADER_INT, DS_HEADER_RANGE, DS_HEADER_NEG, DS_LINE_COUNT, DS_BAD_LABEL,
 DS_LABEL_RANGE, DS_LABEL_DUP, DS_FEAT_TOKEN, DS_FEAT_PARSE, DS_FEAT_RANGE, DS_FEAT_DUP, DS_FEAT_ORDER,
 DS_FEAT_NONFINITE, DS_FEAT_ZERO) = range(17)


def from_matrix(A) -> MultiLabelDataset:
    """datasets.py:62-65: a bare feature matrix as a dataset with zero labels."""
    A = as_csr(A).copy()
    A.sum_duplicates()
    A.eliminate_zeros()
    return MultiLabelDataset(A, sp.csr_matrix((A.shape[0], 0)))


def _parse_error(raw: bytes, info: DatasetInfo) -> ParseError:
    def tok(b, e):
        return raw[b:e].decode("utf-8")

    k, line = info.err_kind, info.err_line
    if k == DS_EMPTY:
        return ParseError(1, "empty file, expected 'm n L' header")
    if k in (DS_HEADER_SHAPE, DS_HEADER_INT, DS_HEADER_NEG, DS_HEADER_RANGE):
        text = tok(info.tok_begin, info.tok_end)
        if k == DS_HEADER_SHAPE:
            return ParseError(1, f"header must be 'm n L', got {text!r}")
        if k == DS_HEADER_INT:
            return ParseError(1, f"header must contain three integers, got {text!r}")
        m, n, L = (int(p) for p in text.split())  # beyond int64: Python integers, as the reference
        if m < 0 or n < 0 or L < 0:
            return ParseError(1, f"header counts must be non-negative, got {text!r}")
        return ParseError(info.n_lines, f"expected {m} instance lines after the header, found {info.n_lines - 1}")
    if k == DS_LINE_COUNT:
        return ParseError(line, f"expected {info.m} instance lines after the header, found {info.n_lines - 1}")
    t = tok(info.tok_begin, info.tok_end)
    if k == DS_BAD_LABEL:
        return ParseError(line, f"bad label index {t!r}")
    if k == DS_LABEL_RANGE:
        return ParseError(line, f"label index {int(t)} out of range [0, {info.L})")
    if k == DS_LABEL_DUP:
        return ParseError(line, f"duplicate label index {int(t)}")
    if k == DS_FEAT_TOKEN:
        return ParseError(line, f"bad feature token {t!r}, expected 'index:value'")
    if k == DS_FEAT_PARSE:
        return ParseError(line, f"bad feature token {t!r}")
    if k == DS_FEAT_RANGE:
        return ParseError(line, f"feature index {int(t)} out of range [0, {info.n})")
    if k == DS_FEAT_DUP:
        return ParseError(line, f"duplicate feature index {int(t)}")
    if k == DS_FEAT_ORDER:
        prev = int(tok(info.tok2_begin, info.tok2_end))
        return ParseError(line, f"feature indices must be strictly increasing, got {int(t)} after {prev}")
    if k == DS_FEAT_NONFINITE:
        return ParseError(line, f"non-finite feature value {t!r}")
    if k == DS_FEAT_ZERO:
        return ParseError(line, f"explicit zero value for feature {int(t)}")
    return ParseError(line, "malformed dataset")


def load_dataset(path) -> MultiLabelDataset:
    """datasets.py:81-167: parse a dataset file (native parser; ParseError on malformed input)."""
    raw = Path(path).read_bytes()
    raw.decode("utf-8")  # the reference reads the file as UTF-8 text (UnicodeDecodeError otherwise)
    lib = _lib.load()
    info = DatasetInfo()
    h = C.c_void_p()
    rc = lib.fpi_dataset_parse(raw, len(raw), C.byref(h), C.byref(info))
    if rc == _lib.FPI_EDOMAIN:
        raise _parse_error(raw, info)
    _lib.raise_for_status(rc, "dataset parser failed", "fpi_dataset_parse")
    try:
        m = info.m
        fptr = np.empty(m + 1, np.int64)
        fidx = np.empty(info.nnz_feat, np.int64)
        fval = np.empty(info.nnz_feat, np.float64)
        lptr = np.empty(m + 1, np.int64)
        lidx = np.empty(info.nnz_lab, np.int64)
        p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        _lib.raise_for_status(lib.fpi_dataset_fetch(h, p(fptr), p(fidx), p(fval), p(lptr), p(lidx)), "fetch")
    finally:
        lib.fpi_dataset_free(h)
    features = sp.csr_matrix((fval, fidx, fptr), shape=(m, info.n))
    labels = sp.csr_matrix((np.ones(info.nnz_lab), lidx, lptr), shape=(m, info.L))
    return MultiLabelDataset(features, labels)


def save_dataset(dataset: MultiLabelDataset, path):
    """datasets.py:170-186: the text format; values written as Python-float repr (exact round trip)."""
    F, Lb = dataset.features, dataset.labels
    out = [f"{dataset.n_instances} {dataset.n_features} {dataset.n_labels}"]
    for i in range(dataset.n_instances):
        labs = ",".join(map(str, np.sort(Lb.indices[Lb.indptr[i]:Lb.indptr[i + 1]]).tolist()))
        lo, hi = F.indptr[i], F.indptr[i + 1]
        feats = " ".join(f"{j}:{v!r}" for j, v in zip(F.indices[lo:hi].tolist(), F.data[lo:hi].tolist()))
        out.append(f"{labs} {feats}" if feats else labs)
    Path(path).write_text("\n".join(out) + "\n", encoding="utf-8")
