"""CPU: the native dataset parser (csrc/dataset_io.cpp via datasets.load_dataset)
against the reference loader (datasets.py:81-167), case by case: the same CSR
arrays for accepted files, the same ParseError message and line for rejected
ones.  The reference is imported from /root/reference (present in this
container only; skipped elsewhere)."""
import sys
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2011_04235_b200 as fp
from paper_2011_04235_b200.validation import ParseError

REF_SRC = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def ref_load():
    if not (REF_SRC / "fastpi" / "__init__.py").exists():
        pytest.skip("reference package not present")
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import importlib
    return importlib.import_module("fastpi.datasets").load_dataset


def _outcome(loader, path):
    try:
        d = loader(path)
    except Exception as e:  # noqa: BLE001 -- the type and message are the comparison
        return ("err", type(e).__name__, str(e), getattr(e, "line", None))
    F, L = d.features.tocsr(), d.labels.tocsr()
    return ("ok", F.shape, F.indptr.tolist(), F.indices.tolist(), F.data.tolist(), L.shape, L.indptr.tolist(),
            L.indices.tolist())


BODIES = {
    "empty": "",
    "only_newline": "\n",
    "hdr_two": "1 2\n0 1:1\n",
    "hdr_four": "1 2 3 4\n",
    "hdr_alpha": "a 2 3\n",
    "hdr_neg": "1 -2 3\n0 1:1\n",
    "hdr_huge": "99999999999999999999 1 1\n",
    "hdr_huge_neg": "1 -99999999999999999999 1\n",
    "hdr_ws": "  2\t3   4  \n0 1:1\n1,2 0:2\n",
    "hdr_underscore_plus": "+2 1_0 0_3\n\n\n",
    "count_short": "3 2 2\n0 1:1\n",
    "count_long": "1 2 2\n0 1:1\n1 0:1\n",
    "trailing_blank": "1 2 2\n0 1:1\n\n",
    "crlf": "2 3 2\r\n1 0:1.5 2:2\r\n0\r\n",
    "cr_only": "2 3 2\r1 0:1.5\r0 2:3\r",
    "vt_ff_seps": "2 3 2\x0b1 0:1\x0c0 2:3\n",
    "unicode_sep": "2 3 2 1 0:1 0 2:3\n",
    "labels_unsorted": "1 4 5\n3,1,4 0:1\n",
    "labels_empty_tok": "1 4 5\n1,,2 0:1\n",
    "labels_dup": "1 4 5\n2,2 0:1\n",
    "labels_neg": "1 4 5\n-1 0:1\n",
    "labels_plus": "1 4 5\n+1 0:1\n",
    "labels_range": "1 4 5\n5 0:1\n",
    "labels_huge": "1 4 5\n123456789012345678901234 0:1\n",
    "labels_hex": "1 4 5\n0x1 0:1\n",
    "labels_tab": "1 4 5\n\t3 0:1\n",
    "labels_tab_inner": "1 4 5\n1\t2 0:1\n",
    "labels_underscore": "1 4 20\n1_0 0:1\n",
    "labels_only_no_space": "1 4 5\n1,2\n",
    "labels_colon_field": "1 4 5\n1:2\n",
    "labels_colon_field2": "1 4 5\n1:2 3:4\n",
    "feat_no_value": "1 4 2\n0 1:\n",
    "feat_no_colon": "1 4 2\n0 12\n",
    "feat_empty_index": "1 4 2\n0 :5\n",
    "feat_alpha": "1 4 2\n0 1:abc\n",
    "feat_two_colons": "1 4 2\n0 1:1:2\n",
    "feat_inf": "1 4 2\n0 1:inf\n",
    "feat_Infinity": "1 4 2\n0 1:-Infinity\n",
    "feat_nan": "1 4 2\n0 1:nan\n",
    "feat_zero": "1 4 2\n0 1:0\n",
    "feat_negzero": "1 4 2\n0 1:-0.0\n",
    "feat_underflow": "1 4 2\n0 1:1e-400\n",
    "feat_overflow": "1 4 2\n0 1:1e400\n",
    "feat_grouped": "1 4 2\n0 1:1_000.5 2:1_0e1_0\n",
    "feat_bad_group": "1 4 2\n0 1:1__0\n",
    "feat_hex": "1 4 2\n0 1:0x10\n",
    "feat_order": "1 4 2\n0 2:1 1:1\n",
    "feat_dup": "1 4 2\n0 1:1 1:2\n",
    "feat_range": "1 4 2\n0 4:1\n",
    "feat_neg_index": "1 4 2\n0 -1:1\n",
    "feat_forms": "1 9 2\n0 0:1. 1:.5 2:1e5 3:1E+5 4:+1 5:-2.5e-3 6:7 7:00012 08:3\n",
    "feat_dot_only": "1 4 2\n0 1:.\n",
    "feat_exp_only": "1 4 2\n0 1:1e\n",
    "multi_space": "1 4 2\n0   1:1    2:2   \n",
    "tab_features": "1 4 2\n0 1:1\t2:2\n",
    "unicode_token": "1 4 2\n0 1:é\n",
    "no_labels_features": "2 3 1\n 0:1 2:2\n\n",
    "valid_mix": "3 5 4\n0,3 0:1.25 4:-2\n\n2 1:3.5e-8\n",
}


@pytest.mark.parametrize("name", sorted(BODIES))
def test_parser_matches_reference(ref_load, tmp_path, name):
    path = tmp_path / f"{name}.txt"
    path.write_bytes(BODIES[name].encode("utf-8"))
    assert _outcome(fp.load_dataset, path) == _outcome(ref_load, path)


def test_random_roundtrips_match_reference(ref_load, tmp_path):
    rng = np.random.default_rng(7)
    for t in range(20):
        m, n, L = int(rng.integers(0, 40)), int(rng.integers(1, 30)), int(rng.integers(0, 12))
        X = sp.random(m, n, density=0.2, random_state=t, format="csr")
        X.data = rng.standard_normal(X.nnz) * 10.0 ** rng.integers(-12, 12, X.nnz)
        Y = sp.csr_matrix((rng.random((m, L)) < 0.3).astype(np.float64)) if L else sp.csr_matrix((m, 0))
        path = tmp_path / f"r{t}.txt"
        fp.save_dataset(fp.MultiLabelDataset(X, Y), path)
        mine = _outcome(fp.load_dataset, path)
        assert mine == _outcome(ref_load, path)
        assert mine[0] == "ok"
        got = fp.load_dataset(path)
        assert (got.features != X).nnz == 0 and (got.labels != Y).nnz == 0  # exact value round trip


def test_parse_error_carries_line(tmp_path):
    path = tmp_path / "bad.txt"
    path.write_text("2 3 2\n0 1:1\n1 2:0\n")
    with pytest.raises(ParseError) as ei:
        fp.load_dataset(path)
    assert ei.value.line == 3 and "explicit zero value for feature 2" in str(ei.value)


def test_from_matrix():
    d = fp.from_matrix(np.array([[0.0, 2.0], [3.0, 0.0]]))
    assert d.n_labels == 0 and d.n_instances == 2 and d.features.nnz == 2
