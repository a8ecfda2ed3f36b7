"""CPU: the C-ABI library loads and exports every symbol include/fastpi_b200.h declares."""
import re
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "fastpi_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(fpi_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2011_04235_b200 import _lib
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    # the Python binding covers the whole header
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert lib.fpi_abi_version() == 1


def test_seedsequence_pcg64_state_matches_numpy():
    import ctypes as C
    from paper_2011_04235_b200 import _lib
    lib = _lib.load()
    for seed in [0, 1, 2, 3, 4, 5, 6, 7, 42, 2**31 - 1, 2**32 + 5, 2**40 + 3]:
        out = (C.c_uint64 * 4)()
        assert lib.fpi_pcg64_seed(seed, out) == 0
        st = np.random.PCG64(seed).state["state"]
        assert (out[0] << 64 | out[1]) == st["state"], seed
        assert (out[2] << 64 | out[3]) == st["inc"], seed
