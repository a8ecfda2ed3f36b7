import ctypes as C
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2011_04235_b200 import _lib
lib = _lib.load()
h = _lib.handle()
fn = lib.fpi_dbg_subsolve_bench
fn.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double)]
v = C.c_double()
for it in (10, 200, -200):
    fn(h, it, C.byref(v))
    print(f"iters={it} ({'all 31' if it > 0 else 'cross 16'} steps): {v.value:.1f} ns per step")
