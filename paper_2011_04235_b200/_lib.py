"""ctypes binding of libfastpi_b200.so (the C ABI declared in include/fastpi_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, every numerical entry point raises.  torch is used
only as device-memory / stream plumbing (tensors are handed to the library as
raw device pointers on the current torch stream).
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

from .validation import CapacityError, StructuralViolationError

LIB_PATH = Path(__file__).resolve().with_name("libfastpi_b200.so")

FPI_OK, FPI_EDOMAIN, FPI_ECAPACITY, FPI_ESTRUCT, FPI_ECUDA, FPI_ENUMERIC, FPI_ERETRY = range(7)


class RetryError(RuntimeError):
    """FPI_ERETRY: a speculative fast path did not apply; the caller repeats the call without it."""


i64 = C.c_int64
i32 = C.c_int32
f64 = C.c_double
vp = C.c_void_p
P_i64 = C.POINTER(C.c_int64)
P_u64 = C.POINTER(C.c_uint64)


class ReorderInfo(C.Structure):
    _fields_ = [("m1", i64), ("n1", i64), ("m2", i64), ("n2", i64),
                ("n_iterations", i64), ("n_spans", i64), ("n_gcc", i64), ("edges_visited", i64),
                ("nodes_visited", i64)]


class PartitionInfo(C.Structure):
    _fields_ = [("nnz_a11", i64), ("nnz_a12", i64), ("nnz_a21", i64), ("nnz_a22", i64)]


class BlockPlan(C.Structure):
    _fields_ = [("rank11", i64), ("nnz_u11", i64), ("nnz_vt11", i64),
                ("n_blocks_svd", i64), ("n_blocks_large", i64)]


class DatasetInfo(C.Structure):
    _fields_ = [("m", C.c_int64), ("n", C.c_int64), ("L", C.c_int64), ("nnz_feat", C.c_int64),
                ("nnz_lab", C.c_int64), ("n_lines", C.c_int64), ("err_kind", C.c_int32), ("pad_", C.c_int32),
                ("err_line", C.c_int64), ("tok_begin", C.c_int64), ("tok_end", C.c_int64),
                ("tok2_begin", C.c_int64), ("tok2_end", C.c_int64)]


class FastpiInfo(C.Structure):
    _fields_ = [("m", i64), ("n", i64), ("rank", i64), ("m1", i64), ("n1", i64), ("m2", i64), ("n2", i64),
                ("n_iterations", i64), ("n_spans", i64), ("rank11", i64), ("s", i64), ("row_engine", i32),
                ("col_engine", i32), ("rank_clamped", i32), ("all_filtered", i32), ("tolerance_used", f64),
                ("n_gcc", i64), ("edges_visited", i64), ("nodes_visited", i64)]


FASTPI_CANONICAL = 1  # fpi_fastpi_ex flag: the CSR is canonical already
FASTPI_DEFERRED_VALUES = 2  # fpi_fastpi_ex flag: d_values is still uploading (fpi_fastpi_values_hook)
VALUES_HOOK = C.CFUNCTYPE(C.c_int, vp, C.POINTER(vp))


class FastpiBuffers(C.Structure):
    _fields_ = [("U", vp), ("sigma", vp), ("Vt", vp), ("sigma_dagger", vp), ("row_fwd", vp), ("col_fwd", vp),
                ("spans", vp)]


class SvdDiag(C.Structure):
    _fields_ = [("engine", i32), ("cholqr_passes", i32), ("cond_estimate", f64),
                ("eig_sweeps", i32 * 4), ("null_completed", i32)]


# exchange callback of a sharded solve (fpi_comm_fn): (user, op, send, recv, count, root) -> status
COMM_FN = C.CFUNCTYPE(C.c_int, vp, C.c_int, vp, vp, i64, C.c_int)

# name -> (restype, argtypes); mirrors include/fastpi_b200.h
SIGNATURES = {
    "fpi_abi_version": (C.c_int, []),
    "fpi_create": (C.c_int, [C.POINTER(vp), C.c_int]),
    "fpi_destroy": (C.c_int, [vp]),
    "fpi_set_stream": (C.c_int, [vp, vp]),
    "fpi_last_error": (C.c_char_p, [vp]),
    "fpi_kernel_launches": (i64, [vp]),
    "fpi_get_svd_diag": (C.c_int, [vp, C.POINTER(SvdDiag)]),
    "fpi_sparse_core_info": (C.c_int, [vp, C.POINTER(C.c_int64)]),
    "fpi_csr_canonicalize": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp, vp, P_i64]),
    "fpi_csr_transpose": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp, vp]),
    "fpi_reorder": (C.c_int, [vp, i64, i64, i64, vp, vp, f64, vp, vp, C.POINTER(ReorderInfo)]),
    "fpi_reorder_fetch": (C.c_int, [vp, vp, P_i64]),
    "fpi_partition_count": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, i64, i64, i64, vp,
                                      C.POINTER(PartitionInfo)]),
    "fpi_partition": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp, i64, i64, i64, vp]
                      + [vp] * 15),
    "fpi_permute": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp]),
    "fpi_sketch_normal": (C.c_int, [vp, i64, i64, i64, vp, i64]),
    "fpi_pcg64_seed": (C.c_int, [i64, P_u64]),
    "fpi_gemm": (C.c_int, [vp, C.c_int, C.c_int, i64, i64, i64, f64, vp, i64, vp, i64, f64, vp, i64]),
    "fpi_spmm": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, f64, vp, i64, f64, vp, i64]),
    "fpi_cholesky": (C.c_int, [vp, i64, vp, i64]),
    "fpi_sym_eig": (C.c_int, [vp, i64, vp, i64, vp, vp, i64, C.POINTER(i32)]),
    "fpi_block_svd_plan": (C.c_int, [vp, i64, vp, f64, C.POINTER(BlockPlan)]),
    "fpi_block_svd": (C.c_int, [vp, i64, i64, vp, vp, vp, i64, vp, f64, vp, vp, vp, vp, vp, vp, vp,
                                C.POINTER(BlockPlan)]),
    "fpi_dense_svd": (C.c_int, [vp, i64, i64, vp, i64, i64, vp, vp, vp]),
    "fpi_randomized_svd": (C.c_int, [vp, i64, i64, vp, vp, vp, vp, vp, vp, i64, i64, vp, vp, vp]),
    "fpi_dataset_parse": (C.c_int, [C.c_char_p, i64, C.POINTER(vp), C.POINTER(DatasetInfo)]),
    "fpi_dataset_fetch": (C.c_int, [vp, vp, vp, vp, vp, vp]),
    "fpi_dataset_free": (C.c_int, [vp]),
    "fpi_topk_hits": (C.c_int, [vp, i64, i64, vp, i64, vp, vp, i32, vp]),
    "fpi_gram": (C.c_int, [vp, C.c_int, i64, i64, vp, i64, vp, i64]),
    "fpi_orth_factor": (C.c_int, [vp, i64, vp, vp, C.POINTER(f64)]),
    "fpi_scale_rows": (C.c_int, [vp, i64, i64, vp, i64, vp]),
    "fpi_canonical_signs": (C.c_int, [vp, i64, i64, i64, vp, i64, vp, i64]),
    "fpi_transpose": (C.c_int, [vp, i64, i64, vp, i64, vp, i64]),
    "fpi_row_update": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp, vp, vp, i64, vp, vp, vp, i64, f64, i64,
                                 vp, vp, vp, C.POINTER(i32)]),
    "fpi_column_update": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, i64, f64, i64,
                                    vp, vp, vp, C.POINTER(i32)]),
    "fpi_pinv_assemble": (C.c_int, [vp, i64, vp, i64, i64, f64, vp, C.POINTER(f64), C.POINTER(i32)]),
    "fpi_unfold": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp, vp]),
    "fpi_pinv_apply_csr": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp, i64, i64, vp, vp, vp, vp]),
    "fpi_pinv_apply_csr_host": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp, i64, i64, vp, vp, vp, vp]),
    "fpi_pinv_project_csr": (C.c_int, [vp, i64, i64, i64, vp, vp, i64, i64, i64, vp, vp, vp, vp]),
    "fpi_pinv_lift": (C.c_int, [vp, i64, i64, vp, vp, vp, i64, vp, vp]),
    "fpi_pinv_apply_dense": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, vp, vp, i64, vp, i64, vp]),
    "fpi_fastpi": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, f64, f64, i64, f64, f64, C.POINTER(FastpiInfo)]),
    "fpi_fastpi_get": (C.c_int, [vp] + [C.POINTER(vp)] * 6),
    "fpi_fastpi_release": (C.c_int, [vp]),
    "fpi_fastpi_ex": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, f64, f64, i64, f64, f64, i32,
                                C.POINTER(FastpiInfo)]),
    "fpi_fastpi_values_hook": (C.c_int, [vp, VALUES_HOOK, vp]),
    "fpi_fastpi_take": (C.c_int, [vp, C.POINTER(FastpiBuffers), C.POINTER(i64), i64, C.POINTER(C.c_float)]),
    "fpi_device_free": (C.c_int, [vp, vp]),
    "fpi_timing_enable": (C.c_int, [vp, C.c_int]),
    "fpi_timing_report": (C.c_int, [vp, C.c_char_p, i64, C.c_int]),
    "fpi_dmma_peak": (C.c_int, [vp, C.POINTER(f64)]),
    # sharded solve (csrc/comm.cu, csrc/sharded.cu)
    "fpi_comm_nccl_id": (C.c_int, [C.c_char_p, C.c_char_p, i64]),
    "fpi_comm_init_nccl": (C.c_int, [vp, C.c_char_p, C.c_int, C.c_int]),
    "fpi_comm_init_callback": (C.c_int, [vp, C.c_int, C.c_int, COMM_FN, vp]),
    "fpi_comm_init_self": (C.c_int, [vp]),
    "fpi_comm_free": (C.c_int, [vp]),
    "fpi_comm_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "fpi_comm_allreduce": (C.c_int, [vp, vp, i64]),
    "fpi_shard_plan": (C.c_int, [vp, i64, i64, i64, i64, i64, vp, vp, C.c_int, vp]),
    "fpi_block_svd_range": (C.c_int, [vp, i64, i64, vp, vp, vp, i64, vp, f64, i64, i64, vp, vp, vp, vp, vp, vp, vp,
                                      C.POINTER(BlockPlan), C.POINTER(i64)]),
    "fpi_row_update_shard": (C.c_int, [vp, i64, vp, vp, vp, vp, i64, i64, vp, vp, vp, i64, i64, vp, vp, vp, i64, i64,
                                       i64, i64, f64, i64, vp, vp, vp, vp]),
    "fpi_column_update_shard": (C.c_int, [vp, i64, i64, vp, vp, vp, i64, i64, vp, vp, vp, vp, vp, vp, i64, i64, i64,
                                          i64, f64, i64, vp, vp, vp]),
    "fpi_pinv_apply_shard": (C.c_int, [vp, i64, i64, i64, i64, i64, i64, i64, vp, vp, vp, i64, vp, i64, i64, vp, vp,
                                       vp, vp]),
}

_lib = None
_lib_lock = threading.Lock()


def load():
    """Load the shared library once (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH.name} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def exported_symbols():
    return sorted(SIGNATURES)


_handles = threading.local()


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2011_04235_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch


def handle():
    """Per-thread, per-device library handle bound to the current torch stream."""
    torch = _torch()
    lib = load()
    dev = torch.cuda.current_device()
    table = getattr(_handles, "table", None)
    if table is None:
        table = _handles.table = {}
    h = table.get(dev)
    if h is None:
        hp = vp()
        rc = lib.fpi_create(C.byref(hp), dev)
        if rc != FPI_OK:
            raise RuntimeError(f"fpi_create failed on device {dev} (code {rc})")
        h = table[dev] = hp
    lib.fpi_set_stream(h, vp(torch.cuda.current_stream().cuda_stream))
    return h


def raise_for_status(rc: int, msg: str, name: str = "") -> None:
    """Map a C-ABI status code to the reference's exception types (validation.py:22-35)."""
    if rc == FPI_OK:
        return
    if rc == FPI_EDOMAIN:
        raise ValueError(msg)
    if rc == FPI_ECAPACITY:
        raise CapacityError(msg)
    if rc == FPI_ESTRUCT:
        raise StructuralViolationError(msg)
    if rc == FPI_ERETRY:
        raise RetryError(msg)
    raise RuntimeError(f"{name}: {msg}" if name else msg)


def call(name, *args):
    """Invoke ``name(handle, *args)`` and map its status code to the reference's exceptions."""
    lib = load()
    h = handle()
    rc = getattr(lib, name)(h, *args)
    if rc != FPI_OK:
        raise_for_status(rc, lib.fpi_last_error(h).decode(errors="replace"), name)
    return h


def ptr(t):
    """Raw device pointer of a torch tensor (or None -> NULL)."""
    return None if t is None else vp(t.data_ptr())


def kernel_launches() -> int:
    return int(load().fpi_kernel_launches(handle()))


def svd_diag() -> dict:
    d = SvdDiag()
    load().fpi_get_svd_diag(handle(), C.byref(d))
    return {"engine": d.engine, "cholqr_passes": d.cholqr_passes, "cond_estimate": d.cond_estimate,
            "eig_sweeps": list(d.eig_sweeps), "null_completed": d.null_completed}


def sparse_core_info() -> dict:
    """Dense core of the last column update's sparse block (csrc/sparse_core.cu); zeros = plain SpMM."""
    v = (C.c_int64 * 4)()
    load().fpi_sparse_core_info(handle(), v)
    return {"rows": int(v[0]), "cols": int(v[1]), "core_nnz": int(v[2]), "rem_nnz": int(v[3])}


def timing_enable(on: bool = True):
    call("fpi_timing_enable", 1 if on else 0)


def timing_report(reset: bool = True) -> dict:
    """Per kernel class: launches, total ms, algorithmic flops and bytes (CUDA events)."""
    buf = C.create_string_buffer(1 << 16)
    call("fpi_timing_report", buf, len(buf), 1 if reset else 0)
    out = {}
    for line in buf.value.decode().splitlines():
        name, n, ms, fl, by = line.split("\t")
        out[name] = {"launches": int(n), "ms": float(ms), "flops": float(fl), "bytes": float(by)}
    return out


def dmma_peak_tflops() -> float:
    v = C.c_double(0.0)
    call("fpi_dmma_peak", C.byref(v))
    return float(v.value)
