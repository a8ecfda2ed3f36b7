"""FP64 DMMA GEMM throughput on the c4/c5 shapes (CUDA events, L2-cold for big operands)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2011_04235_b200 import _lib  # noqa: E402

SHAPES = [  # (name, ta, tb, M, N, K)
    ("gram_BtB_c4", 1, 0, 1000, 1000, 200000),
    ("U_eq_B_Mx_c4", 0, 0, 200000, 500, 1000),
    ("B_eq_U_X1_c4", 0, 0, 200000, 1000, 399),
    ("DtB_c4", 1, 0, 399, 1000, 200000),
    ("Z_VtT_WT_c4", 1, 1, 50000, 4000, 500),
    ("gram_Yt_c4", 1, 0, 1000, 1000, 10684),
    ("square_4096", 0, 0, 4096, 4096, 4096),
    ("Y_eq_U_X_c5", 0, 0, 2000000, 2000, 1000),
    ("gram_YtY_c5", 1, 0, 2000, 2000, 2000000),
    ("YtU_c5", 1, 0, 2000, 1000, 2000000),
    ("U_eq_Y_X_c5", 0, 0, 2000000, 1000, 2000),
    ("Gram_NT_c4", 0, 1, 1000, 1000, 200000),
    ("HH_TN_c5", 1, 0, 256, 256, 2000000),
    ("H11_TN_c5", 1, 0, 939, 939, 349000),
    ("H21h_TN_c5", 1, 0, 256, 939, 349000),
    ("Z_L_NT_c4", 0, 1, 10684, 1000, 1000),
    ("XtZ_c4_odd", 1, 0, 399, 1000, 8497),   # lda = 399: the s-wide operands of c4's row update
    ("XtZ_c4_even", 1, 0, 400, 1000, 8497),
    ("WZ_c4_odd", 0, 0, 6491, 399, 798),
    ("G_c4_odd", 1, 0, 798, 798, 6491),
]


def main():
    only = sys.argv[1:]
    for name, ta, tb, M, N, K in SHAPES:
        if only and name not in only:
            continue
        A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda")
        B = torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device="cuda")
        C = torch.empty((M, N), dtype=torch.float64, device="cuda")
        args = (ta, tb, M, N, K, 1.0, _lib.ptr(A), A.shape[1], _lib.ptr(B), B.shape[1], 0.0, _lib.ptr(C), N)
        _lib.call("fpi_gemm", *args)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            _lib.call("fpi_gemm", *args)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        ref = (A.t() if ta else A) @ (B.t() if tb else B)
        err = (C - ref).abs().max().item() / ref.abs().max().item()
        e0.record()
        for _ in range(reps):
            torch.matmul(A.t() if ta else A, B.t() if tb else B, out=C)
        e1.record()
        torch.cuda.synchronize()
        ms_cublas = e0.elapsed_time(e1) / reps
        print(f"{name:16s} M={M} N={N} K={K}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.2f} TFLOP/s  relerr {err:.1e}  "
              f"(cuBLAS {2*M*N*K/ms_cublas/1e9:.2f} TFLOP/s)", flush=True)
        A = B = C = ref = None
        A = B = C = ref = None


if __name__ == "__main__":
    main()
