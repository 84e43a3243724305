"""Batched ZGEMM (the GEMM batcher's device path, tg_zgemm_strided_launch) vs cuBLAS
(torch.bmm on complex128 = cublasZgemmStridedBatched) on device-resident operands.

    python tools/zgemm_bench.py
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09353_b200 as tg  # noqa: E402

L = tg.lib()
dev = torch.device("cuda:0")
one = (C.c_double * 2)(1.0, 0.0)
zero = (C.c_double * 2)(0.0, 0.0)


def ours(a, b, out, m, n, k, batch):
    # column-major interleaved: A[i + p*m] of entry e at 2*(sA*e + ...) doubles
    st = torch.cuda.current_stream().cuda_stream
    rc = L.tg_zgemm_strided_launch(batch, m, n, k, one, C.c_void_p(a.data_ptr()), m * k, C.c_void_p(b.data_ptr()),
                                   k * n, zero, None, 0, C.c_void_p(out.data_ptr()), m * n, 0, C.c_void_p(st))
    assert rc == 0, tg.lib().tg_last_error()


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


peak, _ = tg.fp64_dmma_peak(0)
for m, batch in ((64, 4096), (128, 2048), (256, 256), (512, 64), (1024, 16)):
    n = k = m
    a = torch.randn(batch, k, m, dtype=torch.complex128, device=dev)  # column-major m x k per entry
    b = torch.randn(batch, n, k, dtype=torch.complex128, device=dev)
    out = torch.empty(batch, n, m, dtype=torch.complex128, device=dev)
    t_ours = timeit(lambda: ours(a, b, out, m, n, k, batch))
    at, bt = a.transpose(1, 2), b.transpose(1, 2)  # row-major views of the same matrices
    ref = torch.bmm(at, bt)
    err = (out.transpose(1, 2) - ref).abs().max().item() / ref.abs().max().item()
    t_cublas = timeit(lambda: torch.bmm(at, bt))
    fl = 8.0 * m * n * k * batch
    print(f"{m:5d}^3 x {batch:5d}: ours {fl / t_ours / 1e12:6.2f} TF ({fl / t_ours / 1e12 / peak:5.1%} of DMMA peak), "
          f"cuBLAS {fl / t_cublas / 1e12:6.2f} TF, max rel err {err:.1e}")
