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
sizes = ((64, 4096), (96, 2048), (128, 2048), (192, 512), (256, 256), (512, 64), (1024, 16))
for m, batch in sizes:
    n = k = m
    a = torch.randn(batch, k, m, dtype=torch.complex128, device=dev)  # column-major m x k per entry
    b = torch.randn(batch, n, k, dtype=torch.complex128, device=dev)
    out = torch.empty(batch, n, m, dtype=torch.complex128, device=dev)
    fl = 8.0 * m * n * k * batch
    res, outs = {}, {}
    for w in ("4", "5", "8", "9", "16", "default"):
        if w == "default":
            os.environ.pop("TG_ZGEMM_WARPS", None)
        else:
            os.environ["TG_ZGEMM_WARPS"] = w
        t = timeit(lambda: ours(a, b, out, m, n, k, batch))
        res[w] = fl / t / 1e12
        outs[w] = out.clone()
    os.environ.pop("TG_ZGEMM_WARPS", None)
    same = all(torch.equal(outs[w].view(torch.float64), outs["8"].view(torch.float64)) for w in outs)
    at, bt = a.transpose(1, 2), b.transpose(1, 2)  # row-major views of the same matrices
    ref = torch.bmm(at, bt)
    err = (out.transpose(1, 2) - ref).abs().max().item() / ref.abs().max().item()
    t_cublas = timeit(lambda: torch.bmm(at, bt))
    cub = fl / t_cublas / 1e12
    print(f"{m:5d}^3 x {batch:5d}: ours {res['default']:6.2f} TF ({res['default'] / peak:5.1%} of DMMA peak, "
          f"{res['default'] / cub:6.1%} of cuBLAS) [4w {res['4']:.2f}, 4w+producer {res['5']:.2f}, 8w {res['8']:.2f}, 8w+producer {res['9']:.2f}, 16w {res['16']:.2f}], "
          f"cuBLAS {cub:6.2f} TF, variants bitwise equal: {same}, max rel err {err:.1e}")

# ---- the GEMM batcher's public API with HOST buffers (tg_zgemm_batched: copies in, kernel,
# copies out; exec.hpp:146 ownership) vs the same through torch/cuBLAS (pinned host stack
# -> device -> bmm -> host)
import time  # noqa: E402

import numpy as np  # noqa: E402

_dp = C.POINTER(C.c_double)
ctx = C.c_void_p()
gpus = (C.c_int * 1)(0)
assert L.tg_create(gpus, 1, C.byref(ctx)) == 0
for m, batch in ((64, 4096), (256, 256)):
    n = k = m
    rng = np.random.default_rng(m)
    A = [np.asfortranarray(rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))) for _ in range(batch)]
    B = [np.asfortranarray(rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))) for _ in range(batch)]
    O = [np.zeros((m, n), np.complex128, order="F") for _ in range(batch)]
    P = lambda arrs: (_dp * batch)(*[x.ctypes.data_as(_dp) for x in arrs])  # noqa: E731
    pa, pb, po = P(A), P(B), P(O)
    al = (C.c_double * 2)(1.0, 0.0)
    be = (C.c_double * 2)(0.0, 0.0)

    def api():
        rc = L.tg_zgemm_batched(ctx, 0, batch, m, n, k, al, pa, pb, be, None, po, None, None)
        assert rc == 0, L.tg_last_error()

    ha = torch.from_numpy(np.stack([a.T for a in A])).pin_memory()  # row-major A^T stacks
    hb = torch.from_numpy(np.stack([b.T for b in B])).pin_memory()

    def via_torch():
        out = torch.bmm(hb.to(dev, non_blocking=True), ha.to(dev, non_blocking=True)).cpu()  # (AB)^T
        return out

    for fn in (api, via_torch):
        fn()
    t = {}
    for name, fn in (("api", api), ("torch", via_torch)):
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        t[name] = (time.perf_counter() - t0) / reps
    ref = via_torch().numpy()
    err = max(np.abs(O[i] - ref[i].T).max() for i in range(0, batch, max(1, batch // 8)))
    fl = 8.0 * m * n * k * batch
    print(f"API host buffers {m}^3 x {batch}: tg_zgemm_batched {t['api'] * 1e3:8.2f} ms ({fl / t['api'] / 1e12:5.2f} TF), "
          f"torch pinned->bmm->host {t['torch'] * 1e3:8.2f} ms ({fl / t['torch'] / 1e12:5.2f} TF), max abs diff {err:.1e}")
L.tg_destroy(ctx)
