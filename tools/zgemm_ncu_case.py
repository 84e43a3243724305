"""One batched ZGEMM of 1024^3 x 16 (ours, then cuBLAS via torch.bmm), twice each: the
workload of profiles/r01_ncu_zgemm_tma_1024.json.

    ncu --set full -k regex:zgemm_tma -c 1 python tools/zgemm_ncu_case.py
"""
import ctypes as C, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2203_09353_b200 as tg
L = tg.lib()
one = (C.c_double * 2)(1.0, 0.0); zero = (C.c_double * 2)(0.0, 0.0)
m = n = k = 1024; batch = 16
a = torch.randn(batch, k, m, dtype=torch.complex128, device="cuda")  # column-major m x k per entry
b = torch.randn(batch, n, k, dtype=torch.complex128, device="cuda")
out = torch.empty(batch, n, m, dtype=torch.complex128, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    rc = L.tg_zgemm_strided_launch(batch, m, n, k, one, C.c_void_p(a.data_ptr()), m * k, C.c_void_p(b.data_ptr()), k * n, zero, None, 0, C.c_void_p(out.data_ptr()), m * n, 0, C.c_void_p(st))
    torch.bmm(a, b)
torch.cuda.synchronize()
