"""ctypes wrapper of integration/libtgc.so — the paper's GPU schemes (ranks-per-GPU tasked
cuBLAS, lock-step strided-batched cuBLAS) built from the reference's own host code.
Comparators for BASELINE.json config 5 only; never on the product path."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libtgc.so")

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_i64p = C.POINTER(C.c_int64)


class Comparators:
    def __init__(self, path: str = SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C integration libtgc.so)")
        self.lib = L = C.CDLL(path)
        L.tgc_last_error.restype = C.c_char_p
        L.tgc_tasked.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _dp, _dp, _u8p, _i64p]
        L.tgc_batched.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, _dp, _dp, _u8p, _i64p]

    def _run(self, fn, spins, steps, replicas, seed, *extra):
        init = np.zeros(replicas)
        ent = np.zeros((replicas, steps))
        acc = np.zeros((replicas, steps), np.uint8)
        wall = C.c_int64(0)
        rc = fn(spins, steps, replicas, seed, *extra, init.ctypes.data_as(_dp), ent.ctypes.data_as(_dp),
                acc.ctypes.data_as(_u8p), C.byref(wall))
        if rc != 0:
            raise RuntimeError(self.lib.tgc_last_error().decode())
        return {"initial": init, "entropies": ent, "accepted": acc, "wall_s": wall.value * 1e-9}

    def tasked(self, spins: int, steps: int, replicas: int, seed: int = 0, ranks: int = 16):
        """Ranks-per-GPU: `ranks` host threads (one stream + cuBLAS handle each) run the
        reference's mc_procedure for replicas p = r (mod ranks), every GEMM on the GPU."""
        return self._run(self.lib.tgc_tasked, spins, steps, replicas, seed, min(ranks, replicas))

    def batched(self, spins: int, steps: int, replicas: int, seed: int = 0):
        """batchedGEMM: all replicas in lock-step, one cublasZgemmStridedBatched per step."""
        return self._run(self.lib.tgc_batched, spins, steps, replicas, seed)
