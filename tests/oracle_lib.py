"""ctypes wrappers over the CPU checker libraries (TEST INFRASTRUCTURE ONLY).

- ``Oracle``  : oracle/liboracle.so, the C restatement (oracle/oracle.c)
- ``RefLib``  : oracle/_ref/libtgref.so, the unmodified reference sources + our
                C entry points (oracle/ref_driver.cpp); present only where it was
                built (this container, or shipped prebuilt to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libtgref.so")

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)


class CConfig(C.Structure):
    """tgo_config / tgr_config (oracle/oracle.h)."""

    _fields_ = [
        ("spins", C.c_int32),
        ("entropy_kind", C.c_int32),
        ("objective", C.c_int32),
        ("initial_state", C.c_int32),
        ("steps", C.c_uint64),
        ("seed", C.c_uint64),
        ("t0", C.c_double),
        ("t_min", C.c_double),
        ("renormalize_interval", C.c_uint64),
    ]


@dataclass
class McCfg:
    spins: int = 8
    steps: int = 1000
    seed: int = 0
    entropy_kind: int = 1  # 1 renyi-2 (bench default, bench.hpp:40), 0 von-neumann
    objective: int = 0  # 0 max, 1 min
    initial_state: int = 0  # 0 product, 1 random
    t0: float = 1.0
    t_min: float = 1e-3
    renormalize_interval: int = 1000

    def c(self) -> CConfig:
        return CConfig(self.spins, self.entropy_kind, self.objective, self.initial_state,
                       self.steps, self.seed, self.t0, self.t_min, self.renormalize_interval)


def _ptr(a, t):
    return a.ctypes.data_as(t) if a is not None else None


@dataclass
class Traces:
    initial: np.ndarray  # [P] f64
    entropies: np.ndarray  # [P, S] f64
    accepted: np.ndarray  # [P, S] u8
    sites: np.ndarray | None  # [P, S] u8


class Oracle:
    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        L = self.L = C.CDLL(path)
        L.tgo_stream_init.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64]
        L.tgo_next_u64.argtypes = [C.c_void_p]
        L.tgo_next_u64.restype = C.c_uint64
        L.tgo_haar.argtypes = [C.c_void_p, _dp]
        L.tgo_uniform_index.argtypes = [C.c_void_p, C.c_uint64]
        L.tgo_uniform_index.restype = C.c_uint64
        L.tgo_uniform01.argtypes = [C.c_void_p]
        L.tgo_uniform01.restype = C.c_double
        L.tgo_apply_gate.argtypes = [C.c_int, _dp, C.c_int, _dp, _dp]
        L.tgo_gemm.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
        L.tgo_entropy.argtypes = [C.c_int, _dp, C.c_int, _dp]
        L.tgo_temperature.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_uint64]
        L.tgo_temperature.restype = C.c_double
        L.tgo_acceptance.argtypes = [C.c_double, C.c_double]
        L.tgo_acceptance.restype = C.c_double
        L.tgo_hermitian_eigenvalues.argtypes = [C.c_int, _dp, _dp]
        L.tgo_mc_procedure.argtypes = [C.POINTER(CConfig), C.c_uint64, _dp, _dp, _u8p, _u8p, _dp, _dp]
        L.tgo_run_pool.argtypes = [C.POINTER(CConfig), C.c_uint64, C.c_uint64, C.c_int, _dp, _dp, _u8p, _u8p]
        L.tgo_average_entropy.argtypes = [C.c_uint64, C.c_uint64, _dp, _dp]
        L.tgo_average_entropy.restype = C.c_double

    def first_u64(self, seed: int, p: int, n: int) -> np.ndarray:
        st = (C.c_uint64 * 4)()
        self.L.tgo_stream_init(st, seed, p)
        return np.array([self.L.tgo_next_u64(st) for _ in range(n)], dtype=np.uint64)

    def haar(self, seed: int, p: int, count: int) -> np.ndarray:
        st = (C.c_uint64 * 4)()
        self.L.tgo_stream_init(st, seed, p)
        out = np.zeros((count, 32))
        for i in range(count):
            row = np.zeros(32)
            self.L.tgo_haar(st, _ptr(row, _dp))
            out[i] = row
        return out

    def haar_stream(self, spins: int, seed: int, p: int, steps: int, random_start: bool) -> np.ndarray:
        """The Haar unitaries of steps 0..steps-1 of replica p (draw order of spinmc.cpp:229-232,198-207)."""
        st = (C.c_uint64 * 4)()
        self.L.tgo_stream_init(st, seed, p)
        if random_start:
            for _ in range(2 << spins):
                self.L.tgo_next_u64(st)
        out = np.zeros((steps, 32))
        for i in range(steps):
            self.L.tgo_uniform_index(st, spins - 1)
            row = np.zeros(32)
            self.L.tgo_haar(st, _ptr(row, _dp))
            out[i] = row
            self.L.tgo_uniform01(st)
        return out

    def apply_gate(self, spins: int, psi: np.ndarray, site: int, u: np.ndarray) -> np.ndarray:
        psi = np.ascontiguousarray(psi, dtype=np.complex128)
        u = np.ascontiguousarray(u, dtype=np.complex128)
        out = np.zeros_like(psi)
        rc = self.L.tgo_apply_gate(spins, psi.ctypes.data_as(_dp), site, u.ctypes.data_as(_dp),
                                   out.ctypes.data_as(_dp))
        if rc != 0:
            raise ValueError("apply_two_site_gate: site out of range")
        return out

    def gemm(self, alpha, a, b, beta, c) -> np.ndarray:
        """a: (m,k), b: (k,n), c: (m,n) complex ndarrays (any order) -> column-major result."""
        m, k = a.shape
        n = b.shape[1]
        fa = np.asfortranarray(a, dtype=np.complex128)
        fb = np.asfortranarray(b, dtype=np.complex128)
        fc = np.asfortranarray(c, dtype=np.complex128)
        out = np.zeros((m, n), dtype=np.complex128, order="F")
        al = np.array([alpha.real, alpha.imag])
        be = np.array([beta.real, beta.imag])
        self.L.tgo_gemm(m, n, k, _ptr(al, _dp), fa.ctypes.data_as(_dp), fb.ctypes.data_as(_dp),
                        _ptr(be, _dp), fc.ctypes.data_as(_dp), out.ctypes.data_as(_dp))
        return out

    def entropy(self, spins: int, psi: np.ndarray, kind: int = 1) -> float:
        psi = np.ascontiguousarray(psi, dtype=np.complex128)
        e = C.c_double()
        if self.L.tgo_entropy(spins, psi.ctypes.data_as(_dp), kind, C.byref(e)) != 0:
            raise ValueError("entanglement_entropy: state not normalized")
        return e.value

    def temperature(self, t0, t_min, step, total):
        return self.L.tgo_temperature(t0, t_min, step, total)

    def acceptance(self, delta, t):
        return self.L.tgo_acceptance(delta, t)

    def mc_procedure(self, cfg: McCfg, p: int):
        init = C.c_double()
        ent = np.zeros(cfg.steps)
        acc = np.zeros(cfg.steps, np.uint8)
        sites = np.zeros(cfg.steps, np.uint8)
        u = np.zeros(cfg.steps)
        pr = np.zeros(cfg.steps)
        cc = cfg.c()
        rc = self.L.tgo_mc_procedure(C.byref(cc), p, C.byref(init), _ptr(ent, _dp), _ptr(acc, _u8p),
                                     _ptr(sites, _u8p), _ptr(u, _dp), _ptr(pr, _dp))
        if rc != 0:
            raise RuntimeError(f"tgo_mc_procedure rc={rc}")
        return init.value, ent, acc, sites, u, pr

    def run(self, cfg: McCfg, p0: int, count: int, threads: int = 0) -> Traces:
        threads = threads or (os.cpu_count() or 1)
        init = np.zeros(count)
        ent = np.zeros((count, cfg.steps))
        acc = np.zeros((count, cfg.steps), np.uint8)
        sites = np.zeros((count, cfg.steps), np.uint8)
        cc = cfg.c()
        rc = self.L.tgo_run_pool(C.byref(cc), p0, count, threads, _ptr(init, _dp), _ptr(ent, _dp),
                                 _ptr(acc, _u8p), _ptr(sites, _u8p))
        if rc != 0:
            raise RuntimeError(f"tgo_run_pool rc={rc}")
        return Traces(init, ent, acc, sites)


class RefLib:
    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.L = C.CDLL(path)
        L.tgr_last_error.restype = C.c_char_p
        L.tgr_first_u64.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _u64p]
        L.tgr_normal_pairs.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _dp]
        L.tgr_haar.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _dp]
        L.tgr_apply_gate.argtypes = [C.c_int, _dp, C.c_int, _dp, _dp]
        L.tgr_entropy.argtypes = [C.c_int, _dp, C.c_int, _dp]
        L.tgr_gemm.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
        L.tgr_hermitian_eigenvalues.argtypes = [C.c_int, _dp, _dp]
        L.tgr_temperature.argtypes = [C.c_double, C.c_double, C.c_uint64, C.c_uint64]
        L.tgr_temperature.restype = C.c_double
        L.tgr_acceptance.argtypes = [C.c_double, C.c_double]
        L.tgr_acceptance.restype = C.c_double
        L.tgr_run_pool.argtypes = [C.POINTER(CConfig), C.c_uint64, C.c_uint64, C.c_int, _dp, _dp, _u8p,
                                   _u8p, C.POINTER(C.c_int64)]
        L.tgr_time_sample.argtypes = [C.POINTER(CConfig), C.c_uint64, C.c_uint64, C.c_int,
                                      C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.tgr_run_experiment.argtypes = [C.POINTER(CConfig), C.c_uint64, C.c_uint64, C.c_char_p, _dp, _dp,
                                         _u8p, _dp, C.POINTER(C.c_int64)]

    def err(self) -> str:
        return self.L.tgr_last_error().decode()

    def first_u64(self, seed, p, n):
        out = np.zeros(n, np.uint64)
        self.L.tgr_first_u64(seed, p, n, out.ctypes.data_as(_u64p))
        return out

    def normal_pairs(self, seed, p, n):
        out = np.zeros((n, 2))
        self.L.tgr_normal_pairs(seed, p, n, out.ctypes.data_as(_dp))
        return out

    def haar(self, seed, p, count):
        out = np.zeros((count, 32))
        self.L.tgr_haar(seed, p, count, out.ctypes.data_as(_dp))
        return out

    def apply_gate(self, spins, psi, site, u):
        psi = np.ascontiguousarray(psi, dtype=np.complex128)
        u = np.ascontiguousarray(u, dtype=np.complex128)
        out = np.zeros_like(psi)
        if self.L.tgr_apply_gate(spins, psi.ctypes.data_as(_dp), site, u.ctypes.data_as(_dp),
                                 out.ctypes.data_as(_dp)) != 0:
            raise ValueError(self.err())
        return out

    def entropy(self, spins, psi, kind=1):
        psi = np.ascontiguousarray(psi, dtype=np.complex128)
        e = C.c_double()
        if self.L.tgr_entropy(spins, psi.ctypes.data_as(_dp), kind, C.byref(e)) != 0:
            raise ValueError(self.err())
        return e.value

    def gemm(self, alpha, a, b, beta, c):
        m, k = a.shape
        n = b.shape[1]
        fa = np.asfortranarray(a, dtype=np.complex128)
        fb = np.asfortranarray(b, dtype=np.complex128)
        fc = np.asfortranarray(c, dtype=np.complex128)
        out = np.zeros((m, n), dtype=np.complex128, order="F")
        al = np.array([alpha.real, alpha.imag])
        be = np.array([beta.real, beta.imag])
        if self.L.tgr_gemm(m, n, k, _ptr(al, _dp), fa.ctypes.data_as(_dp), fb.ctypes.data_as(_dp),
                           _ptr(be, _dp), fc.ctypes.data_as(_dp), out.ctypes.data_as(_dp)) != 0:
            raise ValueError(self.err())
        return out

    def run(self, cfg: McCfg, p0: int, count: int, threads: int = 0, sites: bool = True):
        threads = threads or (os.cpu_count() or 1)
        init = np.zeros(count)
        ent = np.zeros((count, cfg.steps))
        acc = np.zeros((count, cfg.steps), np.uint8)
        st = np.zeros((count, cfg.steps), np.uint8) if sites else None
        wall = C.c_int64()
        cc = cfg.c()
        rc = self.L.tgr_run_pool(C.byref(cc), p0, count, threads, _ptr(init, _dp), _ptr(ent, _dp),
                                 _ptr(acc, _u8p), _ptr(st, _u8p), C.byref(wall))
        if rc != 0:
            raise RuntimeError(f"reference run failed ({rc}): {self.err()}")
        return Traces(init, ent, acc, st), wall.value

    def time_sample(self, cfg: McCfg, p0: int, count: int, threads: int):
        """Pooled mc_procedure runs; per replica the total wall ns and the sum of its
        per-step wall times (ref_driver.cpp tgr_time_sample). Returns (total, steps, wall)."""
        total = np.zeros(count, np.int64)
        steps = np.zeros(count, np.int64)
        wall = C.c_int64()
        cc = cfg.c()
        rc = self.L.tgr_time_sample(C.byref(cc), p0, count, threads, _ptr(total, C.POINTER(C.c_int64)),
                                    _ptr(steps, C.POINTER(C.c_int64)), C.byref(wall))
        if rc != 0:
            raise RuntimeError(f"reference sample failed ({rc}): {self.err()}")
        return total, steps, wall.value

    def run_experiment(self, cfg: McCfg, procedures: int, devices: int = 1, mode: str = "cpu-reference"):
        init = np.zeros(procedures)
        ent = np.zeros((procedures, cfg.steps))
        acc = np.zeros((procedures, cfg.steps), np.uint8)
        avg = C.c_double()
        wall = C.c_int64()
        cc = cfg.c()
        rc = self.L.tgr_run_experiment(C.byref(cc), procedures, devices, mode.encode(), _ptr(init, _dp),
                                       _ptr(ent, _dp), _ptr(acc, _u8p), C.byref(avg), C.byref(wall))
        if rc != 0:
            raise RuntimeError(f"run_experiment failed ({rc}): {self.err()}")
        return Traces(init, ent, acc, None), avg.value, wall.value
