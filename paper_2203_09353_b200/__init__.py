"""taskgemm-b200: B200-native annealing Monte Carlo / small-GEMM hot path of arXiv 2203.09353.

Python binding over the in-tree C-ABI library ``libtaskgemm_b200.so``
(include/taskgemm_b200.h). The names mirror the reference's C++ interface
(/root/reference/proj/include/taskgemm/bench.hpp, exec.hpp, spinmc.hpp) so tests read like
the reference's own tests:

- ``ExperimentConfig`` / ``run_experiment``   = bench::ExperimentConfig / run_experiment
  (bench.hpp:28-45, 75) for the new ExecutionMode "device".
- ``EntropyTrace``                             = spinmc::EntropyTrace (spinmc.hpp:44-50) + sites.
- ``Device.batched_gemm``                     = exec::VirtualDevice::batched_gemm (exec.hpp:146).
- ``ConfigError`` / ``KernelError`` / ``SubmissionError`` mirror errors.hpp:9-12 and
  exec.hpp:66-86; precondition failures raise ``ValueError`` (std::invalid_argument).

There is no CPU fallback: on a machine without a CUDA device every compute entry point
raises ``DeviceUnavailable``. Loading the library (symbols only) works anywhere.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "ExperimentConfig", "RunReport", "EntropyTrace", "Device", "KernelRecord", "run_experiment",
    "ConfigError", "KernelError", "SubmissionError", "DeviceUnavailable", "lib", "step_flops",
    "dims_for_spins", "LIB_PATH", "NearTie",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtaskgemm_b200.so")

TG_OK, TG_ECONFIG, TG_EINVAL, TG_EKERNEL, TG_ESHUTDOWN, TG_ECUDA = range(6)


class ConfigError(RuntimeError):
    """taskgemm::ConfigError (errors.hpp:9-12); the CLI exits 2 on these."""


class KernelError(RuntimeError):
    """exec::KernelError: 'kernel failed for procedure N: ...' (exec.hpp:76-86)."""

    def __init__(self, msg: str):
        super().__init__(msg)
        try:
            self.procedure = int(msg.split("procedure ")[1].split(":")[0])
        except (IndexError, ValueError):
            self.procedure = -1


class SubmissionError(RuntimeError):
    """exec::SubmissionError (exec.hpp:66-69)."""


class DeviceUnavailable(RuntimeError):
    """No CUDA device / CUDA failure. The product path never falls back to the CPU."""


class CAnnealConfig(C.Structure):
    _fields_ = [
        ("spins", C.c_uint32), ("devices", C.c_uint32), ("steps", C.c_uint64),
        ("procedures", C.c_uint64), ("seed", C.c_uint64), ("entropy_kind", C.c_int32),
        ("objective", C.c_int32), ("initial_state", C.c_int32), ("inject_fault", C.c_int32),
        ("t0", C.c_double), ("t_min", C.c_double), ("renormalize_interval", C.c_uint64),
        ("shard_index", C.c_uint32), ("shard_count", C.c_uint32),
        ("fault_procedure", C.c_uint64), ("fault_step", C.c_uint64), ("rho_half", C.c_int32),
    ]


class CNearTie(C.Structure):
    """tg_near_tie: a logged accept decision with |u - p| < 1e-9."""

    _fields_ = [
        ("procedure", C.c_uint64), ("step", C.c_uint64), ("u", C.c_double), ("p", C.c_double),
        ("site", C.c_uint32), ("accepted", C.c_int32),
    ]


class CAnnealResult(C.Structure):
    _fields_ = [
        ("initial_entropy", C.POINTER(C.c_double)), ("entropies", C.POINTER(C.c_double)),
        ("accepted", C.POINTER(C.c_uint8)), ("sites", C.POINTER(C.c_uint8)),
        ("wall_ns", C.POINTER(C.c_int64)), ("final_entropy", C.POINTER(C.c_double)),
        ("average_entropy", C.c_double), ("total_wall_ns", C.c_int64),
        ("total_flops", C.c_uint64), ("kernel_ms", C.c_double),
        ("device_kernel_ms", C.POINTER(C.c_double)), ("device_resident", C.POINTER(C.c_uint64)),
        ("initial_wall_ns", C.POINTER(C.c_int64)), ("fallback_decisions", C.c_uint64),
        ("near_ties", C.c_uint64), ("near_tie_log", C.POINTER(CNearTie)), ("near_tie_capacity", C.c_uint64),
        ("executed_flops", C.c_uint64), ("nccl_ranks", C.c_uint32),
    ]


class CDeviceBuffers(C.Structure):
    _fields_ = [
        ("initial_entropy", C.c_void_p), ("entropies", C.c_void_p), ("accepted", C.c_void_p),
        ("sites", C.c_void_p), ("wall_ns", C.c_void_p), ("final_entropy", C.c_void_p),
        ("status", C.c_void_p), ("status_step", C.c_void_p), ("workspace", C.c_void_p),
        ("status_norm", C.c_void_p), ("initial_wall_ns", C.c_void_p), ("tie_stats", C.c_void_p), ("tie_log", C.c_void_p),
        ("tie_capacity", C.c_uint64),
    ]


class CKernelRecord(C.Structure):
    _fields_ = [
        ("device_id", C.c_uint64), ("procedure", C.c_uint64), ("m", C.c_uint64), ("n", C.c_uint64),
        ("k", C.c_uint64), ("queue_wait_ns", C.c_int64), ("exec_time_ns", C.c_int64),
        ("flops", C.c_uint64),
    ]


# Every symbol declared in include/taskgemm_b200.h (checked by tests/test_capi_symbols.py).
EXPORTS = [
    "tg_last_error", "tg_version", "tg_kernel_launches", "tg_create", "tg_shutdown", "tg_destroy", "tg_validate",
    "tg_anneal_rows", "tg_step_flops", "tg_anneal_run", "tg_anneal_launch",
    "tg_anneal_workspace_bytes", "tg_zgemm_batched", "tg_zgemm_strided_launch",
    "tg_fp64_dmma_peak", "tg_probe_rng", "tg_probe_gates", "tg_probe_apply_gate",
    "tg_probe_entropy", "tg_probe_entropy_kind", "tg_probe_phase_trace", "tg_probe_rng_chunking",
    "tg_rng_jump_words", "tg_rng_chunk_steps",
    "tg_set_perturb_gemm", "tg_hbm_schedule", "tg_probe_queue_stats",
]

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_lib = None


def _pin_nccl() -> None:
    """The C++ multi-GPU gather dlopen()s libnccl.so.2 by soname (capi.cpp nccl_api). If that
    resolved to the system NCCL before torch is imported, torch's own libtorch_cuda.so would then
    bind to it by the same soname and fail to load (missing newer symbols). Load the NCCL that
    torch ships with (pip nvidia-nccl) first, when it is installed, so there is one NCCL per process."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for root in (spec.submodule_search_locations or []) if spec else []:
        path = os.path.join(root, "nccl", "lib", "libnccl.so.2")
        if os.path.exists(path):
            try:
                C.CDLL(path, mode=C.RTLD_GLOBAL)
            except OSError:
                pass
            return


def lib() -> C.CDLL:
    """Load libtaskgemm_b200.so (fails loudly if it was not built: no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (make -C paper_2203_09353_b200/csrc)")
    _pin_nccl()
    L = C.CDLL(LIB_PATH)
    L.tg_last_error.restype = C.c_char_p
    L.tg_version.restype = C.c_char_p
    L.tg_kernel_launches.restype = C.c_uint64
    L.tg_create.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p)]
    L.tg_shutdown.argtypes = [C.c_void_p]
    L.tg_destroy.argtypes = [C.c_void_p]
    L.tg_validate.argtypes = [C.POINTER(CAnnealConfig)]
    L.tg_anneal_rows.argtypes = [C.POINTER(CAnnealConfig)]
    L.tg_anneal_rows.restype = C.c_uint64
    L.tg_step_flops.argtypes = [C.c_uint32]
    L.tg_step_flops.restype = C.c_uint64
    L.tg_anneal_run.argtypes = [C.c_void_p, C.POINTER(CAnnealConfig), C.POINTER(CAnnealResult)]
    L.tg_anneal_launch.argtypes = [C.POINTER(CAnnealConfig), C.POINTER(CDeviceBuffers), C.c_void_p]
    L.tg_anneal_workspace_bytes.argtypes = [C.POINTER(CAnnealConfig)]
    L.tg_anneal_workspace_bytes.restype = C.c_size_t
    L.tg_zgemm_batched.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp,
                                   C.POINTER(_dp), C.POINTER(_dp), _dp, C.POINTER(_dp), C.POINTER(_dp),
                                   C.POINTER(C.c_uint64), C.POINTER(CKernelRecord)]
    L.tg_zgemm_strided_launch.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.c_void_p, C.c_int64,
                                          C.c_void_p, C.c_int64, _dp, C.c_void_p, C.c_int64, C.c_void_p,
                                          C.c_int64, C.c_int, C.c_void_p]
    L.tg_fp64_dmma_peak.argtypes = [C.c_int, _dp, _dp]
    L.tg_probe_rng.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
    L.tg_probe_gates.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, _u8p, _dp, _dp]
    L.tg_probe_apply_gate.argtypes = [C.c_uint32, _dp, C.c_int, _dp, _dp]
    L.tg_probe_entropy.argtypes = [C.c_uint32, C.c_uint64, _dp, _dp, _dp]
    L.tg_probe_entropy_kind.argtypes = [C.c_uint32, C.c_uint64, _dp, C.c_int32, _dp, _dp]
    L.tg_set_perturb_gemm.argtypes = [C.c_int]
    L.tg_hbm_schedule.argtypes = [C.c_uint32, C.c_uint64, C.c_int32]
    L.tg_probe_queue_stats.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_int32, C.POINTER(C.c_int64),
                                       C.POINTER(C.c_int)]
    L.tg_probe_phase_trace.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.POINTER(C.c_int64)]
    L.tg_probe_rng_chunking.argtypes = [C.c_uint32, C.c_uint64, C.c_uint64, C.c_int32, C.c_uint64,
                                        C.POINTER(C.c_uint64)]
    L.tg_rng_chunk_steps.restype = C.c_uint64
    L.tg_rng_jump_words.argtypes = [C.c_uint64, C.c_uint64, C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64,
                                    C.POINTER(C.c_uint64)]
    for name in EXPORTS:
        if name not in ("tg_last_error", "tg_version", "tg_kernel_launches", "tg_anneal_rows", "tg_step_flops",
                        "tg_anneal_workspace_bytes"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc == TG_OK:
        return
    msg = lib().tg_last_error().decode()
    if rc == TG_ECONFIG:
        raise ConfigError(msg)
    if rc == TG_EINVAL:
        raise ValueError(msg)
    if rc == TG_EKERNEL:
        raise KernelError(msg)
    if rc == TG_ESHUTDOWN:
        raise SubmissionError(msg)
    raise DeviceUnavailable(msg)


def dims_for_spins(spins: int) -> tuple[int, int]:
    """spinmc::dims_for_spins (spinmc.cpp:15-26): (d_a, d_b); GEMM (M,N,K) = (d_a, d_a, d_b)."""
    if spins < 2 or spins > 30:
        raise ConfigError(f"spins out of range [2,30]: {spins}")
    return 1 << (spins // 2), 1 << (spins - spins // 2)


def step_flops(spins: int) -> int:
    """gemm_flops(d_a, d_a, d_b) = 8*d_a^2*d_b of one step (linalg.cpp:140-144)."""
    return int(lib().tg_step_flops(spins))


_ENTROPY = {"von-neumann": 0, "renyi-2": 1}
_OBJECTIVE = {"max": 0, "min": 1}
_INITIAL = {"product": 0, "random": 1}


@dataclass
class ExperimentConfig:
    """bench::ExperimentConfig (bench.hpp:28-45) workload fields + McConfig.renormalize_interval."""

    spins: int = 6
    steps: int = 100
    procedures: int = 1
    devices: int = 1
    entropy_kind: str = "renyi-2"
    objective: str = "max"
    t0: float = 1.0
    t_min: float = 1e-3
    initial_state: str = "product"
    seed: int = 0
    renormalize_interval: int = 1000
    shard_index: int = 0
    shard_count: int = 1
    inject_fault: int = 0       # 1: perturb_gemm (linalg.hpp:74-79); 2: non-unitary gate (below)
    fault_procedure: int = 0    # inject_fault == 2: this procedure's gate at fault_step is scaled by 1.001
    fault_step: int = 0
    rho_half: bool = False      # opt-in Hermitian half of rho (Renyi-2): executed flops reported apart

    def to_c(self) -> CAnnealConfig:
        for name, table in (("entropy_kind", _ENTROPY), ("objective", _OBJECTIVE),
                            ("initial_state", _INITIAL)):
            if getattr(self, name) not in table:
                raise ConfigError(f"unknown {name}: {getattr(self, name)!r}")
        if self.procedures < 0 or self.steps < 0 or self.devices < 0:
            raise ConfigError("counts must be non-negative")
        return CAnnealConfig(self.spins, self.devices, self.steps, self.procedures, self.seed & (2**64 - 1),
                             _ENTROPY[self.entropy_kind], _OBJECTIVE[self.objective],
                             _INITIAL[self.initial_state], int(self.inject_fault), self.t0, self.t_min,
                             self.renormalize_interval, self.shard_index, self.shard_count,
                             self.fault_procedure, self.fault_step, int(bool(self.rho_half)))

    def rows(self) -> int:
        c = self.to_c()
        return int(lib().tg_anneal_rows(C.byref(c)))

    def validate(self) -> None:
        """bench::validate (bench.cpp:321-329) plus the device-tier limits."""
        c = self.to_c()
        _check(lib().tg_validate(C.byref(c)))


@dataclass
class EntropyTrace:
    procedure_index: int
    initial_entropy: float
    entropies: np.ndarray
    accepted_flags: np.ndarray
    sites: np.ndarray | None = None
    wall_times: np.ndarray | None = None


@dataclass
class RunReport:
    """bench::RunReport (bench.hpp:54-62), arrays instead of per-trace vectors."""

    config: ExperimentConfig
    procedures: np.ndarray           # procedure index of each row
    initial_entropy: np.ndarray      # [rows]
    entropies: np.ndarray            # [rows, steps]
    accepted: np.ndarray             # [rows, steps] u8
    sites: np.ndarray | None
    wall_ns: np.ndarray | None
    final_entropy: np.ndarray
    average_entropy: float
    total_wall_ns: int
    total_flops: int
    kernel_ms: float
    traces: list = field(default_factory=list)
    device_kernel_ms: list = field(default_factory=list)  # per GPU of the context
    device_resident: list = field(default_factory=list)   # replicas resident at once per GPU
    initial_wall_ns: np.ndarray | None = None             # [rows] (wall=True)
    fallback_decisions: int = 0  # decisions re-taken with the reference formula (lean margin in the window)
    near_ties: int = 0           # decisions with |u - p| < 1e-9
    near_tie_log: list = field(default_factory=list)  # NearTie, (procedure, step) order
    executed_flops: int = 0      # GEMM flops executed on the device (< total_flops with rho_half)
    nccl_ranks: int = 0          # GPUs of the NCCL all-gather of the finals (0: host copies)

    def trace(self, row: int) -> EntropyTrace:
        return EntropyTrace(int(self.procedures[row]), float(self.initial_entropy[row]),
                            self.entropies[row], self.accepted[row].astype(bool),
                            None if self.sites is None else self.sites[row],
                            None if self.wall_ns is None else self.wall_ns[row])


@dataclass
class NearTie:
    """tg_near_tie: accept test u < p (spinmc.cpp:207) with |u - p| < 1e-9."""

    procedure: int
    step: int
    u: float
    p: float
    site: int
    accepted: bool


@dataclass
class KernelRecord:
    """exec::KernelRecord (exec.hpp:46-55)."""

    device_id: int
    procedure: int
    m: int
    n: int
    k: int
    queue_wait_ns: int
    exec_time_ns: int
    flops: int


class Device:
    """A context over one or more GPUs (owns streams and device buffers)."""

    def __init__(self, gpus: list[int] | int | None = None):
        L = lib()
        if gpus is None:
            gpus = [0]
        elif isinstance(gpus, int):
            gpus = list(range(gpus))
        arr = (C.c_int * len(gpus))(*gpus)
        h = C.c_void_p()
        _check(L.tg_create(arr, len(gpus), C.byref(h)))
        self._h = h
        self.gpus = list(gpus)

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().tg_destroy(self._h)
            self._h = None

    def shutdown(self) -> None:
        _check(lib().tg_shutdown(self._h))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def run(self, cfg: ExperimentConfig, sites: bool = True, wall: bool = False,
            out: dict | None = None, near_tie_capacity: int = 256) -> RunReport:
        """The device annealing driver (tg_anneal_run). `out` may supply preallocated (pinned)
        host arrays keyed initial/entropies/accepted/sites/final. A state that leaves
        normalization raises ValueError (std::invalid_argument, spinmc.cpp:152-156)."""
        c = cfg.to_c()
        _check(lib().tg_validate(C.byref(c)))
        rows = int(lib().tg_anneal_rows(C.byref(c)))
        steps = cfg.steps
        out = out or {}
        init = out.get("initial", np.zeros(rows))
        ent = out.get("entropies", np.zeros((rows, steps)))
        acc = out.get("accepted", np.zeros((rows, steps), np.uint8))
        st = out.get("sites", np.zeros((rows, steps), np.uint8)) if sites else None
        wl = np.zeros((rows, steps), np.int64) if wall else None
        fin = out.get("final", np.zeros(rows))
        res = CAnnealResult()
        res.initial_entropy = init.ctypes.data_as(_dp)
        res.entropies = ent.ctypes.data_as(_dp)
        res.accepted = acc.ctypes.data_as(_u8p)
        res.sites = st.ctypes.data_as(_u8p) if st is not None else None
        res.wall_ns = wl.ctypes.data_as(C.POINTER(C.c_int64)) if wl is not None else None
        res.final_entropy = fin.ctypes.data_as(_dp)
        dms = (C.c_double * max(cfg.devices, 1))()
        res.device_kernel_ms = C.cast(dms, C.POINTER(C.c_double))
        drs = (C.c_uint64 * max(cfg.devices, 1))()
        res.device_resident = C.cast(drs, C.POINTER(C.c_uint64))
        iw = np.zeros(rows, np.int64) if wall else None
        res.initial_wall_ns = iw.ctypes.data_as(C.POINTER(C.c_int64)) if iw is not None else None
        log = (CNearTie * max(near_tie_capacity, 1))()
        res.near_tie_log = C.cast(log, C.POINTER(CNearTie)) if near_tie_capacity > 0 else None
        res.near_tie_capacity = near_tie_capacity
        _check(lib().tg_anneal_run(self._h, C.byref(c), C.byref(res)))
        procs = cfg.shard_index + np.arange(rows, dtype=np.int64) * max(cfg.shard_count, 1)
        ties = [NearTie(t.procedure, t.step, t.u, t.p, t.site, bool(t.accepted))
                for t in log[:min(res.near_ties, near_tie_capacity)]]
        return RunReport(cfg, procs, init, ent, acc, st, wl, fin, res.average_entropy, res.total_wall_ns,
                         res.total_flops, res.kernel_ms, device_kernel_ms=list(dms[:max(cfg.devices, 1)]),
                         device_resident=list(drs[:max(cfg.devices, 1)]), initial_wall_ns=iw,
                         fallback_decisions=res.fallback_decisions, near_ties=res.near_ties, near_tie_log=ties,
                         executed_flops=res.executed_flops, nccl_ranks=res.nccl_ranks)

    def batched_gemm(self, a_list, b_list, c_list=None, alpha=1.0, beta=0.0, device: int = 0,
                     procedures=None, records: bool = False):
        """exec::VirtualDevice::batched_gemm (exec.hpp:146): fixed-size batch, results ordered as
        inputs. Matrices are complex 2-D arrays (any memory order)."""
        if len(a_list) == 0:
            raise ValueError("batched_gemm: batch must be non-empty")
        shapes = {(a.shape[0], b.shape[1], a.shape[1]) for a, b in zip(a_list, b_list)}
        if len(shapes) != 1 or len(a_list) != len(b_list) or (c_list is not None and len(c_list) != len(a_list)):
            raise ValueError("batched_gemm: fixed-size contract violated, batch mixes GEMM shapes")
        m, n, k = shapes.pop()
        for a, b in zip(a_list, b_list):
            if a.shape[1] != b.shape[0]:
                raise ValueError(f"gemm: A.cols ({a.shape[1]}) != B.rows ({b.shape[0]})")
        if c_list is not None:
            for cc in c_list:
                if cc.shape != (m, n):
                    raise ValueError(f"gemm: C.rows ({cc.shape[0]}) != A.rows ({m})")
        batch = len(a_list)
        fa = [np.asfortranarray(a, dtype=np.complex128) for a in a_list]
        fb = [np.asfortranarray(b, dtype=np.complex128) for b in b_list]
        fc = [np.asfortranarray(c, dtype=np.complex128) for c in c_list] if c_list is not None else None
        outs = [np.zeros((m, n), np.complex128, order="F") for _ in range(batch)]
        P = lambda arrs: (_dp * batch)(*[x.ctypes.data_as(_dp) for x in arrs])  # noqa: E731
        al = np.array([complex(alpha).real, complex(alpha).imag])
        be = np.array([complex(beta).real, complex(beta).imag])
        procs = (C.c_uint64 * batch)(*(procedures if procedures is not None else range(batch)))
        recs = (CKernelRecord * batch)()
        _check(lib().tg_zgemm_batched(self._h, device, batch, m, n, k, al.ctypes.data_as(_dp), P(fa), P(fb),
                                      be.ctypes.data_as(_dp), P(fc) if fc is not None else None, P(outs),
                                      procs, recs))
        if records:
            return outs, [KernelRecord(r.device_id, r.procedure, r.m, r.n, r.k, r.queue_wait_ns,
                                       r.exec_time_ns, r.flops) for r in recs]
        return outs


def run_experiment(cfg: ExperimentConfig) -> RunReport:
    """bench::run_experiment (bench.cpp:341-417) in ExecutionMode "device": procedure p is bound to
    GPU p mod devices; traces depend only on (seed, workload)."""
    cfg.validate()
    with Device(cfg.devices) as dev:
        return dev.run(cfg)


# ----------------------------------------------------------------- device-piece probes
def probe_rng(seed: int, p: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.uint64)
    _check(lib().tg_probe_rng(seed & (2**64 - 1), p, n, out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return out


def probe_gates(spins: int, seed: int, p: int, steps: int, initial_state: str = "product"):
    sites = np.zeros(steps, np.uint8)
    u = np.zeros((steps, 32))
    ua = np.zeros(steps)
    _check(lib().tg_probe_gates(spins, seed & (2**64 - 1), p, steps, _INITIAL[initial_state],
                                sites.ctypes.data_as(_u8p), u.ctypes.data_as(_dp), ua.ctypes.data_as(_dp)))
    return sites, u, ua


def probe_apply_gate(spins: int, psi: np.ndarray, site: int, u: np.ndarray) -> np.ndarray:
    psi = np.ascontiguousarray(psi, np.complex128)
    u = np.ascontiguousarray(u, np.complex128)
    out = np.zeros_like(psi)
    _check(lib().tg_probe_apply_gate(spins, psi.ctypes.data_as(_dp), site, u.ctypes.data_as(_dp),
                                     out.ctypes.data_as(_dp)))
    return out


def probe_entropy(spins: int, states: np.ndarray, kind: str = "renyi-2"):
    """Device entropy (and ||psi||) of host states [count, 2^spins] through the anneal
    kernels' rho path; kind "renyi-2" or "von-neumann"."""
    if kind not in _ENTROPY:
        raise ConfigError(f"unknown entropy_kind: {kind!r}")
    states = np.ascontiguousarray(states, np.complex128).reshape(-1, 1 << spins)
    e = np.zeros(states.shape[0])
    n = np.zeros(states.shape[0])
    _check(lib().tg_probe_entropy_kind(spins, states.shape[0], states.ctypes.data_as(_dp), _ENTROPY[kind],
                                       e.ctypes.data_as(_dp), n.ctypes.data_as(_dp)))
    return e, n


def probe_phase_trace(spins: int, replicas: int, steps: int) -> np.ndarray:
    """clock64 phase stamps [steps, 8] of CTA 0's first replica (profiling only)."""
    out = np.zeros((steps, 8), np.int64)
    _check(lib().tg_probe_phase_trace(spins, replicas, steps, out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out


def probe_rng_chunking(spins: int, rows: int, steps: int, random_init: bool = False,
                       reject_below: int = 0) -> int:
    """Differing draw words + sites between the chunked jump-ahead pre-pass and one
    sequential stream per replica (0 = identical); reject_below > 0 forces rejections."""
    mm = C.c_uint64()
    _check(lib().tg_probe_rng_chunking(spins, rows, steps, int(random_init), reject_below, C.byref(mm)))
    return int(mm.value)


def rng_jump_words(seed: int, p: int, chunks: int, extra: int = 0, n: int = 4, init_spins: int = -1) -> np.ndarray:
    """Host (no GPU): stream words after the pre-pass's GF(2) jumps (tg_rng_jump_words)."""
    out = np.zeros(n, np.uint64)
    _check(lib().tg_rng_jump_words(seed, p, init_spins, chunks, extra, n, out.ctypes.data_as(C.POINTER(C.c_uint64))))
    return out


def kernel_launches() -> int:
    """Kernels the library has launched in this process (tg_kernel_launches)."""
    return int(lib().tg_kernel_launches())


def fp64_dmma_peak(device: int = 0) -> tuple[float, float]:
    t = C.c_double()
    g = C.c_double()
    _check(lib().tg_fp64_dmma_peak(device, C.byref(t), C.byref(g)))
    return t.value, g.value
