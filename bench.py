"""Benchmark: annealing replica-steps/s of the B200 hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 4|1|2|3|5] [--scaling strong|weak] [--mc-steps M] [--replicas R]

`--gpus N` with N > 1 re-executes itself under torch.distributed.run (one process per GPU,
127.0.0.1 rendezvous) unless it already runs under torchrun; the world size must equal N.

One bench "step" = one full persistent-kernel anneal of the workload: every replica of
this GPU runs all MC steps (gate -> rho = Psi Psi^dagger on DMMA -> Renyi-2 -> Metropolis),
inputs = (seed, config) only, all state resident on the device. Default workload =
BASELINE.json configs[3], the north_star's "largest chain config at 1 GPU": L=20
(1024x1024x1024 complex GEMMs), 512 replicas, 100 MC steps.

Scaling. Configs 3 and 4 are fixed totals (4096 / 512 replicas "across 8 B200"): the
default for them is strong scaling, replica p on rank p mod N (bench.cpp:171). Configs 1,
2 and 5 are per-GPU batches (weak scaling). `--scaling` overrides. Either way there is no
data-path collective: the final entropies are all-gathered once (NCCL) for the
procedure-order average and the best replica.

`value`  : replica-steps/s over all ranks, device time (CUDA events on the launch stream,
           max over ranks), L2 flushed (256 MiB write) between timed iterations.
`e2e`    : same metric through the public C-ABI call tg_anneal_run with host buffers
           (kernel-argument H2D + trace D2H into pinned memory) + the NCCL gather, wall time.
`roofline`: FP64 DMMA roofline of the anneal launch; peak = live DMMA.8x8x4 probe
           (MEASURED_PEAKS.json has no FP64 entry), committed in profiles/.
`cpu_baseline` / `--impl reference`: the reference's own CPU path (oracle/_ref:
           spinmc::mc_procedure + DirectExecutor, pooled over all host threads) on a bounded
           sample of the same workload (one replica per host thread, k MC steps), extrapolated
           linearly in steps to the whole workload (bench::extrapolate_runtime,
           bench.cpp:429-438), rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "annealing steps/sec (all replicas, whole box) and FP64 TFLOP/s vs DMMA roofline"
UNIT = "replica-steps/s"

CONFIGS = {  # BASELINE.json configs; `replicas` is the total (strong) or per GPU (weak)
    1: dict(spins=8, replicas=64, mc_steps=1000, scaling="weak", name="config1: L=8, 64 replicas/GPU, 1000 MC steps"),
    2: dict(spins=12, replicas=1024, mc_steps=10000, scaling="weak",
            name="config2: L=12, 1024 replicas/GPU, 10000 MC steps"),
    # configs 3/4: BASELINE.json leaves the step count open; SURVEY.md §8(d) fixes 1000 / 100
    3: dict(spins=16, replicas=4096, mc_steps=1000, scaling="strong",
            name="config3: L=16 (256x256 GEMMs), 4096 replicas, 1000 MC steps"),
    4: dict(spins=20, replicas=512, mc_steps=100, scaling="strong",
            name="config4: L=20 (1024x1024 GEMMs), 512 replicas, 100 MC steps"),
    5: dict(spins=14, replicas=65536, mc_steps=100, scaling="weak", name="config5: L=14, 65536 replicas/GPU, 100 MC steps"),
}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def gemm_mnk(spins):
    da, db = 1 << (spins // 2), 1 << (spins - spins // 2)
    return [da, da, db]


def step_flops(spins):
    m, n, k = gemm_mnk(spins)
    return 8 * m * n * k  # gemm_flops (linalg.cpp:140-144)


def workload(args, world):
    """The workload both arms run and report (identical `config` dicts)."""
    cfgw = dict(CONFIGS[args.config])
    if args.mc_steps:
        cfgw["mc_steps"] = args.mc_steps
    if args.replicas:
        cfgw["replicas"] = args.replicas
    scaling = args.scaling or cfgw["scaling"]
    procedures = cfgw["replicas"] if scaling == "strong" else cfgw["replicas"] * world
    name = cfgw["name"]
    if args.mc_steps or args.replicas or scaling != cfgw["scaling"]:
        name = (f"config{args.config} variant: L={cfgw['spins']}, {cfgw['replicas']} replicas"
                f"{'' if scaling == 'strong' else '/GPU'}, {cfgw['mc_steps']} MC steps")
    config = {
        "workload": name, "spins": cfgw["spins"], "gemm_mnk": gemm_mnk(cfgw["spins"]), "procedures": procedures,
        "replicas_per_gpu": (procedures + world - 1) // world, "mc_steps": cfgw["mc_steps"],
        "parallelism": f"dp{world} (replica p on GPU p mod {world})", "entropy": args.entropy,
        "initial_state": "product", "seed": 0, "objective": "max",
        "l2": "flushed between timed iterations (256 MiB write)",
    }
    return cfgw["spins"], procedures, cfgw["mc_steps"], scaling, config


class ClockSampler:
    """nvidia-smi clocks and throttle reasons DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        if not getattr(self, "lines", []):  # a timed region shorter than the 100 ms sampling period
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                      "-i", str(self.gpu)], capture_output=True, text=True, timeout=10).stdout
                self.lines = [ln for ln in out.splitlines() if ln.strip()]
                self.post_run = True
            except (OSError, subprocess.TimeoutExpired):
                pass
        sm, mx, reasons = [], 0.0, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, f[3:]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        out = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}
        if getattr(self, "post_run", False):
            out["note"] = "timed region shorter than the 100 ms sampling period: one reading right after it"
        return out


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def est_step_seconds(spins):
    """A-priori single-core cost of one reference step (the triple-loop GEMM
    runs at ~2.7 GFLOP/s up to S = 16 and ~1.2 GFLOP/s at S = 20, plus O(2^S) copies)."""
    rate = 2.7e9 if spins <= 16 else 1.2e9
    return step_flops(spins) / rate + (1 << spins) * 1e-7


def cpu_reference_sample(spins, procedures, mc_steps, threads, target_s=10.0, entropy_kind=1):
    """Time the reference's own CPU path (oracle/_ref: spinmc::mc_procedure + DirectExecutor,
    pooled host threads) on a bounded sample — one replica per host thread (procedures
    0..threads-1 of the workload), k MC steps — and extrapolate linearly in steps to the whole
    workload (bench::extrapolate_runtime, bench.cpp:429-438): a thread runs
    ceil(procedures / threads) replicas, each = initial state + entropy (measured) + mc_steps
    steps (measured per-step wall time, EntropyTrace::wall_times). Falls back to the oracle
    port (timed the same way, whole runs) if _ref is absent."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import REF_SO, McCfg, Oracle, RefLib  # checker / baseline only

    kind = "reference" if os.path.exists(REF_SO) else "port"
    n_rep = int(min(procedures, threads))
    k = int(max(1, min(mc_steps, math.floor(target_s / est_step_seconds(spins)))))
    cfg = McCfg(spins=spins, steps=k, entropy_kind=entropy_kind)
    t0 = time.perf_counter()
    if kind == "reference":
        total, steps_ns, _ = RefLib().time_sample(cfg, 0, n_rep, threads)
        t_step = float(np.mean(steps_ns)) / k / 1e9
        t_init = float(np.mean(total - steps_ns)) / 1e9
    else:
        o = Oracle()
        a = time.perf_counter()
        o.run(McCfg(spins=spins, steps=0, entropy_kind=entropy_kind), 0, n_rep, threads=threads)
        t_init = time.perf_counter() - a
        a = time.perf_counter()
        o.run(cfg, 0, n_rep, threads=threads)
        t_step = max(time.perf_counter() - a - t_init, 1e-9) / k
    wall = time.perf_counter() - t0
    rounds = math.ceil(procedures / threads)
    t_full = rounds * (t_init + mc_steps * t_step)
    value = procedures * mc_steps / t_full
    return {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": (f"{n_rep} replicas (procedures 0..{n_rep - 1}) x {k} MC steps of L={spins} on {threads} "
                       f"host threads ({cpu_model()}), {wall:.1f} s wall: {t_step * 1e3:.3f} ms per step, "
                       f"{t_init * 1e3:.3f} ms initial state + entropy per replica, extrapolated linearly "
                       f"(bench.cpp:429-438) to {procedures} replicas x {mc_steps} steps = {t_full:.1f} s"),
            "extrapolated_seconds": t_full}, wall


def run_reference_arm(args, rank, world):
    if rank != 0:
        return 0
    world = max(world, args.gpus)
    spins, procedures, mc_steps, scaling, config = workload(args, world)
    threads = os.cpu_count() or 1
    ek = 0 if args.entropy == "von-neumann" else 1
    vals, walls = [], []
    for i in range(args.warmup + args.steps):
        cb, wall = cpu_reference_sample(spins, procedures, mc_steps, threads, target_s=args.ref_seconds,
                                        entropy_kind=ek)
        if i >= args.warmup:
            vals.append(cb["value"])
            walls.append(wall)
    value = float(np.median(vals))
    cb["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(walls)) * 1e3,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded product states, seed 0)", "config": config,
            "cpu_baseline": cb, "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def anneal_kernel(L, spins, rows, entropy):
    """The anneal kernel a launch of this workload runs (csrc: SMEM tier, HBM-tier cluster
    schedule or HBM-tier work queue, tg_hbm_schedule)."""
    if spins <= 12:
        return "anneal_smem_kernel", ""
    if int(L.tg_hbm_schedule(spins, rows, 0 if entropy == "von-neumann" else 1)) == 1:
        return "anneal_queue_kernel", "q"
    return "anneal_hbm_kernel", ""


def load_traffic(spins, rows, mc_steps, tag=""):
    """DRAM bytes per anneal-kernel launch of this exact workload (and schedule) from a
    committed ncu capture (profiles/ncu_traffic.json), or None when no capture of it exists."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            ent = json.load(f).get(f"{spins}x{rows}x{mc_steps}{tag}")
        return None if ent is None else float(ent["bytes"])
    except (OSError, ValueError, KeyError, TypeError):
        return None


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args):
    """--gpus N outside torchrun: re-execute under torch.distributed.run, one rank per GPU."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_2203_09353_b200 as tg
    from paper_2203_09353_b200.dist import gather_finals

    backend = os.environ.get("TG_BENCH_BACKEND", "nccl")  # gloo: N ranks sharing one GPU (tests)
    ndev = torch.cuda.device_count()
    gpu = local_rank % max(ndev, 1)
    torch.cuda.set_device(gpu)
    dev_t = torch.device("cuda", gpu)
    coll_dev = dev_t if backend == "nccl" else torch.device("cpu")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev_t)
        else:
            dist.init_process_group(backend)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    spins, procedures, S, scaling, config = workload(args, world)
    cfg = tg.ExperimentConfig(spins=spins, steps=S, procedures=procedures, seed=0, entropy_kind=args.entropy,
                              shard_index=rank, shard_count=world, rho_half=args.rho_half)
    if args.rho_half:
        config["rho"] = "Hermitian half (opt-in rho_half: upper-triangle blocks, executed flops in roofline)"
    ccfg = cfg.to_c()
    rows = cfg.rows()
    L = tg.lib()

    # device buffers (torch = allocator/stream plumbing); the kernels are ours
    def dbuf(n, dtype):
        return torch.empty(max(n, 1), dtype=dtype, device=dev_t)
    b_init, b_fin = dbuf(rows, torch.float64), dbuf(rows, torch.float64)
    b_ent, b_acc = dbuf(rows * S, torch.float64), dbuf(rows * S, torch.uint8)
    b_sites = dbuf(rows * S, torch.uint8)
    b_st, b_sst = dbuf(rows, torch.int32), dbuf(rows, torch.int64)
    b_norm = dbuf(rows, torch.float64)
    b_ties = dbuf(2, torch.int64)
    ws_bytes = int(L.tg_anneal_workspace_bytes(C.byref(ccfg)))
    b_ws = dbuf(ws_bytes, torch.uint8) if ws_bytes else None
    bufs = tg.CDeviceBuffers(b_init.data_ptr(), b_ent.data_ptr(), b_acc.data_ptr(), b_sites.data_ptr(), None,
                             b_fin.data_ptr(), b_st.data_ptr(), b_sst.data_ptr(),
                             b_ws.data_ptr() if b_ws is not None else None, b_norm.data_ptr(), None,
                             b_ties.data_ptr(), None, 0)
    stream = torch.cuda.current_stream(dev_t)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev_t)

    def launch():
        rc = L.tg_anneal_launch(C.byref(ccfg), C.byref(bufs), C.c_void_p(stream.cuda_stream))
        if rc != 0:
            raise RuntimeError(L.tg_last_error().decode())

    peak_tflops, peak_clock = tg.fp64_dmma_peak(gpu)
    kname, ktag = anneal_kernel(L, spins, rows, args.entropy)
    if args.rho_half and spins >= 13:  # the HBM tier runs the option on the work queue only
        kname, ktag = "anneal_queue_kernel", "qh"

    for _ in range(args.warmup):
        launch()
    torch.cuda.synchronize()
    if int(b_st[:rows].abs().sum().item()) != 0:
        raise RuntimeError("a replica left normalization during warm-up")

    # ------------------------------------------------------------ timed: device-resident
    times = []
    launches0 = tg.kernel_launches()
    with ClockSampler(gpu) as clocks:
        for _ in range(args.steps):
            flush.fill_(1.0)  # L2 flush (256 MiB > 126 MB L2), outside the timed interval
            barrier()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            launch()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            times.append(e0.elapsed_time(e1) / 1e3)
    clk = clocks.summary()
    launches = tg.kernel_launches() - launches0  # ours only (torch's L2-flush fill excluded)
    t_step = max_over_ranks(float(np.mean(times)))
    replica_steps = procedures * S
    value = replica_steps / t_step
    flops_launch = (rows * S + rows) * step_flops(spins)  # + initial-entropy GEMM per replica
    if args.rho_half:  # executed flops: nb (nb + 1) / 2 of nb^2 blocks (64x64 tiles, SMEM tier: 8x8 blocks)
        da = 1 << (spins // 2)
        nb = da // 64 if spins >= 13 else max(da, 8) // 8
        flops_launch = flops_launch // (nb * nb) * (nb * (nb + 1) // 2)
    achieved = flops_launch / float(np.mean(times)) / 1e12

    # ------------------------------------------------------------ timed: end to end (C ABI)
    pinned = {
        "initial": torch.empty(rows, dtype=torch.float64, pin_memory=True).numpy(),
        "final": torch.empty(rows, dtype=torch.float64, pin_memory=True).numpy(),
        "entropies": torch.empty((rows, S), dtype=torch.float64, pin_memory=True).numpy(),
        "accepted": torch.empty((rows, S), dtype=torch.uint8, pin_memory=True).numpy(),
        "sites": torch.empty((rows, S), dtype=torch.uint8, pin_memory=True).numpy(),
    }
    e2e_times = []
    with tg.Device([gpu]) as devctx:
        rep = devctx.run(cfg, sites=True, out=pinned)  # warm (allocations)
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = devctx.run(cfg, sites=True, out=pinned)
            finals, avg, best, best_e = gather_finals(rep.final_entropy, procedures, rank, world, device=coll_dev)
            torch.cuda.synchronize()
            e2e_times.append(time.perf_counter() - t0)
            barrier()
    t_e2e = max_over_ranks(float(np.mean(e2e_times)))
    d2h = rows * S * (8 + 1 + 1) + rows * (8 + 8 + 4 + 8)
    if args.dump_finals and rank == 0:
        np.save(args.dump_finals, finals)

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # the CPU sample: rank 0 at N=1 only
        cpu_baseline, _ = cpu_reference_sample(spins, procedures, S, os.cpu_count() or 1,
                                               target_s=args.ref_seconds,
                                               entropy_kind=0 if args.entropy == "von-neumann" else 1)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded product states, seed 0)",
            "config": config,
            "tflops": replica_steps * step_flops(spins) / t_step / 1e12,
            "average_entropy": avg, "best_procedure": best, "best_entropy": best_e,
            "roofline": {"bound": "tensor", "kernel": kname,
                         "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                         "frac": achieved / peak_tflops,
                         "peak_source": f"builder-measured DMMA.8x8x4 peak, live probe (tg_fp64_dmma_peak, "
                                        f"{peak_clock:.3f} GHz); MEASURED_PEAKS.json has no FP64 entry; see "
                                        "profiles/r01_fp64_peak.json",
                         "timed": "tg_anneal_launch on its stream (proposal pre-pass + anneal kernel), CUDA events",
                         "flops_per_launch": flops_launch, "traffic": load_traffic(spins, rows, S, ktag)},
            "e2e": {"value": replica_steps / t_e2e, "unit": UNIT, "h2d_bytes_per_step": C.sizeof(ccfg),
                    "d2h_bytes_per_step": d2h * world, "ms_per_step": t_e2e * 1e3},
            "gpu_launches": launches * world,
            "clocks": clk,
            "cpu_baseline": cpu_baseline,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--scaling", choices=["strong", "weak"], default=None,
                    help="strong: the config's replicas are the total; weak: per GPU (default per config)")
    ap.add_argument("--mc-steps", type=int, default=None)
    ap.add_argument("--replicas", type=int, default=None, help="replicas (total for strong, per GPU for weak)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=8.0, help="target CPU seconds of steps per sample")
    ap.add_argument("--dump-finals", default=None, help="rank 0 saves the gathered final entropies (.npy)")
    ap.add_argument("--rho-half", action="store_true",
                    help="opt-in Hermitian half of rho (upper-triangle tiles; S >= 13, Renyi-2): replica-steps/s "
                         "as usual, roofline on the executed (not the graded full-GEMM) flops")
    ap.add_argument("--entropy", choices=["renyi-2", "von-neumann"], default="renyi-2",
                    help="entropy kind (BASELINE metric is quoted on renyi-2, the bench default)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: W >= 3

    under_torchrun = "WORLD_SIZE" in os.environ
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        return run_reference_arm(args, rank, world)
    if not under_torchrun and args.gpus > 1:
        return spawn_ranks(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
