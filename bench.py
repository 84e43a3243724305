"""Benchmark: annealing replica-steps/s of the B200 hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2|1|3|4|5] [--mc-steps M] [--replicas R]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU)

One bench "step" = one full persistent-kernel anneal of the workload: every replica of
this GPU runs all MC steps (gate -> rho = Psi Psi^dagger on DMMA -> Renyi-2 -> Metropolis),
inputs = (seed, config) only, all state resident on the device. Default workload =
BASELINE.json configs[1]: L=12, 1024 replicas per GPU, 10,000 MC steps. Multi-GPU is weak
scaling: rank r runs replicas p = r + N*q (p mod N binding, bench.cpp:171), no data-path
collective; the final entropies are all-gathered once (NCCL) for the procedure-order
average / best replica.

`value`  : replica-steps/s over all ranks, device time (CUDA events on the launch stream,
           max over ranks), L2 flushed (256 MiB write) between timed iterations.
`e2e`    : same metric through the public C-ABI call tg_anneal_run with host buffers
           (kernel-argument H2D + trace D2H into pinned memory) + the NCCL gather, wall time.
`roofline`: FP64 DMMA roofline of the anneal kernel; peak = live DMMA.8x8x4 probe
           (MEASURED_PEAKS.json has no FP64 entry), committed in profiles/.
`cpu_baseline`: the reference's own CPU code (oracle/_ref, pooled host threads) on a
           bounded sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "annealing steps/sec (all replicas, whole box) and FP64 TFLOP/s vs DMMA roofline"
UNIT = "replica-steps/s"

CONFIGS = {  # BASELINE.json configs (per GPU for the weak-scaling multi-GPU runs)
    1: dict(spins=8, replicas=64, mc_steps=1000, name="config1: L=8, 64 replicas, 1000 MC steps"),
    2: dict(spins=12, replicas=1024, mc_steps=10000, name="config2: L=12, 1024 replicas/GPU, 10000 MC steps"),
    # configs 3/4: BASELINE.json leaves the step count open; SURVEY.md §8(d) fixes 1000 / 100
    3: dict(spins=16, replicas=4096, mc_steps=1000, name="config3: L=16 (256x256 GEMMs), 4096 replicas/GPU, 1000 MC steps"),
    4: dict(spins=20, replicas=512, mc_steps=100, name="config4: L=20 (1024x1024 GEMMs), 512 replicas/GPU, 100 MC steps"),
    5: dict(spins=14, replicas=65536, mc_steps=100, name="config5: L=14, 65536 replicas/GPU, 100 MC steps"),
}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


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
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_reference_sample(cfg_spins, replicas, mc_steps, threads, target_s=15.0, entropy_kind=1):
    """Time the reference's own CPU path (oracle/_ref: spinmc::mc_procedure + DirectExecutor,
    pooled host threads) on a bounded sample; falls back to the oracle port if _ref is absent."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import REF_SO, McCfg, Oracle, RefLib  # checker / baseline only

    kind = "reference" if os.path.exists(REF_SO) else "port"
    lib = RefLib() if kind == "reference" else Oracle()
    # calibrate: one replica, few steps
    cal_steps = 20
    t0 = time.perf_counter()
    if kind == "reference":
        lib.run(McCfg(spins=cfg_spins, steps=cal_steps, entropy_kind=entropy_kind), 0, 1, threads=1, sites=False)
    else:
        lib.run(McCfg(spins=cfg_spins, steps=cal_steps, entropy_kind=entropy_kind), 0, 1, threads=1)
    per_step = max((time.perf_counter() - t0) / cal_steps, 1e-7)
    # sample: `threads*2` replicas (or fewer), steps chosen for ~target_s of wall time
    n_rep = int(min(replicas, max(threads * 2, 1)))
    steps = int(max(5, min(mc_steps, target_s * threads / (per_step * n_rep))))
    cfg = McCfg(spins=cfg_spins, steps=steps, entropy_kind=entropy_kind)
    t0 = time.perf_counter()
    if kind == "reference":
        lib.run(cfg, 0, n_rep, threads=threads, sites=False)
    else:
        lib.run(cfg, 0, n_rep, threads=threads)
    wall = time.perf_counter() - t0
    value = n_rep * steps / wall
    return {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{n_rep} replicas x {steps} MC steps of L={cfg_spins} (first steps of the "
                      f"workload's replicas 0..{n_rep - 1}), {wall:.2f} s wall, {threads} host threads"}, wall


def run_reference_arm(args, cfgw, rank, world):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        cb, wall = cpu_reference_sample(cfgw["spins"], cfgw["replicas"], cfgw["mc_steps"], threads,
                                        target_s=args.ref_seconds,
                                        entropy_kind=0 if args.entropy == "von-neumann" else 1)
        if i >= args.warmup:
            vals.append(cb["value"])
    value = float(np.median(vals))
    cb["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded product states)",
            "config": {"workload": cfgw["name"], "spins": cfgw["spins"], "replicas_per_gpu": cfgw["replicas"],
                       "mc_steps": cfgw["mc_steps"], "note": "each step = bounded CPU sample of the workload"},
            "cpu_baseline": cb, "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def load_traffic(spins, rows, mc_steps):
    """DRAM bytes per anneal-kernel launch of this exact workload from a committed ncu --set
    full capture (profiles/ncu_traffic.json), or None when no capture of it exists."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            ent = json.load(f).get(f"{spins}x{rows}x{mc_steps}")
        return None if ent is None else float(ent["bytes"])
    except (OSError, ValueError, KeyError, TypeError):
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--mc-steps", type=int, default=None)
    ap.add_argument("--replicas", type=int, default=None, help="replicas per GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-seconds", type=float, default=15.0)
    ap.add_argument("--entropy", choices=["renyi-2", "von-neumann"], default="renyi-2",
                    help="entropy kind (BASELINE metric is quoted on renyi-2, the bench default)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: W >= 3

    cfgw = dict(CONFIGS[args.config])
    if args.mc_steps:
        cfgw["mc_steps"] = args.mc_steps
    if args.replicas:
        cfgw["replicas"] = args.replicas

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local_rank = env_int("LOCAL_RANK", 0)

    if args.impl == "reference":
        return run_reference_arm(args, cfgw, rank, world)

    import torch
    import torch.distributed as dist

    import paper_2203_09353_b200 as tg
    from paper_2203_09353_b200.dist import gather_finals

    torch.cuda.set_device(local_rank)
    dev_t = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev_t)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev_t)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    spins, R, S = cfgw["spins"], cfgw["replicas"], cfgw["mc_steps"]
    procedures = R * world
    cfg = tg.ExperimentConfig(spins=spins, steps=S, procedures=procedures, seed=0, entropy_kind=args.entropy,
                              shard_index=rank, shard_count=world)
    ccfg = cfg.to_c()
    rows = cfg.rows()
    L = tg.lib()

    # device buffers (torch = allocator/stream plumbing); the kernel is ours
    def dbuf(n, dtype):
        return torch.empty(max(n, 1), dtype=dtype, device=dev_t)
    b_init, b_fin = dbuf(rows, torch.float64), dbuf(rows, torch.float64)
    b_ent, b_acc = dbuf(rows * S, torch.float64), dbuf(rows * S, torch.uint8)
    b_sites = dbuf(rows * S, torch.uint8)
    b_st, b_sst = dbuf(rows, torch.int32), dbuf(rows, torch.int64)
    ws_bytes = int(L.tg_anneal_workspace_bytes(C.byref(ccfg)))
    b_ws = dbuf(ws_bytes, torch.uint8) if ws_bytes else None
    bufs = tg.CDeviceBuffers(b_init.data_ptr(), b_ent.data_ptr(), b_acc.data_ptr(), b_sites.data_ptr(), None,
                             b_fin.data_ptr(), b_st.data_ptr(), b_sst.data_ptr(),
                             b_ws.data_ptr() if b_ws is not None else None)
    stream = torch.cuda.current_stream(dev_t)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev_t)

    def launch():
        rc = L.tg_anneal_launch(C.byref(ccfg), C.byref(bufs), C.c_void_p(stream.cuda_stream))
        if rc != 0:
            raise RuntimeError(L.tg_last_error().decode())

    peak_tflops, peak_clock = tg.fp64_dmma_peak(local_rank)

    for _ in range(args.warmup):
        launch()
    torch.cuda.synchronize()
    if int(b_st[:rows].abs().sum().item()) != 0:
        raise RuntimeError("a replica left normalization during warm-up")

    # ------------------------------------------------------------ timed: device-resident
    times = []
    launches0 = tg.kernel_launches()
    with ClockSampler(local_rank) as clocks:
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
    flops_launch = (rows * S + rows) * tg.step_flops(spins)  # + initial-entropy GEMM per replica
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
    with tg.Device([local_rank]) as devctx:
        rep = devctx.run(cfg, sites=True, out=pinned)  # warm (allocations)
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = devctx.run(cfg, sites=True, out=pinned)
            finals, avg, best, best_e = gather_finals(rep.final_entropy, procedures, rank, world, device=dev_t)
            torch.cuda.synchronize()
            e2e_times.append(time.perf_counter() - t0)
            barrier()
    t_e2e = max_over_ranks(float(np.mean(e2e_times)))
    d2h = rows * S * (8 + 1 + 1) + rows * (8 + 8 + 4 + 8)

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # the CPU sample: rank 0 at N=1 only
        cpu_baseline, _ = cpu_reference_sample(spins, R, S, os.cpu_count() or 1,
                                               entropy_kind=0 if args.entropy == "von-neumann" else 1)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded product states, seed 0)",
            "config": {"workload": cfgw["name"], "spins": spins, "gemm_mnk": [tg.dims_for_spins(spins)[0]] * 2 + [tg.dims_for_spins(spins)[1]], "replicas_per_gpu": R, "procedures": procedures,
                       "mc_steps": S, "parallelism": f"dp{world} (replica p on GPU p mod {world})",
                       "entropy": args.entropy, "l2": "flushed between timed iterations (256 MiB write)"},
            "tflops": replica_steps * tg.step_flops(spins) / t_step / 1e12,
            "average_entropy": avg, "best_procedure": best, "best_entropy": best_e,
            "roofline": {"bound": "tensor", "kernel": "anneal_smem_kernel" if spins <= 12 else "anneal_hbm_kernel",
                         "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                         "frac": achieved / peak_tflops,
                         "peak_source": f"live DMMA.8x8x4 probe (tg_fp64_dmma_peak, {peak_clock:.3f} GHz); "
                                        "MEASURED_PEAKS.json has no FP64 entry; see profiles/r01_fp64_peak.json",
                         "timed": "tg_anneal_launch on its stream (proposal pre-pass ~2% + anneal kernel), CUDA events", "flops_per_launch": flops_launch, "traffic": load_traffic(spins, rows, S)},
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


if __name__ == "__main__":
    sys.exit(main())
