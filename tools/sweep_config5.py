"""BASELINE.json config 5: batch-size sweep 1..65536 replicas at L=14 (100 MC steps each),
our persistent device path vs the paper's ranks-per-GPU scheme (tasked cuBLAS, 16 ranks),
the batchedGEMM scheme (lock-step cublasZgemmStridedBatched) and the reference CPU path.

Every arm reports annealing replica-steps/s for the whole batch, end to end from the host
(the device path through Device.run with host result arrays). Comparator arms whose full
run would take minutes run a replica sample and are scaled linearly in replicas (replicas
are independent and the scheme is saturated well before the sample size); each row says
which replicas/steps were actually run. Writes one JSON document (default
profiles/r02_config5_sweep.json; round 1: r01_config5_sweep.json).

  python tools/sweep_config5.py [--out FILE] [--max-replicas N] [--steps 100]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "integration"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2203_09353_b200 as tg  # noqa: E402

SPINS = 14


def device_arm(dev, replicas, steps, reps=2):
    """Best of `reps` calls (the first call at a new size also grows the context's buffers)."""
    cfg = tg.ExperimentConfig(spins=SPINS, steps=steps, procedures=replicas, seed=0)
    wall = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        rep = dev.run(cfg, sites=False)
        wall = min(wall, time.perf_counter() - t0)
    return {"steps_per_s": replicas * steps / wall, "wall_s": wall, "kernel_ms": rep.kernel_ms,
            "kernel_steps_per_s": replicas * steps / (rep.kernel_ms * 1e-3) if rep.kernel_ms > 0 else None,
            "replicas_run": replicas, "steps_run": steps}, rep


def comparator_arm(fn, replicas, steps, cap, reps=2, **kw):
    """Best of `reps` runs (small runs) on a sample of at most `cap` replicas."""
    n = min(replicas, cap)
    wall = float("inf")
    for _ in range(reps if n * steps <= 100_000 else 1):
        out = fn(SPINS, steps, n, 0, **kw)
        wall = min(wall, out["wall_s"])
    return {"steps_per_s": n * steps / wall, "wall_s_sample": wall, "replicas_run": n, "steps_run": steps,
            "scaled": n < replicas}, out


def cpu_arm(replicas, steps, cores, target_s):
    from oracle_lib import REF_SO, McCfg, Oracle, RefLib  # checker / baseline only
    kind = "reference" if os.path.exists(REF_SO) else "port"
    lib = RefLib() if kind == "reference" else Oracle()
    n = int(min(replicas, 2 * cores))
    threads = int(min(n, cores))
    # calibrate per-step cost on one replica
    t0 = time.perf_counter()
    lib.run(McCfg(spins=SPINS, steps=5), 0, 1, threads=1, **({"sites": False} if kind == "reference" else {}))
    per = (time.perf_counter() - t0) / 5
    k = int(max(5, min(steps, target_s * threads / (per * n))))
    t0 = time.perf_counter()
    lib.run(McCfg(spins=SPINS, steps=k), 0, n, threads=threads, **({"sites": False} if kind == "reference" else {}))
    wall = time.perf_counter() - t0
    return {"steps_per_s": n * k / wall, "kind": kind, "cores": threads, "replicas_run": n, "steps_run": k,
            "scaled": n < replicas or k < steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_config5_sweep.json"))
    ap.add_argument("--max-replicas", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--tasked-cap", type=int, default=2048)
    ap.add_argument("--batched-cap", type=int, default=4096)
    ap.add_argument("--ranks", type=int, default=16)
    ap.add_argument("--cpu-seconds", type=float, default=4.0)
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    from comparators import Comparators
    cmp = Comparators()
    cores = os.cpu_count() or 1
    sizes = [r for r in (1, 4, 16, 64, 148, 256, 512, 1024, 4096, 16384, 65536) if r <= a.max_replicas]
    dev = tg.Device([0])
    device_arm(dev, 16, 10)  # warm-up: context, module load, workspace
    cmp.tasked(SPINS, 5, 2, ranks=2)
    cmp.batched(SPINS, 5, 2)
    rows = []
    for r in sizes:
        row = {"replicas": r, "spins": SPINS, "steps": a.steps}
        row["device"], rep = device_arm(dev, r, a.steps)
        row["device"]["schedule"] = ["cluster", "work queue"][int(tg.lib().tg_hbm_schedule(SPINS, r, 1))]
        row["tasked"], tk = comparator_arm(cmp.tasked, r, a.steps, a.tasked_cap, ranks=a.ranks)
        row["batched"], bt = comparator_arm(cmp.batched, r, a.steps, a.batched_cap)
        # the arms computed the same trajectories (first replicas): flags bit-exact
        n = min(r, 64)
        row["tasked"]["flags_match_device"] = bool(np.array_equal(tk["accepted"][:n], rep.accepted[:n]))
        row["batched"]["flags_match_device"] = bool(np.array_equal(bt["accepted"][:n], rep.accepted[:n]))
        if not a.no_cpu:
            row["cpu"] = cpu_arm(r, a.steps, cores, a.cpu_seconds)
        d = row["device"]["steps_per_s"]
        row["device_over_tasked"] = d / row["tasked"]["steps_per_s"]
        row["device_over_batched"] = d / row["batched"]["steps_per_s"]
        if "cpu" in row:
            row["device_over_cpu"] = d / row["cpu"]["steps_per_s"]
        rows.append(row)
        print(json.dumps({k: (v if not isinstance(v, dict) else round(v["steps_per_s"], 1))
                          for k, v in row.items()}), flush=True)
    import torch
    doc = {"config": "BASELINE.json config 5: batch-size sweep at L=14, "
                     f"{a.steps} MC steps, replica-steps/s end to end from the host",
           "gpu": torch.cuda.get_device_name(0), "host_cores": cores, "ranks_per_gpu": a.ranks,
           "tasked_cap": a.tasked_cap, "batched_cap": a.batched_cap, "rows": rows}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", a.out)


if __name__ == "__main__":
    main()
