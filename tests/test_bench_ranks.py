"""bench.py's multi-GPU rank logic: `--gpus N` re-executes itself under
torch.distributed.run, rank r anneals procedures p = r (mod N) (bench.cpp:171) through the
same C ABI, and the one end-of-run all-gather reassembles the finals in procedure order.
On the one-GPU test box both ranks share GPU 0 over gloo (TG_BENCH_BACKEND=gloo; NCCL refuses
two ranks on one device); the gathered finals must equal the one-rank run bit for bit."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(tmp_path, gpus, tag, extra=(), config=2, replicas=37, mc_steps=40):
    out = tmp_path / f"finals_{tag}.npy"
    env = dict(os.environ, TG_BENCH_BACKEND="gloo")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--config", str(config), "--scaling",
           "strong", "--replicas", str(replicas), "--mc-steps", str(mc_steps), "--steps", "1", "--warmup", "3",
           "--no-cpu-baseline", "--dump-finals", str(out), *extra]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints the JSON line
    return json.loads(lines[0]), np.load(out)


@pytest.mark.gpu
def test_bench_two_ranks_bitwise_single(tmp_path):
    one, f1 = _bench(tmp_path, 1, "one")
    two, f2 = _bench(tmp_path, 2, "two")
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2
    assert one["config"]["procedures"] == two["config"]["procedures"] == 37
    assert two["config"]["parallelism"].startswith("dp2")
    assert np.array_equal(f1.view(np.uint64), f2.view(np.uint64))
    assert one["average_entropy"] == two["average_entropy"]
    assert one["best_procedure"] == two["best_procedure"]


def test_bench_configs_identical_between_arms():
    """Both arms report the same `config` dict for the same flags (the driver compares them)."""
    sys.path.insert(0, ROOT)
    import argparse

    import bench
    for cfg in (1, 2, 3, 4, 5):
        for world in (1, 2, 8):
            a = argparse.Namespace(config=cfg, mc_steps=None, replicas=None, scaling=None, entropy="renyi-2")
            s1 = bench.workload(a, world)
            s2 = bench.workload(a, world)
            assert s1 == s2
            spins, procs, steps, scaling, conf = s1
            if cfg in (3, 4):
                assert scaling == "strong" and procs == bench.CONFIGS[cfg]["replicas"]
            else:
                assert scaling == "weak" and procs == bench.CONFIGS[cfg]["replicas"] * world
    a = argparse.Namespace(config=4, mc_steps=None, replicas=None, scaling=None, entropy="renyi-2")
    assert bench.workload(a, 1)[4]["workload"].startswith("config4: L=20")


def test_bench_cpu_sample_extrapolation(reflib):
    """The CPU leg: per-replica total and per-step wall times from the reference's own
    mc_procedure, extrapolated linearly in steps (bench.cpp:429-438)."""
    sys.path.insert(0, ROOT)
    import bench
    cb, wall = bench.cpu_reference_sample(8, 64, 1000, 2, target_s=0.05)
    assert cb["kind"] == "reference" and cb["cores"] == 2 and cb["value"] > 0
    assert "extrapolated linearly" in cb["sample"]
    assert wall < 30


@pytest.mark.gpu
def test_bench_two_ranks_config4_queue(tmp_path):
    """Config 4's chain (L = 20) split over 2 ranks: each rank runs its replicas p = r (mod 2)
    on the HBM tier's work queue (the schedule config 4 uses at every rank count); the
    gathered finals equal the one-rank run's bit for bit."""
    one, f1 = _bench(tmp_path, 1, "one4", config=4, replicas=6, mc_steps=2)
    two, f2 = _bench(tmp_path, 2, "two4", config=4, replicas=6, mc_steps=2)
    assert one["roofline"]["kernel"] == two["roofline"]["kernel"] == "anneal_queue_kernel"
    assert np.array_equal(f1.view(np.uint64), f2.view(np.uint64))
    assert one["average_entropy"] == two["average_entropy"]
