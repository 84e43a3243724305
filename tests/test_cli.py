"""`taskgemm_b200` CLI, mirroring the reference's CLI tests (proj/tests/test_cli.cpp:66-196):
output bundle and keys, byte-identical reruns (wall column stripped), exit codes, seed
precedence, baseline speedup, sweep, kernel log, verify with fault injection."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2203_09353_b200", "taskgemm_b200")


def run(args, env=None, cwd=None):
    e = dict(os.environ)
    e.pop("TASKGEMM_SEED", None)
    if env:
        e.update(env)
    p = subprocess.run([CLI] + args, capture_output=True, text=True, env=e, cwd=cwd)
    return p.returncode, p.stdout + p.stderr


def without_wall(csv):
    return "\n".join(line.rsplit(",", 1)[0] for line in csv.splitlines())


# ------------------------------------------------------------------ CPU: configuration
@pytest.mark.parametrize("args,msg", [
    (["run", "--spins", "40", "--steps", "1"], "spins out of range [2,30]"),
    (["run", "--warp-factor", "9"], "unknown option"),
    (["run", "--mode", "tasked"], "use --mode device"),
    (["run", "--entropy", "bogus"], "unknown value for --entropy"),
    (["run", "--t0", "1e-4", "--t-min", "1"], "anneal schedule requires 0 < t_min <= t0"),
    (["bogus"], "unknown subcommand"),
])
def test_config_errors_exit_2(tmp_path, args, msg):
    code, out = run(args + ["--out", str(tmp_path)] if args[0] == "run" else args)
    assert code == 2, out
    assert msg in out


def test_bad_seed_env_exit_2(tmp_path):
    code, out = run(["run", "--spins", "4", "--out", str(tmp_path)], env={"TASKGEMM_SEED": "x1"})
    assert code == 2 and "TASKGEMM_SEED" in out


# --------------------------------------------------------------------------- GPU: runs
gpu = pytest.mark.gpu


@gpu
def test_run_writes_bundle(tmp_path):
    code, out = run(["run", "--spins", "6", "--steps", "100", "--procedures", "2", "--seed", "7",
                     "--out", str(tmp_path)])
    assert code == 0, out
    csv = (tmp_path / "trace.csv").read_text()
    assert csv.startswith("procedure,step,entropy_nats,accepted,wall_ns\n")
    assert len(csv.splitlines()) == 1 + 200
    rep = json.loads((tmp_path / "report.json").read_text())
    for k in ("config", "total_wall_ns", "average_entropy_nats", "per_device", "speedup_vs"):
        assert k in rep
    assert rep["speedup_vs"] is None
    assert rep["config"]["spins"] == 6 and rep["config"]["seed"] == 7 and rep["config"]["mode"] == "device"
    assert rep["per_device"][0]["kernel_count"] == 2 * 101


@gpu
def test_rerun_byte_identical(tmp_path):
    a, b = tmp_path / "a", tmp_path / "b"
    args = ["run", "--spins", "6", "--steps", "80", "--procedures", "2", "--seed", "7", "--out"]
    assert run(args + [str(a)])[0] == 0
    assert run(args + [str(b)])[0] == 0
    ta, tb = without_wall((a / "trace.csv").read_text()), without_wall((b / "trace.csv").read_text())
    assert ta == tb and ta


@gpu
def test_trace_matches_reference_golden(tmp_path):
    """config 1 through the CLI == the reference's trajectories within tolerance."""
    import numpy as np
    g = np.load(os.path.join(ROOT, "tests", "golden", "traj_cfg1.npz"))
    code, out = run(["run", "--spins", "8", "--steps", "1000", "--procedures", "64", "--seed", "0",
                     "--out", str(tmp_path)])
    assert code == 0, out
    rows = [line.split(",") for line in (tmp_path / "trace.csv").read_text().splitlines()[1:]]
    ent = np.array([float(r[2]) for r in rows]).reshape(64, 1000)
    acc = np.array([int(r[3]) for r in rows], np.uint8).reshape(64, 1000)
    assert np.array_equal(acc, g["accepted"])
    assert (np.abs(ent - g["entropies"]) <= 1e-10 * np.maximum(np.abs(g["entropies"]), 1)).all()
    rep = json.loads((tmp_path / "report.json").read_text())
    assert abs(rep["average_entropy_nats"] - 2.2063680065173292) <= 1e-10 * 2.21


@gpu
def test_run_von_neumann_config1(tmp_path):
    """--entropy von-neumann (the McConfig default kind) on config 1 vs the reference's golden
    trajectory (second line)."""
    import numpy as np
    g = np.load(os.path.join(ROOT, "tests", "golden", "traj_vn_cfg1.npz"))
    code, out = run(["run", "--spins", "8", "--steps", "1000", "--procedures", "64", "--seed", "0",
                     "--entropy", "von-neumann", "--out", str(tmp_path)])
    assert code == 0, out
    rows = [line.split(",") for line in (tmp_path / "trace.csv").read_text().splitlines()[1:]]
    acc = np.array([int(r[3]) for r in rows], np.uint8).reshape(64, 1000)
    assert np.array_equal(acc, g["accepted"])
    rep = json.loads((tmp_path / "report.json").read_text())
    assert rep["config"]["entropy"] == "von-neumann"
    assert abs(rep["average_entropy_nats"] - 2.360208109374111) <= 1e-10 * 2.37
    code, out = run(["run", "--spins", "22", "--steps", "1", "--entropy", "von-neumann", "--out", str(tmp_path / "x")])
    assert code != 0 and "device von-neumann entropy covers spins <= 21" in out


@gpu
def test_seed_env_and_flag_precedence(tmp_path):
    env_dir, flag_dir = tmp_path / "env", tmp_path / "flag"
    base = ["run", "--spins", "6", "--steps", "60", "--procedures", "1", "--out"]
    assert run(base + [str(env_dir)], env={"TASKGEMM_SEED": "1234"})[0] == 0
    assert run(base + [str(flag_dir), "--seed", "1234"], env={"TASKGEMM_SEED": "999"})[0] == 0
    assert without_wall((env_dir / "trace.csv").read_text()) == without_wall((flag_dir / "trace.csv").read_text())
    assert json.loads((env_dir / "report.json").read_text())["config"]["seed"] == 1234


@gpu
def test_baseline_speedup(tmp_path):
    a, b, bad = tmp_path / "a", tmp_path / "b", tmp_path / "bad"
    work = ["--spins", "6", "--steps", "60", "--procedures", "4", "--seed", "5"]
    assert run(["run"] + work + ["--out", str(a)])[0] == 0
    assert run(["run"] + work + ["--baseline", str(a / "report.json"), "--out", str(b)])[0] == 0
    rep = json.loads((b / "report.json").read_text())
    assert rep["speedup_vs"]["value"] > 0
    code, _ = run(["run", "--spins", "6", "--steps", "61", "--procedures", "4", "--seed", "5",
                   "--baseline", str(a / "report.json"), "--out", str(bad)])
    assert code == 1  # mismatched workload (bench.cpp:440-455)


@gpu
def test_sweep(tmp_path):
    code, out = run(["run", "--spins", "6", "--steps", "30", "--seed", "3", "--sweep-procedures", "1,2",
                     "--repeats", "1", "--out", str(tmp_path)])
    assert code == 0, out
    rep = json.loads((tmp_path / "report.json").read_text())
    assert [c["procedures"] for c in rep["sweep"]] == [1, 2]
    assert rep["sweep"][0]["mode"] == "device"
    assert "\n1,0," in (tmp_path / "trace.csv").read_text()


@gpu
def test_kernel_log(tmp_path):
    code, out = run(["run", "--spins", "6", "--steps", "20", "--procedures", "2", "--seed", "7",
                     "--kernel-log", "--out", str(tmp_path)])
    assert code == 0, out
    csv = (tmp_path / "kernels.csv").read_text()
    assert csv.startswith("device,procedure,m,n,k,queue_wait_ns,exec_ns,flops\n")
    assert "\n0,0,8,8,8," in csv


@gpu
def test_verify_clean_and_fault():
    code, out = run(["verify", "--seed", "11"])
    assert code == 0, out
    for s in ("PASS gemm", "PASS entropy", "PASS cross-executor"):
        assert s in out
    code, out = run(["verify", "--suite", "gemm", "--seed", "11"])
    assert code == 0 and "entropy" not in out
    code, out = run(["verify", "--inject-fault", "--seed", "11"])
    assert code == 1 and "FAIL" in out
