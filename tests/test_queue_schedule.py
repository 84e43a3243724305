"""GPU: the HBM tier's work-queue schedule (csrc/hbm_queue.cuh) — every CTA pulls INIT / TILE /
DEC / GATE items from one queue instead of owning whole replicas. Its traces must be bitwise
those of the cluster schedule (the tiles' per-thread partials are folded in the canonical
order whichever CTA computed them) and match the oracle (sites and accept flags bit-exact,
entropies within 1e-10)."""
import numpy as np
import pytest
from oracle_lib import McCfg

import paper_2203_09353_b200 as tg

pytestmark = pytest.mark.gpu
TOL = 1e-10


def close(got, want, tol=TOL):
    got, want = np.asarray(got), np.asarray(want)
    return np.abs(got - want) <= tol * np.maximum(np.abs(want), 1.0)


def run_with(device, cfg, monkeypatch, **env):
    for k in ("TG_HBM_QUEUE", "TG_HBM_CTAS_PER_REPLICA"):
        monkeypatch.delenv(k, raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    return device.run(cfg, wall=True)


def assert_bitwise(a, b):
    assert np.array_equal(a.initial_entropy.view(np.uint64), b.initial_entropy.view(np.uint64))
    assert np.array_equal(a.entropies.view(np.uint64), b.entropies.view(np.uint64))
    assert np.array_equal(a.final_entropy.view(np.uint64), b.final_entropy.view(np.uint64))
    assert np.array_equal(a.accepted, b.accepted)
    assert np.array_equal(a.sites, b.sites)
    assert a.average_entropy == b.average_entropy


CASES = [  # spins, procedures, steps, initial state, objective, renormalize_interval
    (13, 4, 12, "random", "max", 1000),   # d_a = 64: one tile per replica
    (14, 5, 20, "product", "max", 7),     # renormalisation inside DEC items
    (14, 1, 30, "random", "min", 9),      # one replica: lag 0, strictly sequential queue
    (15, 2, 10, "product", "min", 4),
    (16, 3, 6, "random", "max", 1000),    # 16 tiles, 4 gate parts per replica
    (14, 37, 8, "product", "max", 1000),  # more replicas than tiles in flight
    (18, 2, 3, "random", "max", 2),       # 16 gate parts, 64 tiles
    (14, 200, 6, "product", "max", 4),    # 800 tiles per step, renormalisations inside DEC items
    (16, 40, 4, "random", "min", 1000),
    (20, 1, 2, "product", "max", 1000),   # one replica of config 4's chain: lag 0 over 256 tiles
]


@pytest.mark.parametrize("spins,procs,steps,init,obj,renorm", CASES)
def test_queue_vs_cluster_bitwise(device, oracle, monkeypatch, spins, procs, steps, init, obj, renorm):
    cfg = tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=31, initial_state=init,
                              objective=obj, renormalize_interval=renorm)
    a = run_with(device, cfg, monkeypatch, TG_HBM_QUEUE="0", TG_HBM_CTAS_PER_REPLICA="1")
    b = run_with(device, cfg, monkeypatch, TG_HBM_QUEUE="1")
    assert_bitwise(a, b)
    assert np.all(b.wall_ns > 0)
    if spins <= 16:
        want = oracle.run(McCfg(spins=spins, steps=steps, seed=31, initial_state=1 if init == "random" else 0,
                                objective=1 if obj == "min" else 0, renormalize_interval=renorm), 0, procs)
        assert np.array_equal(b.sites, want.sites)
        assert np.array_equal(b.accepted, want.accepted)
        assert close(b.entropies, want.entropies).all()
        assert close(b.initial_entropy, want.initial).all()


def test_queue_rerun_bitwise_and_zero_steps(device, monkeypatch):
    cfg = tg.ExperimentConfig(spins=14, steps=15, procedures=9, seed=2)
    a = run_with(device, cfg, monkeypatch, TG_HBM_QUEUE="1")
    b = run_with(device, cfg, monkeypatch, TG_HBM_QUEUE="1")
    assert_bitwise(a, b)
    z = tg.ExperimentConfig(spins=14, steps=0, procedures=3, seed=2)
    c = run_with(device, z, monkeypatch, TG_HBM_QUEUE="1")
    d = run_with(device, z, monkeypatch, TG_HBM_QUEUE="0", TG_HBM_CTAS_PER_REPLICA="1")
    assert c.entropies.shape == (3, 0)
    assert np.array_equal(c.initial_entropy.view(np.uint64), d.initial_entropy.view(np.uint64))
    assert c.average_entropy == d.average_entropy


def test_queue_fault_injection_bitwise(device, monkeypatch):
    """inject_fault = 1 (perturb_gemm on tile 0 of every GEMM): the queue applies the same
    perturbation with the same rounding as the cluster schedule."""
    cfg = tg.ExperimentConfig(spins=14, steps=6, procedures=3, seed=5, inject_fault=1)
    a = run_with(device, cfg, monkeypatch, TG_HBM_QUEUE="0", TG_HBM_CTAS_PER_REPLICA="2")
    b = run_with(device, cfg, monkeypatch, TG_HBM_QUEUE="1")
    assert_bitwise(a, b)


def test_queue_not_normalized_error(device, monkeypatch):
    """A non-unitary gate (inject_fault = 2) on one replica: the queue schedule reports the
    reference's std::invalid_argument message, like the cluster schedule."""
    cfg = tg.ExperimentConfig(spins=14, steps=8, procedures=4, seed=5, inject_fault=2, fault_procedure=2,
                              fault_step=3)
    msgs = []
    for env in ({"TG_HBM_QUEUE": "0", "TG_HBM_CTAS_PER_REPLICA": "1"}, {"TG_HBM_QUEUE": "1"}):
        with pytest.raises(ValueError, match="entanglement_entropy: state not normalized") as ei:
            run_with(device, cfg, monkeypatch, **env)
        msgs.append(str(ei.value))
    assert msgs[0] == msgs[1]


def test_queue_two_contexts_share_gpu(oracle, monkeypatch):
    """Two host threads (devices [0, 0]) each launch a queue kernel on GPU 0 at the same time:
    neither grid is fully resident, which the dependency-ordered queue tolerates (no grid
    barrier); traces are bitwise the one-device run's."""
    monkeypatch.setenv("TG_HBM_QUEUE", "1")
    cfg1 = tg.ExperimentConfig(spins=14, steps=12, procedures=6, seed=21, devices=1)
    cfg2 = tg.ExperimentConfig(spins=14, steps=12, procedures=6, seed=21, devices=2)
    with tg.Device([0]) as d1:
        a = d1.run(cfg1)
    with tg.Device([0, 0]) as d2:
        b = d2.run(cfg2)
    assert_bitwise(a, b)
    want = oracle.run(McCfg(spins=14, steps=12, seed=21), 0, 6)
    assert np.array_equal(b.accepted, want.accepted)


@pytest.mark.slow
def test_queue_config4_shape(device, oracle, monkeypatch):
    """L = 20 (256 tiles of 64x64 per replica, 16 gate parts): queue vs 1-CTA cluster
    bitwise on 3 replicas x 2 steps; replica 0 against the oracle."""
    cfg = tg.ExperimentConfig(spins=20, steps=2, procedures=3, seed=4)
    a = run_with(device, cfg, monkeypatch, TG_HBM_QUEUE="0", TG_HBM_CTAS_PER_REPLICA="1")
    b = run_with(device, cfg, monkeypatch, TG_HBM_QUEUE="1")
    assert_bitwise(a, b)
    _, ent, acc, sites, _, _ = oracle.mc_procedure(McCfg(spins=20, steps=2, seed=4), 0)
    assert np.array_equal(b.accepted[0], acc) and np.array_equal(b.sites[0], sites)
    assert close(b.entropies[0], ent).all()


def test_queue_schedule_choice():
    """The model picks the queue where the cluster schedule idles SMs (64 replicas of L = 20:
    128 of 148 SMs) and keeps the cluster schedule for large batches."""
    L = tg.lib()
    if not hasattr(L, "tg_hbm_schedule"):
        pytest.skip("no schedule probe")
    assert L.tg_hbm_schedule(20, 64, 1) == 1
    assert L.tg_hbm_schedule(14, 65536, 1) == 0
    assert L.tg_hbm_schedule(14, 64, 0) == 0  # von Neumann: cluster schedule only


# ----------------------------------------------- opt-in Hermitian half of rho (rho_half)
@pytest.mark.parametrize("spins,procs,steps,init", [(13, 3, 10, "random"), (14, 5, 12, "product"),
                                                     (16, 3, 6, "random"), (18, 2, 3, "product"),
                                                     (4, 5, 40, "random"), (8, 6, 120, "product"),
                                                     (10, 4, 90, "random"), (11, 3, 70, "product"),
                                                     (12, 5, 150, "product"), (12, 3, 1010, "random")])
def test_rho_half_vs_oracle(device, oracle, spins, procs, steps, init):
    """rho_half forms only the upper-triangle 64x64 tiles (HBM tier) or 8x8 blocks (SMEM tier,
    incl. S = 12's speculative gate and the renormalisation at step 1000) of rho: diagonal
    ones once, off-diagonal ones twice in ||rho||_F^2. Sites and accept flags still bit-exact
    against the oracle, entropies within the 1e-10 parity tolerance, reruns bitwise, executed
    flops reported apart from the graded full-GEMM count."""
    cfg = tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=12, initial_state=init)
    full = device.run(cfg)
    cfg.rho_half = True
    half = device.run(cfg)
    again = device.run(cfg)
    assert_bitwise(half, again)
    assert np.array_equal(half.sites, full.sites) and np.array_equal(half.accepted, full.accepted)
    assert close(half.entropies, full.entropies, 1e-12).all()
    da = 1 << (spins // 2)
    nt = da // 64 if spins >= 13 else max(da, 8) // 8  # 64x64 tiles (HBM tier) or 8x8 blocks (SMEM tier)
    assert half.total_flops == full.total_flops == full.executed_flops
    assert half.executed_flops == full.total_flops // (nt * nt) * (nt * (nt + 1) // 2)
    if spins <= 16:
        want = oracle.run(McCfg(spins=spins, steps=steps, seed=12, initial_state=1 if init == "random" else 0), 0, procs)
        assert np.array_equal(half.sites, want.sites)
        assert np.array_equal(half.accepted, want.accepted)
        assert close(half.entropies, want.entropies).all()
        assert close(half.initial_entropy, want.initial).all()


def test_rho_half_renormalisation_and_errors(device, monkeypatch):
    """rho_half across renormalisations and with the cluster schedule forced off-limits (the
    option always runs on the work queue); the not-normalised error keeps the reference message."""
    monkeypatch.setenv("TG_HBM_QUEUE", "0")
    cfg = tg.ExperimentConfig(spins=14, steps=20, procedures=4, seed=3, renormalize_interval=6, rho_half=True)
    a = device.run(cfg)
    cfg.rho_half = False
    b = device.run(cfg)
    assert np.array_equal(a.accepted, b.accepted) and close(a.entropies, b.entropies, 1e-12).all()
    bad = tg.ExperimentConfig(spins=14, steps=8, procedures=4, seed=5, inject_fault=2, fault_procedure=1,
                              fault_step=2, rho_half=True)
    with pytest.raises(ValueError, match="entanglement_entropy: state not normalized"):
        device.run(bad)


# --------------------------------- von Neumann above S = 15 (vn_large.cuh, work queue only)
@pytest.mark.parametrize("spins,procs,steps,obj", [(16, 2, 3, "max"), (17, 1, 2, "min")])
def test_von_neumann_large_vs_oracle(device, oracle, spins, procs, steps, obj):
    """d_a = 256: TILE items store rho, the DEC item tridiagonalises it in global memory
    (Householder, one fused update + matvec pass per reflector) and bisects the Sturm counts;
    the oracle diagonalises with the reference's cyclic Jacobi. Sites and accept flags
    bit-exact, entropies within 1e-10."""
    cfg = tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=19, entropy_kind="von-neumann",
                              objective=obj, initial_state="random")
    rep = device.run(cfg)
    again = device.run(cfg)
    assert_bitwise(rep, again)
    want = oracle.run(McCfg(spins=spins, steps=steps, seed=19, entropy_kind=0, objective=1 if obj == "min" else 0,
                            initial_state=1), 0, procs, threads=procs)
    assert np.array_equal(rep.sites, want.sites)
    assert np.array_equal(rep.accepted, want.accepted)
    assert close(rep.initial_entropy, want.initial).all(), np.abs(rep.initial_entropy - want.initial).max()
    assert close(rep.entropies, want.entropies).all(), np.abs(rep.entropies - want.entropies).max()


@pytest.mark.parametrize("spins", [18, 20])
def test_von_neumann_large_invariants(device, spins):
    """d_a = 512 and 1024 (config 4's chain), beyond the oracle's reach: a Haar-random start's
    von Neumann entropy is at least its Renyi-2 entropy (same state, same seed) and below
    floor(S/2) ln 2; traces stay in that range; reruns bitwise."""
    import math
    base = dict(spins=spins, steps=2, procedures=2, seed=23, initial_state="random")
    vn = device.run(tg.ExperimentConfig(entropy_kind="von-neumann", **base))
    r2 = device.run(tg.ExperimentConfig(entropy_kind="renyi-2", **base))
    assert_bitwise(vn, device.run(tg.ExperimentConfig(entropy_kind="von-neumann", **base)))
    bound = (spins // 2) * math.log(2) + 1e-9
    assert np.all(vn.initial_entropy >= r2.initial_entropy - 1e-12)
    assert np.all(vn.initial_entropy <= bound) and np.all(vn.entropies <= bound) and np.all(vn.entropies >= 0)
    assert np.array_equal(vn.sites, r2.sites)  # the proposal stream does not depend on the entropy


@pytest.mark.parametrize("spins", [16, 17])
def test_von_neumann_large_not_normalized(device, spins):
    """A non-unitary gate under the large-S von Neumann path (DEC items that pause the
    producer): the reference's std::invalid_argument message, and the run without the hook is
    clean (the paused producer is released on every DEC, failed rows included)."""
    cfg = tg.ExperimentConfig(spins=spins, steps=3, procedures=3, seed=2, entropy_kind="von-neumann",
                              inject_fault=2, fault_procedure=1, fault_step=1)
    with pytest.raises(ValueError, match="entanglement_entropy: state not normalized"):
        device.run(cfg)
    cfg.inject_fault = 0
    assert device.run(cfg).entropies.shape == (3, 3)


@pytest.mark.slow
@pytest.mark.parametrize("spins,procs,steps", [(20, 4, 6), (16, 8, 60), (18, 3, 12)])
def test_queue_long_trajectories_vs_oracle(device, oracle, monkeypatch, spins, procs, steps):
    """The headline kernel (work queue) on config 4's chain and on longer L = 16 / 18 runs,
    against the oracle (the reference's O(d^3) CPU GEMM: ~7 s per L = 20 step on one core,
    so the replicas run on parallel host threads): sites and accept flags bit-exact,
    entropies within 1e-10."""
    monkeypatch.setenv("TG_HBM_QUEUE", "1")
    cfg = tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=77, initial_state="random")
    rep = device.run(cfg)
    want = oracle.run(McCfg(spins=spins, steps=steps, seed=77, initial_state=1), 0, procs)
    assert np.array_equal(rep.sites, want.sites)
    assert np.array_equal(rep.accepted, want.accepted)
    assert close(rep.entropies, want.entropies).all(), np.abs(rep.entropies - want.entropies).max()
    assert close(rep.initial_entropy, want.initial).all()


@pytest.mark.slow
@pytest.mark.parametrize("spins,steps", [(22, 2), (24, 1)])
def test_queue_largest_chains_vs_cluster(device, monkeypatch, spins, steps):
    """The largest chains (2048^3 and 4096^3 complex GEMMs) default to the work queue, all
    SMs on one replica's tiles: bitwise the 4-CTA cluster schedule's traces, and the model's
    choice is the queue."""
    assert tg.lib().tg_hbm_schedule(spins, 1, 1) == 1
    cfg = tg.ExperimentConfig(spins=spins, steps=steps, procedures=1, seed=5, initial_state="random")
    a = run_with(device, cfg, monkeypatch, TG_HBM_QUEUE="0", TG_HBM_CTAS_PER_REPLICA="4")
    b = run_with(device, cfg, monkeypatch)
    assert_bitwise(a, b)


@pytest.mark.slow
def test_queue_only_options_split_into_batches(device):
    """rho_half runs on the work queue only, which takes at most 8192 rows per launch: a
    larger run is split into batches (capi.cpp launch). Every replica still matches its own
    run in a small batch bit for bit (traces depend only on (seed, procedure))."""
    big = tg.ExperimentConfig(spins=14, steps=2, procedures=9000, seed=3, rho_half=True)
    rep = device.run(big)
    for p in (0, 8191, 8192, 8999):
        one = device.run(tg.ExperimentConfig(spins=14, steps=2, procedures=p + 1, seed=3, rho_half=True))
        assert np.array_equal(rep.entropies[p].view(np.uint64), one.entropies[p].view(np.uint64)), p
        assert np.array_equal(rep.accepted[p], one.accepted[p])


def test_queue_failing_replica_positions(device, monkeypatch):
    """A replica that fails its norm check early (procedure 5, step 1) or late (procedure 0,
    step 4) inside one queue launch: its remaining items are skipped while the others run to
    the end, and the reference's message is reported."""
    monkeypatch.setenv("TG_HBM_QUEUE", "1")
    cfg = tg.ExperimentConfig(spins=16, steps=6, procedures=7, seed=9, inject_fault=2, fault_procedure=5,
                              fault_step=1)
    with pytest.raises(ValueError, match="entanglement_entropy: state not normalized"):
        device.run(cfg)
    cfg.fault_procedure, cfg.fault_step = 0, 4
    with pytest.raises(ValueError, match="entanglement_entropy: state not normalized"):
        device.run(cfg)
