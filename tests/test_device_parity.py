"""GPU parity suite: the CUDA path through the C ABI against the
oracle / the reference's golden outputs. Integer work (RNG words, sites, accept flags) is
bit-exact; floating point within the north-star tolerance |got-want| <= 1e-10*max(|want|,1)
(SURVEY fact 8). Run on a B200: `python -m pytest tests -m gpu`."""
import math

import numpy as np
import pytest
from conftest import TRAJ_CASES, VN_CASES, cfg_from_golden, entropy_kind_of, load_traj
from oracle_lib import McCfg

import paper_2203_09353_b200 as tg

pytestmark = pytest.mark.gpu
TOL = 1e-10


def close(got, want, tol=TOL):
    got, want = np.asarray(got), np.asarray(want)
    return np.abs(got - want) <= tol * np.maximum(np.abs(want), 1.0)


# ---------------------------------------------------------------- T1/T2 RNG and gates
@pytest.mark.parametrize("seed", [0, 1, 42, 2**64 - 1])
@pytest.mark.parametrize("p", [0, 1, 7, 65535])
def test_t1_device_xoshiro_bitwise(kats, oracle, seed, p):
    got = tg.probe_rng(seed, p, 10000)
    assert np.array_equal(got, oracle.first_u64(seed, p, 10000))
    idx = [i for i, (s, q) in enumerate(kats["u64_pairs"]) if int(s) == seed and int(q) == p][0]
    assert np.array_equal(got[:256], kats["u64"][idx])


@pytest.mark.parametrize("spins,initial", [(8, "product"), (2, "product"), (13, "product"), (6, "random")])
def test_t2_t3_gate_stream(oracle, spins, initial):
    """Sites bit-exact, Haar U within a few ulp of the reference, u_accept bit-exact."""
    steps = 300
    sites, u, ua = tg.probe_gates(spins, 11, 5, steps, initial)
    _, _, _, osites, ou, _ = oracle.mc_procedure(
        McCfg(spins=spins, steps=steps, seed=11, initial_state=1 if initial == "random" else 0), 5)
    assert np.array_equal(sites, osites)
    assert np.array_equal(ua, ou)
    # Haar matrices: replay the stream on the oracle side
    st_u = oracle.haar_stream(spins, 11, 5, steps, initial == "random")
    ulp = np.abs(u - st_u) / np.spacing(np.maximum(np.abs(st_u), 1e-300))
    assert np.abs(u - st_u).max() <= 1e-14
    us = u.view(np.complex128).reshape(-1, 4, 4).transpose(0, 2, 1)
    gram = np.einsum("nki,nkj->nij", us.conj(), us) - np.eye(4)
    assert np.abs(gram).max() <= 1e-12
    assert np.median(ulp) <= 4


@pytest.mark.parametrize("spins,rows,steps,random_init,reject_below", [
    (12, 37, 1000, False, 0),          # 4 chunks, the reference threshold (no rejection)
    (8, 5, 700, True, 0),              # random-start draws before the steps (T^(2^(S+1)) jump)
    (12, 9, 900, False, 1 << 62),      # forced rejections: every replica takes the fixup path
    (5, 3, 300, True, (1 << 63) + 5),  # forced rejections after random-start draws
])
def test_t2_rng_chunked_jump_ahead(spins, rows, steps, random_init, reject_below):
    """The pre-pass's chunked xoshiro256++ (chunks of 64 steps started by GF(2) jump
    matrices, rejection fixup) reproduces one sequential stream per replica word for word."""
    assert tg.probe_rng_chunking(spins, rows, steps, random_init, reject_below) == 0


# ------------------------------------------------------------------- T4 gate application
# S <= 12 applies the gate in fused (DFMA) form — DMMA and DFMA share the FP64 pipe on
# sm_100a, so halving the gate's op count is worth ~6% of the step: within
# a few ulp of the reference's unfused rounding. S >= 13 keeps the unfused form: bitwise.
GATE_TOL = 4 * np.finfo(np.float64).eps


def test_t4_gate_vs_reference(kats):
    for i in range(int(kats["n_gates"])):
        spins, site = (int(x) for x in kats[f"gate{i}_meta"])
        got = tg.probe_apply_gate(spins, kats[f"gate{i}_in"], site, kats[f"gate{i}_u"])
        want = kats[f"gate{i}_out"]
        if spins <= 12:
            assert np.abs(got - want).max() <= GATE_TOL * np.abs(want).max(), (spins, site)
        else:
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (spins, site)


@pytest.mark.parametrize("spins", [14, 16])
def test_t4_gate_bitwise_hbm(oracle, spins):
    rng = np.random.default_rng(spins)
    psi = rng.standard_normal(1 << spins) + 1j * rng.standard_normal(1 << spins)
    psi /= np.linalg.norm(psi)
    u = oracle.haar(3, spins, 1)[0].view(np.complex128)
    for site in (0, 1, spins // 2 - 1, spins - 2):
        got = tg.probe_apply_gate(spins, psi, site, u)
        want = oracle.apply_gate(spins, psi, site, u)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), site


# ---------------------------------------------------------------- T5 GEMM (rho and batched)
@pytest.mark.parametrize("spins", [2, 3, 4, 6, 8, 9, 12, 13, 14])
def test_t5_rho_entropy_vs_reference(kats, spins):
    states = kats[f"ent_{spins}_states"]
    e, n = tg.probe_entropy(spins, states)
    assert close(e, kats[f"ent_{spins}_renyi2"]).all()
    assert np.abs(n - 1.0).max() <= 1e-13


@pytest.mark.parametrize("spins", [2, 3, 4, 6, 8, 9, 12, 13, 14])
def test_t5_von_neumann_vs_reference(kats, oracle, spins):
    """Device eigen-solver (vn.cuh, and vn_packed.cuh for d_a = 128: Householder + Sturm
    multisection) against the reference's
    cyclic Jacobi (linalg.cpp:161-232) on the golden states (the oracle's bitwise restatement
    where the fixture has no vN values)."""
    states = kats[f"ent_{spins}_states"]
    want = kats[f"ent_{spins}_vn"]
    if want.size == 0:
        want = np.array([oracle.entropy(spins, s, 0) for s in states])
    e, n = tg.probe_entropy(spins, states, kind="von-neumann")
    assert close(e, want).all(), np.max(np.abs(e - want))
    assert np.abs(n - 1.0).max() <= 1e-13


@pytest.mark.parametrize("spins", [5, 7, 10, 11, 12, 13, 14, 15])
def test_t5_von_neumann_structured_states(oracle, spins):
    """Spectra the annealer produces: product states (rank 1), low Schmidt rank with
    degenerate and tiny (<1e-15, dropped) eigenvalues, and Haar-random (full rank)."""
    rng = np.random.default_rng(7 * spins)
    da, db = 1 << (spins // 2), 1 << (spins - spins // 2)
    states = []
    for rank, weights in [(1, None), (2, [0.5, 0.5]), (3, [0.6, 0.4 - 1e-16, 1e-16]), (4, None),
                          (da, None), (da, "geometric")]:
        a = np.linalg.qr(rng.standard_normal((da, da)) + 1j * rng.standard_normal((da, da)))[0][:, :rank]
        b = np.linalg.qr(rng.standard_normal((db, db)) + 1j * rng.standard_normal((db, db)))[0][:, :rank]
        if weights is None:
            w = rng.random(rank)
        elif weights == "geometric":
            w = 0.5 ** np.arange(rank)
        else:
            w = np.array(weights)
        w = np.sqrt(w / w.sum())
        Psi = (a * w) @ b.T
        psi = Psi.T.reshape(-1)  # psi[a + b*d_a] = Psi[a, b]
        states.append(psi / np.linalg.norm(psi))
    states = np.array(states)
    e, _ = tg.probe_entropy(spins, states, kind="von-neumann")
    want = np.array([oracle.entropy(spins, s, 0) for s in states])
    assert close(e, want).all(), np.max(np.abs(e - want))


@pytest.mark.parametrize("spins", [16, 18])
def test_t5_rho_entropy_large(oracle, spins):
    rng = np.random.default_rng(100 + spins)
    psi = rng.standard_normal(1 << spins) + 1j * rng.standard_normal(1 << spins)
    psi /= np.linalg.norm(psi)
    e, n = tg.probe_entropy(spins, psi[None])
    # numpy reference for the Frobenius norm of rho (the oracle's O(d^3) loop is slow at S=18)
    da = 1 << (spins // 2)
    Psi = psi.reshape(-1, da).T
    rho = Psi @ Psi.conj().T
    want = -math.log(np.sum(np.abs(rho) ** 2))
    assert close(e, [max(want, 0.0)], 1e-11).all()
    if spins == 16:
        assert close(e, [oracle.entropy(spins, psi, 1)]).all()


def test_t5_batched_gemm_vs_reference(device, kats):
    for i in range(40):
        a, b, c = kats[f"g{i}_a"], kats[f"g{i}_b"], kats[f"g{i}_c"]
        al, be = kats[f"g{i}_ab"]
        (out,), recs = device.batched_gemm([a], [b], [c], alpha=al, beta=be, records=True)
        want = kats[f"g{i}_out"]
        err = np.abs(out - want).max() / np.abs(want).max()
        assert err <= 1e-13, (i, err)
        assert recs[0].flops == 8 * a.shape[0] * b.shape[1] * a.shape[1]


def test_t5_batched_gemm_ordered_and_large(device, oracle):
    rng = np.random.default_rng(7)
    for (m, n, k, batch) in [(64, 64, 64, 17), (100, 37, 130, 5), (256, 256, 256, 3), (1, 1, 1, 4)]:
        As = [rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k)) for _ in range(batch)]
        Bs = [rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n)) for _ in range(batch)]
        outs, recs = device.batched_gemm(As, Bs, records=True, procedures=list(range(100, 100 + batch)))
        for i in range(batch):
            want = As[i] @ Bs[i]
            assert np.abs(outs[i] - want).max() <= 1e-13 * max(1.0, np.abs(want).max()) * max(1, k)
        assert [r.procedure for r in recs] == list(range(100, 100 + batch))
    with pytest.raises(ValueError, match="fixed-size"):
        device.batched_gemm([np.eye(2), np.eye(3)], [np.eye(2), np.eye(3)])


def test_batched_gemm_unit_epilogue_bitwise(device, monkeypatch):
    """alpha = 1, beta = 0, no C: the TMA kernels' one-op epilogue (acc + 0.0) is bitwise the
    general alpha/beta formula of the cp.async kernel, including -0 entries (a zero column of
    A makes every product term -0 or +0)."""
    rng = np.random.default_rng(5)
    m = n = k = 64
    As = [rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k)) for _ in range(6)]
    Bs = [rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n)) for _ in range(6)]
    As[0][:, :] = -0.0  # -0 products: the epilogue decides the sign of every zero
    As[1][3, :] = 0.0
    monkeypatch.setenv("TG_ZGEMM_TMA", "0")
    ref = device.batched_gemm(As, Bs)
    monkeypatch.setenv("TG_ZGEMM_TMA", "1")
    for warps in ("4", "5", "8", "9", "16"):
        monkeypatch.setenv("TG_ZGEMM_WARPS", warps)
        got = device.batched_gemm(As, Bs)
        for i in range(6):
            assert np.array_equal(np.ascontiguousarray(got[i]).view(np.uint64),
                                  np.ascontiguousarray(ref[i]).view(np.uint64)), (warps, i)


@pytest.mark.parametrize("m,n,k,batch", [(64, 64, 64, 17), (72, 37, 40, 5), (256, 256, 256, 3), (8, 8, 8, 9),
                                         (200, 64, 136, 3), (128, 130, 1024, 2)])
def test_batched_gemm_tma_vs_cp_async_bitwise(device, monkeypatch, m, n, k, batch):
    """The TMA-staged batched GEMM (m, k multiples of 8; tile edges are TMA out-of-bounds
    zeros) and the cp.async one feed the DMMAs the same operands in the same order:
    bitwise-identical outputs, including alpha/beta with C."""
    rng = np.random.default_rng(m * 7 + n + k)
    As = [rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k)) for _ in range(batch)]
    Bs = [rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n)) for _ in range(batch)]
    Cs = [rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)) for _ in range(batch)]
    monkeypatch.setenv("TG_ZGEMM_TMA", "0")
    ref = device.batched_gemm(As, Bs, Cs, alpha=0.5 - 0.25j, beta=1.5 + 2j)
    monkeypatch.setenv("TG_ZGEMM_TMA", "1")
    got = device.batched_gemm(As, Bs, Cs, alpha=0.5 - 0.25j, beta=1.5 + 2j)
    for warps in ("4", "5", "8", "9", "16"):  # every warp layout of the TMA kernel (5, 9: 4, 8 + producer)
        monkeypatch.setenv("TG_ZGEMM_WARPS", warps)
        again = device.batched_gemm(As, Bs, Cs, alpha=0.5 - 0.25j, beta=1.5 + 2j)
        for i in range(batch):
            assert np.array_equal(np.ascontiguousarray(again[i]).view(np.uint64),
                                  np.ascontiguousarray(got[i]).view(np.uint64)), (warps, i)
    for i in range(batch):
        assert np.array_equal(np.ascontiguousarray(got[i]).view(np.uint64), np.ascontiguousarray(ref[i]).view(np.uint64)), i
        want = 0.5 - 0.25j
        want = want * (As[i] @ Bs[i]) + (1.5 + 2j) * Cs[i]
        assert np.abs(got[i] - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


# -------------------------------------------------------------------- T6 analytic states
def test_t6_analytic_entropies():
    for spins in (4, 6, 8, 12, 14):
        prod = np.zeros(1 << spins, complex)
        prod[0] = 1
        ghz = np.zeros(1 << spins, complex)
        ghz[0] = ghz[-1] = 1 / math.sqrt(2)
        # Bell pairs across the cut: floor(S/2) ... use one Bell pair (sites 0 and S/2): ln 2
        e, _ = tg.probe_entropy(spins, np.stack([prod, ghz]))
        assert abs(e[0]) <= 1e-10
        assert abs(e[1] - math.log(2)) <= 1e-10


# ------------------------------------------------------------ T7 trajectories vs reference
def cfg_from(g, procedures=None):
    return cfg_from_golden(g, procedures)


def assert_traj_parity(rep, g, rows=None):
    rows = rows if rows is not None else slice(None)
    assert np.array_equal(rep.sites, g["sites"][rows]), "site sequence differs"
    mism = np.argwhere(rep.accepted != g["accepted"][rows])
    assert mism.size == 0, f"accept flags differ at {mism[:5].tolist()}"
    ok = close(rep.entropies, g["entropies"][rows])
    assert ok.all(), f"max scaled diff {np.max(np.abs(rep.entropies - g['entropies'][rows]))}"
    assert close(rep.initial_entropy, g["initial"][rows]).all()


@pytest.mark.parametrize("name", TRAJ_CASES)
def test_t7_trajectory_parity(device, name):
    g = load_traj(name)
    rep = device.run(cfg_from(g))
    assert_traj_parity(rep, g)
    assert abs(rep.average_entropy - float(g["average"])) <= TOL * max(1.0, abs(float(g["average"])))
    assert rep.total_flops == (rep.entropies.size + rep.initial_entropy.size) * tg.step_flops(int(g["spins"]))


@pytest.mark.parametrize("name", VN_CASES)
def test_t7_von_neumann_trajectory_parity(device, name):
    g = load_traj(name)
    rep = device.run(cfg_from(g))
    assert_traj_parity(rep, g)
    assert abs(rep.average_entropy - float(g["average"])) <= TOL * max(1.0, abs(float(g["average"])))


@pytest.mark.parametrize("spins,objective", [(14, "max"), (15, "min")])
def test_t7_von_neumann_packed_vs_oracle(device, oracle, spins, objective):
    """d_a = 128 (S = 14, 15): rho through the slab's scratch planes, packed-lower Householder
    (vn_packed.cuh) inside the anneal loop, against the oracle's Jacobi trajectories."""
    cfg = tg.ExperimentConfig(spins=spins, steps=6, procedures=2, seed=5, objective=objective,
                              entropy_kind="von-neumann")
    rep = device.run(cfg)
    want = oracle.run(McCfg(spins=spins, steps=6, seed=5, entropy_kind=0,
                            objective=0 if objective == "max" else 1), 0, 2)
    assert np.array_equal(rep.sites, want.sites)
    assert np.array_equal(rep.accepted, want.accepted)
    assert close(rep.entropies, want.entropies).all(), np.max(np.abs(rep.entropies - want.entropies))
    assert close(rep.initial_entropy, want.initial).all()


@pytest.mark.slow
def test_hbm_renormalisation_vs_oracle(device, oracle, monkeypatch):
    """HBM tier across the every-1000-steps renormalisation (spinmc.cpp:246-248; canonical
    quarter sums) on one CTA and on a 4-CTA cluster: bitwise equal, and equal to the oracle
    (sites, accept flags bit-exact; entropies within 1e-10)."""
    cfg = tg.ExperimentConfig(spins=14, steps=1010, procedures=1, seed=6)
    want = oracle.run(McCfg(spins=14, steps=1010, seed=6), 0, 1)
    monkeypatch.setenv("TG_HBM_CTAS_PER_REPLICA", "1")
    a = device.run(cfg)
    monkeypatch.setenv("TG_HBM_CTAS_PER_REPLICA", "4")
    b = device.run(cfg)
    assert np.array_equal(a.entropies.view(np.uint64), b.entropies.view(np.uint64))
    assert np.array_equal(a.sites, want.sites)
    assert np.array_equal(a.accepted, want.accepted)
    assert close(a.entropies, want.entropies).all(), np.max(np.abs(a.entropies - want.entropies))


@pytest.mark.slow
def test_t7_config4_shape_vs_oracle(device, oracle, monkeypatch):
    """BASELINE config 4's chain (L=20, 1024x1024x1024 complex GEMMs): a replica's initial
    entropy and first steps against the oracle (the reference's O(d^3) GEMM, ~7 s per step
    on one core), on one CTA and on a 4-CTA cluster (bitwise equal)."""
    cfg = tg.ExperimentConfig(spins=20, steps=2, procedures=1, seed=4)
    want = oracle.run(McCfg(spins=20, steps=2, seed=4), 0, 1)
    monkeypatch.setenv("TG_HBM_CTAS_PER_REPLICA", "1")
    a = device.run(cfg)
    monkeypatch.setenv("TG_HBM_CTAS_PER_REPLICA", "4")
    b = device.run(cfg)
    assert np.array_equal(a.entropies.view(np.uint64), b.entropies.view(np.uint64))
    assert np.array_equal(a.sites, want.sites)
    assert np.array_equal(a.accepted, want.accepted)
    assert close(a.entropies, want.entropies).all(), np.max(np.abs(a.entropies - want.entropies))
    assert close(a.initial_entropy, want.initial).all()


def test_t7_von_neumann_appendix_a(device):
    rep = device.run(cfg_from(load_traj("vn_cfg1")))
    assert int(rep.accepted.sum()) == 59795
    assert abs(rep.average_entropy - 2.360208109374111) <= 1e-10 * 2.37


def test_t7_config1_appendix_a(device):
    g = load_traj("cfg1")
    rep = device.run(cfg_from(g))
    assert int(rep.accepted.sum()) == 59437
    assert list(rep.sites[0, :12]) == [0, 1, 5, 6, 2, 2, 0, 5, 4, 2, 0, 2]
    assert abs(rep.average_entropy - 2.2063680065173292) <= 1e-10 * 2.21
    # Appendix A: the product state's initial entropy is -0.0 bit for bit (rho = |0><0| exactly,
    # -log(1) = -0.0, and (e < 0) ? 0 : e keeps it, as std::max does), on every replica
    assert np.all(rep.initial_entropy == 0.0) and np.all(np.signbit(rep.initial_entropy))
    assert np.array_equal(rep.initial_entropy.view(np.uint64), g["initial"].view(np.uint64))


@pytest.mark.parametrize("spins,queue", [(8, "0"), (12, "0"), (14, "0"), (14, "1"), (20, "1")])
def test_product_state_initial_entropy_is_negative_zero(device, monkeypatch, spins, queue):
    """Both tiers and both HBM schedules: -0.0 exactly for the product state, like the reference."""
    monkeypatch.setenv("TG_HBM_QUEUE", queue)
    rep = device.run(tg.ExperimentConfig(spins=spins, steps=1, procedures=3, seed=1))
    assert np.all(rep.initial_entropy == 0.0) and np.all(np.signbit(rep.initial_entropy)), rep.initial_entropy


@pytest.mark.slow
def test_t7_config2_subset_full_length(device, oracle):
    """BASELINE configs[1] (S=12, 1024 replicas, 10k steps) on the device; the oracle checks
    a bounded subset of replicas over the full 10k steps; all rows obey the invariants."""
    cfg = tg.ExperimentConfig(spins=12, steps=10000, procedures=1024)
    rep = device.run(cfg)
    sub = list(range(0, 1024, 128))
    ocfg = McCfg(spins=12, steps=10000)
    for p in sub:
        init, ent, acc, sites, _, _ = oracle.mc_procedure(ocfg, p)
        assert np.array_equal(rep.sites[p], sites)
        assert np.array_equal(rep.accepted[p], acc), p
        assert close(rep.entropies[p], ent).all()
    assert (rep.sites < 11).all()
    assert (rep.entropies >= 0).all() and (rep.entropies <= 6 * math.log(2) + 1e-9).all()
    fin = rep.entropies[:, -1]
    assert rep.average_entropy == pytest.approx(float(np.mean(fin)), rel=1e-12)


# -------------------------------------------------------------- T8 determinism / sharding
def test_t8_rerun_bitwise_and_shards(device):
    cfg = tg.ExperimentConfig(spins=10, steps=300, procedures=37, seed=99)
    a = device.run(cfg)
    b = device.run(cfg)
    assert np.array_equal(a.entropies.view(np.uint64), b.entropies.view(np.uint64))
    assert np.array_equal(a.accepted, b.accepted)
    # shard (rank 1 of 3) sees exactly replicas 1, 4, 7, ... with identical traces
    cfg3 = tg.ExperimentConfig(spins=10, steps=300, procedures=37, seed=99, shard_index=1, shard_count=3)
    s = device.run(cfg3)
    assert np.array_equal(s.procedures, np.arange(1, 37, 3))
    assert np.array_equal(s.entropies.view(np.uint64), a.entropies[1::3].view(np.uint64))


def test_t8_hbm_tier_rerun_bitwise(device):
    cfg = tg.ExperimentConfig(spins=14, steps=20, procedures=5, seed=3)
    a = device.run(cfg)
    b = device.run(cfg)
    assert np.array_equal(a.entropies.view(np.uint64), b.entropies.view(np.uint64))


# ------------------------------------------------------------------------ T9 error paths
def test_t9_fault_injection_detected(device):
    g = load_traj("s12")
    cfg = cfg_from(g)
    cfg.inject_fault = 1
    rep = device.run(cfg)
    assert not close(rep.initial_entropy, g["initial"]).all() or not close(rep.entropies, g["entropies"]).all()


def test_t9_shutdown_and_config_errors():
    dev = tg.Device([0])
    dev.shutdown()
    with pytest.raises(tg.SubmissionError):
        dev.run(tg.ExperimentConfig(spins=4, steps=2, procedures=1))
    dev.close()
    with pytest.raises(tg.ConfigError, match=r"spins out of range \[2,30\]"):
        tg.run_experiment(tg.ExperimentConfig(spins=31))
    with pytest.raises(tg.ConfigError):
        tg.Device([0]).run(tg.ExperimentConfig(spins=4, devices=2))


def test_zero_steps_and_single_replica(device):
    rep = device.run(tg.ExperimentConfig(spins=8, steps=0, procedures=3))
    assert rep.entropies.shape == (3, 0)
    assert np.all(np.abs(rep.initial_entropy) <= 1e-15)
    assert rep.average_entropy == pytest.approx(float(np.mean(rep.initial_entropy)), abs=1e-15)


@pytest.mark.parametrize("spins,procs,steps", [(14, 5, 20), (16, 3, 6), (13, 4, 12)])
def test_hbm_cluster_split_bitwise(device, oracle, spins, procs, steps, monkeypatch):
    """HBM tier: one replica per CTA, per 2-CTA and per 4-CTA cluster (rank k takes the
    tiles t = k mod CS, chain sums exchanged through DSMEM) produce bitwise-identical traces
    (four canonical chains, canonical renormalisation quarters), and match the oracle."""
    cfg = tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=8, initial_state="random")
    monkeypatch.setenv("TG_HBM_CTAS_PER_REPLICA", "1")
    a = device.run(cfg)
    for cs in ("2", "4"):
        monkeypatch.setenv("TG_HBM_CTAS_PER_REPLICA", cs)
        b = device.run(cfg)
        assert np.array_equal(a.entropies.view(np.uint64), b.entropies.view(np.uint64)), cs
        assert np.array_equal(a.accepted, b.accepted), cs
        assert np.array_equal(a.initial_entropy.view(np.uint64), b.initial_entropy.view(np.uint64)), cs
    want = oracle.run(McCfg(spins=spins, steps=steps, seed=8, initial_state=1), 0, procs)
    assert np.array_equal(b.accepted, want.accepted)
    assert close(b.entropies, want.entropies).all()


@pytest.mark.parametrize("spins,procs,steps,cs", [(14, 5, 20, "1"), (16, 3, 6, "2"), (13, 4, 12, "1"), (14, 2, 9, "4")])
def test_hbm_tma_vs_cp_async_bitwise(device, oracle, spins, procs, steps, cs, monkeypatch):
    """HBM tier: the GEMM stages filled by TMA tensor copies (64-B swizzled panels, mbarrier
    pipeline) and by per-thread cp.async (padded panels, barrier per chunk) feed the DMMAs
    the same operands in the same order: bitwise-identical traces, equal to the oracle."""
    cfg = tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=17, initial_state="random")
    monkeypatch.setenv("TG_HBM_CTAS_PER_REPLICA", cs)
    monkeypatch.setenv("TG_HBM_TMA", "0")
    a = device.run(cfg)
    monkeypatch.setenv("TG_HBM_TMA", "1")
    b = device.run(cfg)
    assert np.array_equal(a.entropies.view(np.uint64), b.entropies.view(np.uint64))
    assert np.array_equal(a.initial_entropy.view(np.uint64), b.initial_entropy.view(np.uint64))
    assert np.array_equal(a.accepted, b.accepted)
    want = oracle.run(McCfg(spins=spins, steps=steps, seed=17, initial_state=1), 0, procs)
    assert np.array_equal(b.accepted, want.accepted)
    assert np.array_equal(b.sites, want.sites)
    assert close(b.entropies, want.entropies).all()


@pytest.mark.parametrize("spins,procs,steps", [(12, 7, 40), (14, 5, 6), (8, 9, 300)])
def test_multi_device_binding_same_gpu(oracle, spins, procs, steps):
    """The in-process multi-GPU path (one host thread + stream + buffers per device, replica
    p on device p mod devices, bench.cpp:171) with both "devices" mapped to GPU 0: traces are
    bitwise those of the one-device run, and match the oracle."""
    cfg1 = tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=21, devices=1)
    cfg2 = tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=21, devices=2)
    with tg.Device([0]) as d1:
        a = d1.run(cfg1)
    with tg.Device([0, 0]) as d2:
        b = d2.run(cfg2)
    assert np.array_equal(a.entropies.view(np.uint64), b.entropies.view(np.uint64))
    assert np.array_equal(a.accepted, b.accepted)
    assert np.array_equal(a.sites, b.sites)
    assert a.average_entropy == b.average_entropy
    want = oracle.run(McCfg(spins=spins, steps=steps, seed=21), 0, procs)
    assert np.array_equal(b.accepted, want.accepted)


@pytest.mark.slow
@pytest.mark.parametrize("spins", [22, 24])
def test_largest_chains_invariants(monkeypatch, spins):
    """S = 22 and 24 (2^24 amplitudes, 4096^3 complex GEMMs): too large for the oracle, so
    the invariants — 1-CTA and 4-CTA runs bitwise equal, every state normalised (no kernel
    error), entropies within [0, floor(S/2) ln 2], and a Haar-random start near Page's value."""
    cfg = tg.ExperimentConfig(spins=spins, steps=2, procedures=1, seed=17, initial_state="random")
    monkeypatch.setenv("TG_HBM_CTAS_PER_REPLICA", "1")
    with tg.Device([0]) as d:
        a = d.run(cfg)
    monkeypatch.setenv("TG_HBM_CTAS_PER_REPLICA", "4")
    with tg.Device([0]) as d:
        b = d.run(cfg)
    assert np.array_equal(a.entropies.view(np.uint64), b.entropies.view(np.uint64))
    assert np.array_equal(a.initial_entropy.view(np.uint64), b.initial_entropy.view(np.uint64))
    bound = (spins // 2) * math.log(2) + 1e-9
    assert np.all(a.entropies >= 0) and np.all(a.entropies <= bound)
    assert 0 <= a.initial_entropy[0] <= bound
    # a Haar-random state of 2^S amplitudes is close to maximally entangled (Page)
    assert a.initial_entropy[0] > bound - 1.5


def test_hbm_split_launch_geometry(device, oracle):
    """with pinned trace arrays tg_anneal_run launches all full waves first
    (here rows 0..147 of 174 at L = 13: 148 one-CTA clusters) although the workspace was sized
    for the whole batch's geometry (74 two-CTA clusters). The slab region is now sized for any
    launch of <= rows replicas (min(rows, SMs) slabs) and the launch clamps to it: pinned
    (split) and pageable (single launch) runs are bitwise equal and match the oracle."""
    import torch
    cfg = tg.ExperimentConfig(spins=13, steps=5, procedures=174, seed=9)
    rows, steps = 174, 5
    pinned = {
        "initial": torch.empty(rows, dtype=torch.float64, pin_memory=True).numpy(),
        "final": torch.empty(rows, dtype=torch.float64, pin_memory=True).numpy(),
        "entropies": torch.empty((rows, steps), dtype=torch.float64, pin_memory=True).numpy(),
        "accepted": torch.empty((rows, steps), dtype=torch.uint8, pin_memory=True).numpy(),
        "sites": torch.empty((rows, steps), dtype=torch.uint8, pin_memory=True).numpy(),
    }
    a = device.run(cfg, out=pinned)
    b = device.run(cfg)
    assert np.array_equal(a.entropies.view(np.uint64), b.entropies.view(np.uint64))
    assert np.array_equal(a.accepted, b.accepted)
    for p in (0, 73, 147, 148, 173):
        _, ent, acc, sites, _, _ = oracle.mc_procedure(McCfg(spins=13, steps=steps, seed=9), p)
        assert np.array_equal(a.accepted[p], acc) and np.array_equal(a.sites[p], sites)
        assert close(a.entropies[p], ent).all()


def test_nccl_gather_of_finals(monkeypatch):
    """The in-process multi-GPU path gathers the final entropies with one NCCL all-gather
    (C++ host code, NCCL loaded at run time). Forced on one GPU here (a one-rank
    communicator): the average is bit for bit the host-copy path's. GPUs repeated in a context
    (NCCL: one rank per GPU) fall back to the host copies."""
    cfg = tg.ExperimentConfig(spins=10, steps=30, procedures=9, seed=4)
    with tg.Device([0]) as d:
        host = d.run(cfg)
        monkeypatch.setenv("TG_NCCL_FORCE", "1")
        viaccl = d.run(cfg)
    assert host.nccl_ranks == 0 and viaccl.nccl_ranks == 1
    assert viaccl.average_entropy == host.average_entropy
    assert np.array_equal(viaccl.final_entropy.view(np.uint64), host.final_entropy.view(np.uint64))
    with tg.Device([0, 0]) as d2:
        rep = d2.run(tg.ExperimentConfig(spins=10, steps=30, procedures=9, seed=4, devices=2))
    assert rep.nccl_ranks == 0 and rep.average_entropy == host.average_entropy
