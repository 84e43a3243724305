"""Randomised parity sweep: device trajectories against the oracle over random chain
lengths (both tiers; the HBM tier on its default schedule, the work queue, 1/2/4-CTA
clusters or the opt-in Hermitian half of rho), replica counts, step counts that cross the
pre-pass's chunk boundaries and the renormalisation interval, objectives, initial states
and entropy kinds (von Neumann up to S = 16, the work queue's eigen-solver). Sites and
accept flags bit-exact, entropies within 1e-10 (scaled)."""
import os

import numpy as np
import pytest
from oracle_lib import McCfg

import paper_2203_09353_b200 as tg

TOL = 1e-10


def cases(n=120, seed=2025):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        spins = int(rng.choice([2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 12, 12, 13, 14, 14, 15, 16]))
        vn = spins <= 12 and rng.random() < 0.3
        steps = int(rng.choice([1, 3, 17, 64, 65, 130, 257])) if spins <= 12 else int(rng.choice([1, 5, 9]))
        procs = int(rng.choice([1, 2, 3, 7])) if spins >= 14 else int(rng.choice([1, 2, 5, 13]))
        renorm = int(rng.choice([0, 7, 1000]))
        geom = str(rng.choice(["default", "queue", "cs1", "cs2", "cs4", "half"])) if spins >= 13 else "default"
        if spins == 16 and rng.random() < 0.2:  # von Neumann on the work queue (vn_large.cuh)
            vn, geom, steps, procs = True, "default", int(rng.choice([1, 2])), int(rng.choice([1, 2]))
        out.append(dict(spins=spins, steps=steps, procs=procs, seed=int(rng.integers(0, 1 << 31)),
                        objective=int(rng.integers(0, 2)), initial=int(rng.integers(0, 2)),
                        kind=0 if vn else 1, renorm=renorm, geom=geom))
    return out


GEOM_ENV = {"default": {}, "queue": {"TG_HBM_QUEUE": "1"}, "cs1": {"TG_HBM_QUEUE": "0", "TG_HBM_CTAS_PER_REPLICA": "1"},
            "cs2": {"TG_HBM_QUEUE": "0", "TG_HBM_CTAS_PER_REPLICA": "2"},
            "cs4": {"TG_HBM_QUEUE": "0", "TG_HBM_CTAS_PER_REPLICA": "4"}, "half": {}}


@pytest.mark.gpu
@pytest.mark.slow
# TG_FUZZ_N / TG_FUZZ_SEED widen the sweep on demand (profiles/r01_fuzz_deep.txt)
@pytest.mark.parametrize("c", cases(int(os.environ.get("TG_FUZZ_N", 120)), int(os.environ.get("TG_FUZZ_SEED", 2025))), ids=lambda c: "S{spins}-n{procs}x{steps}-k{kind}-o{objective}-i{initial}-r{renorm}-{geom}".format(**c))
def test_fuzz_trajectory_parity(device, oracle, monkeypatch, c):
    for k, v in GEOM_ENV[c["geom"]].items():
        monkeypatch.setenv(k, v)
    cfg = tg.ExperimentConfig(spins=c["spins"], steps=c["steps"], procedures=c["procs"], seed=c["seed"],
                              objective="max" if c["objective"] == 0 else "min",
                              initial_state="product" if c["initial"] == 0 else "random",
                              entropy_kind="renyi-2" if c["kind"] == 1 else "von-neumann",
                              renormalize_interval=c["renorm"], rho_half=c["geom"] == "half")
    rep = device.run(cfg)
    want = oracle.run(McCfg(spins=c["spins"], steps=c["steps"], seed=c["seed"], entropy_kind=c["kind"],
                            objective=c["objective"], initial_state=c["initial"], renormalize_interval=c["renorm"]),
                      0, c["procs"])
    assert np.array_equal(rep.sites, want.sites)
    mism = np.argwhere(rep.accepted != want.accepted)
    assert mism.size == 0, f"accept flags differ at {mism[:5].tolist()}"
    d = np.abs(rep.entropies - want.entropies) / np.maximum(np.abs(want.entropies), 1.0)
    assert d.size == 0 or d.max() <= TOL, d.max()
    d0 = np.abs(rep.initial_entropy - want.initial) / np.maximum(np.abs(want.initial), 1.0)
    assert d0.max() <= TOL
