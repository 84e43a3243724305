"""Oracle restatement vs the reference compiled from its own sources (oracle/_ref), on
fresh seeds beyond the stored fixtures. CPU; skipped where oracle/_ref was not built."""
import numpy as np
import pytest
from oracle_lib import McCfg


@pytest.mark.parametrize("seed", [1, 42, 2**64 - 1])
def test_rng_and_haar(oracle, reflib, seed):
    for p in (0, 3, 123456):
        assert np.array_equal(oracle.first_u64(seed, p, 500), reflib.first_u64(seed, p, 500))
        a, b = oracle.haar(seed, p, 20), reflib.haar(seed, p, 20)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("cfg,n", [
    (McCfg(spins=9, steps=150, seed=5), 6),
    (McCfg(spins=10, steps=60, seed=9, objective=1, initial_state=1), 4),
    (McCfg(spins=4, steps=400, seed=3, renormalize_interval=13, t0=0.5, t_min=0.5), 6),
    (McCfg(spins=8, steps=200, seed=17, entropy_kind=0), 4),
])
def test_trajectories_match_reference(oracle, reflib, cfg, n):
    a = oracle.run(cfg, 0, n)
    b, _ = reflib.run(cfg, 0, n)
    assert np.array_equal(a.sites, b.sites)
    assert np.array_equal(a.accepted, b.accepted)
    assert np.array_equal(a.entropies.view(np.uint64), b.entropies.view(np.uint64))


def test_reference_driver_modes_agree(reflib):
    # bench.hpp:70-74: traces depend only on (seed, workload), not on the execution mode
    cfg = McCfg(spins=6, steps=30, seed=4)
    base, avg, _ = reflib.run_experiment(cfg, 4, 2, "cpu-reference")
    for mode in ("sequential", "tasked", "batched"):
        t, a2, _ = reflib.run_experiment(cfg, 4, 2, mode)
        assert np.array_equal(t.entropies.view(np.uint64), base.entropies.view(np.uint64))
        assert a2 == avg
