"""Config-5 comparators (integration/comparators.cpp): the paper's ranks-per-GPU tasked
scheme and the lock-step batchedGEMM scheme, cuBLAS ZGEMM on the GPU, host code from the
reference. Their traces must equal the oracle's (flags bit-exact, entropies within 1e-10
relative: cuBLAS rounds the GEMM differently from linalg::gemm), otherwise the timing
comparison is between different computations."""
import os
import sys

import numpy as np
import pytest
from oracle_lib import McCfg, Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "integration"))
from comparators import SO, Comparators  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cmp():
    if not os.path.exists(SO):
        pytest.skip("integration/libtgc.so not built (needs the reference headers at build time)")
    return Comparators()


def _check(out, spins, steps, replicas, seed):
    o = Oracle()
    for p in range(replicas):
        init, ent, acc, _, _, _ = o.mc_procedure(McCfg(spins=spins, steps=steps, seed=seed), p)
        assert abs(out["initial"][p] - init) <= 1e-10 * max(abs(init), 1.0)
        assert np.array_equal(out["accepted"][p], acc), f"replica {p}"
        assert (np.abs(out["entropies"][p] - ent) <= 1e-10 * np.maximum(np.abs(ent), 1.0)).all()


@pytest.mark.parametrize("spins", [8, 11])
def test_tasked_matches_oracle(cmp, spins):
    out = cmp.tasked(spins, 150, 6, seed=3, ranks=4)
    _check(out, spins, 150, 6, 3)
    assert out["wall_s"] > 0


@pytest.mark.parametrize("spins", [8, 11])
def test_batched_matches_oracle(cmp, spins):
    out = cmp.batched(spins, 150, 6, seed=3)
    _check(out, spins, 150, 6, 3)
    assert out["wall_s"] > 0
