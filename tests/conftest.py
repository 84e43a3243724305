"""Test configuration. `-m gpu` tests need a B200 (run through gpurun); everything else runs on CPU.

GPU tests never skip because the CUDA library is missing: a missing/unloadable
libtaskgemm_b200.so is a failure, so a silent CPU fallback cannot pass them.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle_lib import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from oracle_lib import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefLib()


@pytest.fixture(scope="session")
def kats():
    return np.load(os.path.join(GOLDEN, "kats.npz"))


def load_traj(name):
    return np.load(os.path.join(GOLDEN, f"traj_{name}.npz"))


TRAJ_CASES = ["cfg1", "s12", "s14", "s16", "rand_min_s7", "rand_s13", "s5_renorm7", "s2", "s3", "frozen_min_s6"]
VN_CASES = ["vn_cfg1", "vn_s12", "vn_rand_min_s10", "vn_s3", "vn_s5_renorm7", "vn_rand_s13"]  # von Neumann entropy


def entropy_kind_of(g) -> int:
    """0 von Neumann, 1 Renyi-2 (fixtures without the key are Renyi-2)."""
    return int(g["entropy_kind"]) if "entropy_kind" in g.files else 1


@pytest.fixture(scope="session")
def device():
    """A device context; on a GPU box a load/create failure FAILS the test (no fallback)."""
    import paper_2203_09353_b200 as tg
    dev = tg.Device([0])
    yield dev
    dev.close()


def cfg_from_golden(g, procedures=None):
    """The device ExperimentConfig of a golden trajectory fixture."""
    import paper_2203_09353_b200 as tg
    return tg.ExperimentConfig(
        spins=int(g["spins"]), steps=int(g["steps"]), procedures=procedures or int(g["procedures"]),
        seed=int(g["seed"]), objective="max" if int(g["objective"]) == 0 else "min",
        initial_state="product" if int(g["initial_state"]) == 0 else "random",
        t0=float(g["t0"]), t_min=float(g["t_min"]), renormalize_interval=int(g["renorm"]),
        entropy_kind="renyi-2" if entropy_kind_of(g) == 1 else "von-neumann")
