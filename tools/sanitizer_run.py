"""Small anneals of every kernel family, for compute-sanitizer (tests/test_sanitizer.py):
SMEM tier S = 12 (speculative) and S = 8, HBM tier S = 14, von Neumann S = 13 (HBM tier)
and S = 10 (SMEM tier)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09353_b200 as tg  # noqa: E402

with tg.Device([0]) as d:
    for spins, steps, procs, kind in ((12, 12, 2, "renyi-2"), (8, 10, 2, "renyi-2"), (14, 4, 1, "renyi-2"),
                                      (13, 3, 1, "von-neumann"), (10, 3, 1, "von-neumann")):
        r = d.run(tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=1, entropy_kind=kind))
        print(spins, kind, int(r.accepted.sum()))
