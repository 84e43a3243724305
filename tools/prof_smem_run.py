"""Small config-2-shaped anneal for profiling runs (ncu): S=12, 148 replicas, 300 steps.
    ncu --set full --import-source on -k regex:anneal_smem_kernel -c 1 python tools/prof_smem_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09353_b200 as tg  # noqa: E402

spins = int(sys.argv[1]) if len(sys.argv) > 1 else 12
cfg = tg.ExperimentConfig(spins=spins, steps=300, procedures=148, seed=0)
with tg.Device([0]) as d:
    d.run(cfg, sites=False)
