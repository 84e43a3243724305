"""Small HBM-tier anneal for profiling runs (ncu):
    python tools/prof_hbm_run.py SPINS PROCEDURES STEPS
    TG_HBM_QUEUE=1 ncu --set full --import-source on -k regex:anneal_queue -c 1 python tools/prof_hbm_run.py 20 64 2"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09353_b200 as tg  # noqa: E402

spins, procs, steps = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (20, 64, 2)))
cfg = tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=0)
with tg.Device([0]) as d:
    rep = d.run(cfg, sites=False)
print(f"S={spins} {procs}x{steps}: kernel {rep.kernel_ms:.3f} ms")
