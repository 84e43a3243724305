"""Per-CTA clock breakdown of the HBM tier's work-queue schedule (tg_probe_queue_stats).

    python tools/queue_stats.py SPINS REPLICAS STEPS [renyi-2|von-neumann]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09353_b200 as tg  # noqa: E402

spins, reps, steps = (int(a) for a in sys.argv[1:4])
kind = 0 if len(sys.argv) > 4 and sys.argv[4] == "von-neumann" else 1
L = tg.lib()
buf = (C.c_int64 * (24 * 1024))()
ctas = C.c_int(0)
tg._check(L.tg_probe_queue_stats(spins, reps, steps, kind, buf, C.byref(ctas)))
s = np.frombuffer(buf, dtype=np.int64)[: 24 * ctas.value].reshape(ctas.value, 24).astype(np.float64)
names = ["total", "w1 wait stage", "w1 chunk compute", "w1 tile epilogue", "t0 wait stage (+issue)",
         "t0 top issue", "control items", "  dependency waits", "tiles", "DEC", "GATE", "INIT+NORM",
         "DEC clk", "GATE clk", "producer pulls clk", "  gate pass in DEC", "  DEC: wait + loads",
         "  DEC: fold + publish", "  DEC: decision", "  DEC: renorm + dec_done", "  DEC: final signal"]
tot = s[:, 0].mean()
print(f"S={spins} replicas={reps} steps={steps} ctas={ctas.value}: {tot:.4g} clk per CTA")
for i, n in enumerate(names[:21]):
    v = s[:, i]
    share = f"{100 * v.mean() / tot:6.2f} %" if i in (1, 2, 3, 4, 5, 6, 7, 12, 13, 15, 16, 17, 18, 19, 20) else ""
    print(f"  {n:24s} mean {v.mean():12.4g}  min {v.min():12.4g}  max {v.max():12.4g}  {share}")
nt = s[:, 8].sum()
if nt:
    print(f"  per tile: compute {s[:, 2].sum() / nt * 1:.4g} clk (warp 1, all chunks), "
          f"wait {s[:, 1].sum() / nt:.4g}, epilogue {s[:, 3].sum() / nt:.4g}")
