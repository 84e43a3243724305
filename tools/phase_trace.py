"""Per-phase cycle breakdown of the anneal kernel (CTA 0, first replica): the SMEM tier for
spins <= 12, the HBM tier above (TG_HBM_CTAS_PER_REPLICA picks its cluster size).

    python tools/phase_trace.py [spins] [replicas] [steps]

Stamps (clock64): 0 step start, 1 gate pass done, 2 GEMM done (partials posted),
3 decision done; HBM tier also: GEMM-internal chunk waits, tile epilogues, and the
largest per-warp wait (thread 0's view).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09353_b200 as tg  # noqa: E402

spins = int(sys.argv[1]) if len(sys.argv) > 1 else 12
replicas = int(sys.argv[2]) if len(sys.argv) > 2 else 148
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
t = tg.probe_phase_trace(spins, replicas, steps).astype(np.float64)
if steps < 14:
    raise SystemExit("need >= 14 steps")
s, nxt = t[10:-2], t[11:-1]
rows = {
    "step": nxt[:, 0] - s[:, 0],
    "gate pass (+ barrier)": s[:, 1] - s[:, 0],
    "GEMM (+ partials barrier)": s[:, 2] - s[:, 1],
    "decision (thread 0)": s[:, 3] - s[:, 2],
    "decision -> next step start": nxt[:, 0] - s[:, 3],
}
if spins >= 13:  # HBM tier: GEMM-internal clocks (thread 0)
    rows.update({
        "  GEMM: chunk waits + barriers": s[:, 4],
        "  GEMM: tile epilogues": s[:, 5],
        "  GEMM: max per-warp chunk waits": s[:, 6],
    })
print(f"S={spins} replicas={replicas} steps={steps}")
import signal
signal.signal(signal.SIGPIPE, signal.SIG_DFL)
for k, v in rows.items():
    print(f"  {k:32s} median {np.median(v):8.0f} clk   mean {np.mean(v):8.0f}")
