"""Randomised check of the batched GEMM's staging paths: for random shapes (m, k multiples
of 8 so the TMA kernel runs; n, batch, alpha, beta, C random), the TMA kernel with 8 and 16
warps and the cp.async kernel give bitwise-identical outputs, within 1e-12 of numpy.

    python tools/zgemm_fuzz.py [cases] [seed]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09353_b200 as tg  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 300
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
worst = 0.0
with tg.Device([0]) as dev:
    for c in range(n_cases):
        m = 8 * int(rng.integers(1, 40))
        k = 8 * int(rng.integers(1, 40))
        n = int(rng.integers(1, 300))
        batch = int(rng.integers(1, 9))
        al = complex(*rng.standard_normal(2))
        be = complex(*rng.standard_normal(2)) if rng.random() < 0.5 else 0.0
        As = [rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k)) for _ in range(batch)]
        Bs = [rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n)) for _ in range(batch)]
        Cs = [rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)) for _ in range(batch)] if be else None
        outs = {}
        for tag, env in (("cp.async", {"TG_ZGEMM_TMA": "0"}), ("tma8", {"TG_ZGEMM_TMA": "1", "TG_ZGEMM_WARPS": "8"}),
                         ("tma16", {"TG_ZGEMM_TMA": "1", "TG_ZGEMM_WARPS": "16"}), ("tma4", {"TG_ZGEMM_TMA": "1", "TG_ZGEMM_WARPS": "4"}), ("tma9", {"TG_ZGEMM_TMA": "1", "TG_ZGEMM_WARPS": "9"}),
                         ("tma5", {"TG_ZGEMM_TMA": "1", "TG_ZGEMM_WARPS": "5"})):
            os.environ.update(env)
            outs[tag] = [np.ascontiguousarray(o) for o in dev.batched_gemm(As, Bs, Cs, alpha=al, beta=be)]
        for tag in ("tma8", "tma16", "tma4", "tma9", "tma5"):
            for i in range(batch):
                if not np.array_equal(outs[tag][i].view(np.uint64), outs["cp.async"][i].view(np.uint64)):
                    raise SystemExit(f"case {c} ({m}x{n}x{k} x{batch}): {tag} differs from cp.async in entry {i}")
        for i in range(batch):
            want = al * (As[i] @ Bs[i]) + (be * Cs[i] if be else 0)
            err = np.abs(outs["tma16"][i] - want).max() / max(1.0, np.abs(want).max())
            worst = max(worst, err)
            if err > 1e-12:
                raise SystemExit(f"case {c} ({m}x{n}x{k}): error {err}")
print(f"{n_cases} random shapes: TMA (4, 4+producer, 8, 8+producer, 16 warps) bitwise equal to cp.async, max scaled error vs numpy {worst:.2e}")
