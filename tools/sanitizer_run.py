"""Small anneals of every kernel family, for compute-sanitizer (tests/test_sanitizer.py):
SMEM tier S = 12 (speculative) and S = 8, HBM tier S = 14 on the cluster schedule and on the
work queue (Renyi-2, rho_half, von Neumann S = 16 with the global-memory eigen-solver), von
Neumann S = 13 (HBM tier) and S = 10 (SMEM tier); the batched GEMM's kernel variants."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_09353_b200 as tg  # noqa: E402

with tg.Device([0]) as d:
    for spins, steps, procs, kind in ((12, 12, 2, "renyi-2"), (8, 10, 2, "renyi-2"), (14, 4, 1, "renyi-2"),
                                      (13, 3, 1, "von-neumann"), (10, 3, 1, "von-neumann")):
        r = d.run(tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=1, entropy_kind=kind))
        print(spins, kind, int(r.accepted.sum()))
    # the HBM tier's work queue: Renyi-2 (random start: NORM items, renormalisation in DEC items),
    # rho_half, and von Neumann above S = 15
    os.environ["TG_HBM_QUEUE"] = "1"
    for spins, steps, procs, kind, half in ((14, 8, 3, "renyi-2", False), (14, 4, 2, "renyi-2", True),
                                            (16, 1, 1, "von-neumann", False)):
        r = d.run(tg.ExperimentConfig(spins=spins, steps=steps, procedures=procs, seed=1, entropy_kind=kind,
                                      initial_state="random", renormalize_interval=3, rho_half=half))
        print("queue", spins, kind, half, int(r.accepted.sum()))
    del os.environ["TG_HBM_QUEUE"]

# the batched-GEMM kernel, with ragged edges (zero-filled copies) and a C operand
import numpy as np  # noqa: E402

rng = np.random.default_rng(0)
with tg.Device([0]) as d:
    for m, n, k, nb in ((70, 33, 45, 3), (64, 64, 64, 2), (5, 130, 7, 2), (96, 96, 96, 2), (64, 64, 256, 1)):
        A = [rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k)) for _ in range(nb)]
        B = [rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n)) for _ in range(nb)]
        Cm = [rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n)) for _ in range(nb)]
        for w in ("4", "5", "9", "16"):  # the TMA variants (m, k multiples of 8) and the cp.async kernel
            os.environ["TG_ZGEMM_WARPS"] = w
            out = d.batched_gemm(A, B, Cm, alpha=0.5 - 1j, beta=2.0)
            err = max(np.abs(o - ((0.5 - 1j) * a @ b + 2.0 * c)).max() for o, a, b, c in zip(out, A, B, Cm))
            print("zgemm", w, m, n, k, nb, f"{err:.1e}")
            assert err < 1e-9
        os.environ.pop("TG_ZGEMM_WARPS", None)
