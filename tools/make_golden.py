"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref/libtgref.so, built by
`make -C oracle ref` from /root/reference/proj/src). Run in the build container:

    python tools/make_golden.py             # everything
    python tools/make_golden.py vn_cfg1 ... # only the named trajectory cases

The fixtures pin the oracle restatement (oracle/oracle.c) and the device path on machines
where /root/reference does not exist (the GPU box). Config cases follow BASELINE.json
configs[0] and SURVEY.md Appendix A.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle_lib import McCfg, RefLib  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def main() -> None:
    os.makedirs(OUT, exist_ok=True)
    r = RefLib()
    only = set(sys.argv[1:])
    if not only:
        known_answers(r)
    trajectories(r, only)


def known_answers(r) -> None:
    rng = np.random.default_rng(20220317)

    # --- RNG / Haar / gate / entropy / gemm known answers --------------------------------
    pairs = [(s, p) for s in (0, 1, 42, 2**64 - 1) for p in (0, 1, 7, 65535)]
    u64 = np.stack([r.first_u64(s, p, 256) for s, p in pairs])
    normals = r.normal_pairs(7, 0, 256)
    haar = r.haar(7, 3, 64)
    gates = {}
    gi = 0
    sites_for = {12: (0, 5, 10), 13: (6,)}
    for spins in (2, 5, 8, 12, 13):
        for site in sites_for.get(spins, range(spins - 1)):
            psi = rng.standard_normal(1 << spins) + 1j * rng.standard_normal(1 << spins)
            psi /= np.linalg.norm(psi)
            u = r.haar(11, spins * 100 + site, 1)[0].view(np.complex128)
            gates[f"gate{gi}_meta"] = np.array([spins, site])
            gates[f"gate{gi}_in"] = psi
            gates[f"gate{gi}_u"] = u
            gates[f"gate{gi}_out"] = r.apply_gate(spins, psi, site, u)
            gi += 1
    ent_cases = {}
    for spins in (2, 3, 4, 6, 8, 9, 12, 13, 14):
        states = []
        for _ in range(4 if spins <= 12 else 1):
            psi = rng.standard_normal(1 << spins) + 1j * rng.standard_normal(1 << spins)
            psi /= np.linalg.norm(psi)
            states.append(psi)
        e2 = np.array([r.entropy(spins, s, 1) for s in states])
        evn = np.array([r.entropy(spins, s, 0) for s in states]) if spins <= 9 else np.zeros(0)
        ent_cases[f"ent_{spins}_states"] = np.stack(states)
        ent_cases[f"ent_{spins}_renyi2"] = e2
        ent_cases[f"ent_{spins}_vn"] = evn
    gemm = {}
    for i in range(40):
        m, n, k = (int(x) for x in rng.integers(1, 25, size=3))
        a = rng.standard_normal((m, k)) + 1j * rng.standard_normal((m, k))
        b = rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
        c = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        al = complex(*rng.standard_normal(2)) if i % 2 else 1.0 + 0j
        be = complex(*rng.standard_normal(2)) if i % 3 == 0 else 0j
        gemm[f"g{i}_a"], gemm[f"g{i}_b"], gemm[f"g{i}_c"] = a, b, c
        gemm[f"g{i}_ab"] = np.array([al, be])
        gemm[f"g{i}_out"] = r.gemm(al, a, b, be, c)
    np.savez_compressed(os.path.join(OUT, "kats.npz"), u64=u64, u64_pairs=np.array(pairs, dtype=np.uint64),
                        normals=normals, haar=haar, n_gates=gi, **gates, **ent_cases, **gemm)



def trajectories(r, only) -> None:
    # --- trajectories (mc_procedure through the reference's own pooled driver) -------------
    cases = {
        "cfg1": (McCfg(spins=8, steps=1000), 64),                       # BASELINE configs[0]
        "s12": (McCfg(spins=12, steps=200), 8),
        "s14": (McCfg(spins=14, steps=50), 8),
        "s16": (McCfg(spins=16, steps=10), 8),
        "rand_min_s7": (McCfg(spins=7, steps=300, initial_state=1, objective=1), 16),
        "rand_s13": (McCfg(spins=13, steps=20, initial_state=1), 4),
        "s5_renorm7": (McCfg(spins=5, steps=200, renormalize_interval=7), 8),
        "s2": (McCfg(spins=2, steps=100), 4),
        "s3": (McCfg(spins=3, steps=100), 4),
        "frozen_min_s6": (McCfg(spins=6, steps=60, objective=1, t0=1e-12, t_min=1e-12), 4),
        # von Neumann entropy (McConfig default, spinmc.hpp:116; SURVEY App. A second line)
        "vn_cfg1": (McCfg(spins=8, steps=1000, entropy_kind=0), 64),
        "vn_s12": (McCfg(spins=12, steps=120, entropy_kind=0), 4),
        "vn_rand_min_s10": (McCfg(spins=10, steps=200, entropy_kind=0, initial_state=1, objective=1), 4),
        "vn_s3": (McCfg(spins=3, steps=200, entropy_kind=0), 4),
        "vn_s5_renorm7": (McCfg(spins=5, steps=150, entropy_kind=0, renormalize_interval=7), 4),
        "vn_rand_s13": (McCfg(spins=13, steps=60, entropy_kind=0, initial_state=1), 3),  # HBM tier
    }
    for name, (cfg, n) in cases.items():
        if only and name not in only:
            continue
        tr, _ = r.run(cfg, 0, n)
        avg = 0.0
        for x in tr.entropies[:, -1]:  # procedure order, spinmc.cpp:259-268
            avg += float(x)
        avg /= n
        if name == "cfg1":  # the reference's own driver agrees (bench.cpp:401-407)
            _, avg_ref, _ = r.run_experiment(cfg, n)
            assert avg_ref == avg, (avg_ref, avg)
        np.savez_compressed(os.path.join(OUT, f"traj_{name}.npz"), spins=cfg.spins, steps=cfg.steps,
                            seed=cfg.seed, objective=cfg.objective, initial_state=cfg.initial_state,
                            t0=cfg.t0, t_min=cfg.t_min, renorm=cfg.renormalize_interval, procedures=n,
                            entropy_kind=cfg.entropy_kind,
                            initial=tr.initial, entropies=tr.entropies, accepted=tr.accepted, sites=tr.sites,
                            average=avg)
        print(name, "avg", repr(avg), "accepted", int(tr.accepted.sum()))


if __name__ == "__main__":
    main()
