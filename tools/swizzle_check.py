"""Bank-conflict check of the SMEM-tier state layout (csrc/smem_tier.cuh, Dims::phys).

    python tools/swizzle_check.py

Models 64-bit shared-memory accesses as two half-warp wavefront groups (16 lanes, 16
eight-byte bank pairs each); prints the wavefronts per warp access (ideal 2) of
  * the GEMM fragment loads (8 consecutive rows a x 4 consecutive columns b), and
  * the DMMA-form gate's loads and stores at every site,
for the padded layout (pitch d_a + 4) and the swizzled one, S = 8..12.
"""


def make(LA, LB, mode):
    DA = 1 << LA

    def f(b):
        return (b ^ (b >> 2) ^ (b >> 4)) & 3

    def phys(idx):
        a, b = idx & (DA - 1), idx >> LA
        if mode == "pad":
            return a + b * (DA + 4)
        return b * DA + (a ^ (4 * ((f(b) ^ (a >> 4)) & 3)))
    return phys


def wavefronts(addrs):
    tot = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for ad in set(half):
            banks[ad % 16] = banks.get(ad % 16, 0) + 1
        tot += max(banks.values())
    return tot


def deposit(g, site):
    return ((g >> site) << (site + 2)) | (g & ((1 << site) - 1))


def perm(n, site):
    return n if site == 0 else (n & 4) | ((n ^ (n >> 2)) & 3)


def check(LA, LB, mode):
    phys, N, DA = make(LA, LB, mode), 1 << (LA + LB), 1 << LA
    assert len({phys(i) for i in range(N)}) == N
    gemm = max(wavefronts([phys(blk * 8 + (l >> 2) + ((kb + (l & 3)) << LA)) for l in range(32)])
               for blk in range(DA // 8) for kb in range(0, 1 << LB, 4))
    sites = {}
    for site in range(LA + LB - 1):
        wl = ws = 0
        for c in range(N // 32):
            gs = [8 * c + perm(n, site) for n in range(8)]
            wl = max(wl, wavefronts([phys(deposit(gs[l >> 2], site) | ((l & 3) << site)) for l in range(32)]))
            for e in range(2):
                ws = max(ws, wavefronts([phys(deposit(gs[2 * (l & 3) + e], site) | (((l >> 2) & 3) << site))
                                         for l in range(32)]))
        sites[site] = (wl, ws)
    return gemm, sites


if __name__ == "__main__":
    for S in range(8, 13):
        for mode in ("pad", "swz"):
            g, s = check(S // 2, S - S // 2, mode)
            print(f"S={S:2d} {mode}: gemm {g}  gate (load, store) per site {s}")
