// smem_tier.cuh — SMEM-resident tier (S <= 12): the replica's state psi and proposal
// psi' live in shared memory for the whole trajectory (HBM traffic per step ~ 0).
//
// Layout: each buffer is two planes (X = Re, Y = Im) of a column-major d_a x d_b
// matrix Psi[a][b] = psi[a + b*d_a] (spinmc.cpp:145-148).
//  * d_a >= 16 (S >= 8): dense column pitch d_a with an XOR swizzle of row bits 2-3,
//      phys(a, b) = b*d_a + (a ^ 4*((f(b) ^ (a >> 4)) & 3)),  f(b) = (b ^ b>>2 ^ b>>4) & 3.
//    phys is GF(2)-linear in the amplitude index (phys(i ^ j) = phys(i) ^ phys(j)), so an
//    address is one XOR of a per-lane constant and a per-chunk value. It keeps the GEMM
//    fragments (8 consecutive a x 4 consecutive b) and the DMMA gate's fragments
//    (tools/swizzle_check.py) bank-conflict free at every site, and needs no padding:
//    the S=12 buffers are 64 KB.
//  * d_a <= 8: pitch DA_PAD + 4 doubles (2*PITCH == 8 or 24 mod 32 words); rows >= d_a and
//    columns >= d_b are zero padding.
#pragma once
#include "../../include/taskgemm_b200.h"
#include "tg_device.cuh"

namespace tg {
namespace smem {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;

template <int LA, int LB>
struct Dims {
  static constexpr int DA = 1 << LA, DB = 1 << LB;
  static constexpr bool SWZ = LA >= 4;  // swizzled dense layout (else padded)
  static constexpr int DA_PAD = DA < 8 ? 8 : DA;
  static constexpr int DB_PAD = DB < 4 ? 4 : DB;
  static constexpr int PITCH = SWZ ? DA : DA_PAD + 4;
  static constexpr int PLANE = DB_PAD * PITCH;  // doubles per plane
  static constexpr int N = 1 << (LA + LB);
  static constexpr int NB = DA_PAD / 8;  // 8x8 blocks per rho dimension
  static constexpr int S = LA + LB;
  // Physical offset of amplitude idx (linear over GF(2) when SWZ).
  __host__ __device__ static constexpr int phys(int idx) {
    if constexpr (SWZ) {
      const int b = idx >> LA, a = idx & (DA - 1);
      return idx ^ ((((b ^ (b >> 2) ^ (b >> 4)) ^ (a >> 4)) & 3) << 2);
    } else {
      return (idx & (DA - 1)) + (idx >> LA) * PITCH;
    }
  }
  // Offset of Psi[a][b] (a < DA_PAD, b < DB_PAD; the padding rows/columns only when !SWZ).
  __host__ __device__ static constexpr int at(int a, int b) {
    if constexpr (SWZ) return phys(a | (b << LA));
    else return a + b * PITCH;
  }
};

// Warp tiling of the NB x NB block grid over the 8 GEMM warps.
template <int NB>
struct Tile {
  static constexpr int TM = NB >= 8 ? 2 : 1;
  static constexpr int TN = NB >= 8 ? 4 : (NB >= 4 ? 2 : 1);
  static constexpr int WR = NB / TM, WC = NB / TN;
  static_assert(WR * WC <= kConsumerWarps, "tiling");
};

// Gate application (spinmc.cpp:91-136) planar SMEM -> planar SMEM, fused form:
// re = fma(-ui, vi, fma(ur, vr, re)); im = fma(ui, vr, fma(ur, vi, im)) over the four inputs
// (in a lane-rotated order, below).
// Same sum as the reference (re += ur*vr - ui*vi) with fused rounding: 64 DFMA per group
// instead of 128 DMUL/DADD. On sm_100a DMMA and DFMA share the FP64 pipe, so the gate's
// op count is paid directly out of the GEMM's budget; the result differs from the
// reference's unfused rounding by ~1 ulp (parity is within tolerance).
template <class D, class R>  // R: anything with ur[16], ui[16] (GateRec)
__device__ __forceinline__ void gate_pass_fma(const double* __restrict__ sx,
                                              const double* __restrict__ sy,
                                              double* __restrict__ dx, double* __restrict__ dy,
                                              int site, const R& g, int tid, int nthreads) {
  // Bank-conflict-free order: for site <= 3 the 16 groups of a half-warp share few residues
  // mod 16 (site 0: bases 4*gi -> 4 banks, 4-way conflicts). Each lane walks its group's
  // four amplitudes in an order rotated by a lane constant r (r = (tid>>2)&3, or (tid>>3)&1
  // at site 3), which makes the 16 addresses of every load/store distinct mod 16. U is
  // permuted once (rows and columns by r), so the inner loop has no dynamic register index.
  // (nthreads is a multiple of 16, so r only depends on tid.)
  const int r = site <= 2 ? (tid >> 2) & 3 : (site == 3 ? (tid >> 3) & 1 : 0);
  double ur[16], ui[16];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int e = ((a + r) & 3) * 4 + ((b + r) & 3);
      ur[a * 4 + b] = g.ur[e];
      ui[a * 4 + b] = g.ui[e];
    }
  constexpr int GROUPS = D::N / 4;
  const int lo_mask = (1 << site) - 1;
  int off[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) off[t] = ((t + r) & 3) << site;
#pragma unroll 4
  for (int gi = tid; gi < GROUPS; gi += nthreads) {
    const int base = ((gi >> site) << (site + 2)) | (gi & lo_mask);
    int ph[4];
    double vr[4], vi[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      ph[t] = D::phys(base | off[t]);
      vr[t] = sx[ph[t]];
      vi[t] = sy[ph[t]];
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        re = fma(-ui[x * 4 + y], vi[y], fma(ur[x * 4 + y], vr[y], re));
        im = fma(ui[x * 4 + y], vr[y], fma(ur[x * 4 + y], vi[y], im));
      }
      dx[ph[x]] = re;
      dy[ph[x]] = im;
    }
  }
}

// Gate application in DMMA form (swizzled layout, S >= 8). The gate is the real 8x8 matrix
// [[Ur, -Ui], [Ui, Ur]] applied to 8 groups at a time: per chunk of 8 groups, two
// DMMA.8x8x4 (B = the groups' Re / Im amplitudes, k = amplitude y; D rows m < 4 = Re of
// output x = m, m >= 4 = Im of x = m - 4; D columns = groups). 2 LDS + 2 DMMA + 2 STS per
// lane per chunk instead of 8 LDS + 64 DFMA + 8 STS per group: the FP64 pipe cost is the
// same 64 FMA per group, at tensor-pipe issue cost. Same sum as the reference
// (re = sum_y ur*vr - ui*vi) with the tensor unit's rounding (within a few ulp, §4).
// Chunk c holds groups 8c + P(n), P a permutation of 0..7 chosen so that loads (lanes
// 0-15: columns 0-3) and stores (columns 0,2,4,6 / 1,3,5,7) are conflict free; with phys
// and the group -> amplitude deposit both linear, every address is cb ^ lane constant.
__device__ __forceinline__ int deposit(int g, int site) {  // spinmc.cpp:118-121 base index
  return ((g >> site) << (site + 2)) | (g & ((1 << site) - 1));
}
// Per-lane constants of the DMMA gate for one record: the A fragments and the lane's
// load / store offsets (relative to a chunk's base, combined by XOR).
struct GateLane {
  double a1, a2;
  int kload, kst0, kst1, site;
  bool re;  // this lane's D row is a real part (stores go to the X plane)
  // speculative gate (rho_partials SPEC): chunk warp + 8i has base cbw ^ tab[i]
  // (phys and the deposit are linear), tab = the CTA's table for this site
  int cbw;
  const int* tab;
};
template <class D, class R>
__device__ __forceinline__ GateLane gate_lane(const R& g, int site, int lane) {
  GateLane L;
  const int ml = lane >> 2, kl = lane & 3, x = ml & 3;
  L.a1 = ml < 4 ? g.ur[x * 4 + kl] : g.ui[x * 4 + kl];
  L.a2 = ml < 4 ? -g.ui[x * 4 + kl] : g.ur[x * 4 + kl];
  auto P = [site](int n) { return site == 0 ? n : ((n & 4) | ((n ^ (n >> 2)) & 3)); };
  L.kload = D::phys(deposit(P(ml), site) | (kl << site));
  L.kst0 = D::phys(deposit(P(2 * kl), site) | (x << site));
  L.kst1 = D::phys(deposit(P(2 * kl + 1), site) | (x << site));
  L.site = site;
  L.re = ml < 4;
  return L;
}
// One chunk (8 groups, c = chunk index): 2 LDS + 2 DMMA + 2 STS per lane.
template <class D>
__device__ __forceinline__ void gate_chunk(const GateLane& L, const double* __restrict__ sx,
                                           const double* __restrict__ sy, double* __restrict__ dst,
                                           int c) {
  const int cb = D::phys(deposit(8 * c, L.site));
  const double vr = sx[cb ^ L.kload], vi = sy[cb ^ L.kload];
  double d0 = 0.0, d1 = 0.0;
  dmma(d0, d1, L.a1, vr);
  dmma(d0, d1, L.a2, vi);
  dst[cb ^ L.kst0] = d0;
  dst[cb ^ L.kst1] = d1;
}
template <class D, class R>
__device__ __forceinline__ void gate_pass_dmma(const double* __restrict__ sx,
                                               const double* __restrict__ sy,
                                               double* __restrict__ dx, double* __restrict__ dy,
                                               int site, const R& g, int warp, int lane) {
  static_assert(D::SWZ && D::N >= 256, "DMMA gate needs the swizzled layout");
  const GateLane L = gate_lane<D>(g, site, lane);
  double* __restrict__ dst = L.re ? dx : dy;
  // A warp takes chunks warp, warp + 8, ... in batches of B: all loads of a batch, then its
  // 2B DMMAs (B independent chains), then its stores — the loads of a batch never wait
  // behind stores that might alias, and the DMMA latency (26 clk) overlaps across chunks.
  constexpr int CH = D::N / 32;
  constexpr int PER = CH / kConsumerWarps;  // chunks per warp (>= 1 for S >= 8)
  constexpr int B = PER < 4 ? PER : 4;
#pragma unroll 1
  for (int c0 = warp; c0 < CH; c0 += kConsumerWarps * B) {
    int cb[B];
    double vr[B], vi[B], d0[B], d1[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      cb[b] = D::phys(deposit(8 * (c0 + b * kConsumerWarps), L.site));
      vr[b] = sx[cb[b] ^ L.kload];
      vi[b] = sy[cb[b] ^ L.kload];
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      d0[b] = 0.0;
      d1[b] = 0.0;
      dmma(d0[b], d1[b], L.a1, vr[b]);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) dmma(d0[b], d1[b], L.a2, vi[b]);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      dst[cb[b] ^ L.kst0] = d0[b];
      dst[cb[b] ^ L.kst1] = d1[b];
    }
  }
}

// The tier's gate: DMMA form on the swizzled layout, fused DFMA form otherwise.
template <class D, class R>
__device__ __forceinline__ void gate_pass(const double* __restrict__ sx, const double* __restrict__ sy,
                                          double* __restrict__ dx, double* __restrict__ dy, int site,
                                          const R& g, int tid, int nthreads) {
  if constexpr (D::SWZ) gate_pass_dmma<D>(sx, sy, dx, dy, site, g, tid >> 5, tid & 31);
  else gate_pass_fma<D>(sx, sy, dx, dy, site, g, tid, nthreads);
}

// Per-warp sum |rho_ij|^2 and trace(rho) of rho = Psi Psi^dagger (warp-reduced; valid in
// every lane). inject_fault flips the sign of the first accumulation term of rho(0,0)
// (linalg.cpp:94 testhook) AFTER the trace is taken, so only the entropy is corrupted.
// STORE (von Neumann): rho is also written to planar SMEM Rr/Ri (column-major, pitch RP).
// SPEC (swizzled layout; a compile-time switch so the gate stages schedule freely with the
// GEMM's loads and DMMAs): the warps also apply the NEXT step's gate to this Psi (the
// speculative proposal for "accepted", written to gdst = X or Y plane of a third buffer by
// lane), one 8-group chunk interleaved after every RATIO-th k-step of the GEMM, so its
// DMMAs and SMEM traffic share the GEMM's pipeline instead of a separate phase. It is the
// same DMMA computation as gate_pass_dmma: bitwise the non-speculative proposal.
// HALF (opt-in rho_half, Renyi-2): only the upper-triangle 8x8 blocks (bi <= bj) of the
// Hermitian rho are formed, upper block u on warp u mod 8; ||rho||_F^2 = diagonal blocks +
// 2 x off-diagonal blocks (the doubling is exact). Trace, fault hook and the speculative gate
// stages are unchanged.
template <class D, bool STORE = false, bool SPEC = false, bool HALF = false>
__device__ __forceinline__ void rho_partials(const double* __restrict__ X,
                                             const double* __restrict__ Y, int warp, int lane,
                                             bool fault, double& rho2, double& trace,
                                             double* Rr = nullptr, double* Ri = nullptr,
                                             int RP = 0, const GateLane* SL = nullptr,
                                             double* __restrict__ gdst = nullptr) {
  using T = Tile<D::NB>;
  static_assert(!(HALF && STORE), "rho_half is a Renyi-2 option");
  rho2 = 0.0;
  trace = 0.0;
  constexpr int GPW = D::N / 32 / kConsumerWarps;        // gate chunks per warp
  constexpr int KI = D::DB_PAD / 4;                      // GEMM k-steps
  constexpr int RATIO = GPW > 0 && KI >= GPW ? KI / GPW : 1;
  static_assert(!SPEC || (D::SWZ && GPW >= 1 && KI % GPW == 0), "speculative gate layout");
  constexpr int NU = D::NB * (D::NB + 1) / 2;  // HALF: upper-triangle blocks
  constexpr int GEMM_WARPS = HALF ? (NU < kConsumerWarps ? NU : kConsumerWarps) : T::WR * T::WC;
  if (SPEC && warp >= GEMM_WARPS) {  // warps without a GEMM tile (S < 10)
#pragma unroll 1
    for (int i = 0; i < GPW; ++i) gate_chunk<D>(*SL, X, Y, gdst, warp + kConsumerWarps * i);
  }
  // Speculative gate, software-pipelined over the k-steps: chunk j is loaded at k-step
  // j*RATIO, its two DMMAs issue one and two k-steps later and it is stored three k-steps
  // later; a stage runs at the top of its k-step, ahead of the GEMM's loads and DMMAs, so
  // no instruction waits on a gate result (DMMA latency 26 clk) and the warp's GEMM issue
  // never stalls behind the gate.
  int g_cb = 0, h_cb = 0, r_cb = 0;
  double g_vr = 0.0, g_vi = 0.0, h_vi = 0.0, h_d0 = 0.0, h_d1 = 0.0, r_d0 = 0.0, r_d1 = 0.0;
  auto at_chunk = [&](int it, int lag) { return it >= lag && (it - lag) % RATIO == 0 && (it - lag) / RATIO < GPW; };
  auto spec_stage = [&](int it) {
    if (at_chunk(it, 3)) {  // store chunk (it-3)/RATIO
      gdst[r_cb ^ SL->kst0] = r_d0;
      gdst[r_cb ^ SL->kst1] = r_d1;
    }
    if (at_chunk(it, 2)) {  // second DMMA (Im inputs)
      dmma(h_d0, h_d1, SL->a2, h_vi);
      r_d0 = h_d0;
      r_d1 = h_d1;
      r_cb = h_cb;
    }
    if (at_chunk(it, 1)) {  // first DMMA (Re inputs)
      h_d0 = 0.0;
      h_d1 = 0.0;
      dmma(h_d0, h_d1, SL->a1, g_vr);
      h_vi = g_vi;
      h_cb = g_cb;
    }
    if (at_chunk(it, 0)) {  // loads
      g_cb = SL->cbw ^ SL->tab[it / RATIO];
      g_vr = X[g_cb ^ SL->kload];
      g_vi = Y[g_cb ^ SL->kload];
    }
  };
  if constexpr (HALF) {
    if (warp < GEMM_WARPS) {
      constexpr int MAXB = (NU + kConsumerWarps - 1) / kConsumerWarps;
      constexpr int NV = D::SWZ ? 4 : 1;
      const int m = lane >> 2, kq = lane & 3;
      int bi[MAXB], bj[MAXB];
      bool on[MAXB];
      int roa[MAXB][NV], rob[MAXB][NV];
#pragma unroll
      for (int b = 0; b < MAXB; ++b) {
        int u = warp + kConsumerWarps * b;
        on[b] = u < NU;
        int r = 0;
        while (on[b] && u >= D::NB - r) {  // upper block u, row-major
          u -= D::NB - r;
          ++r;
        }
        bi[b] = on[b] ? r : 0;
        bj[b] = on[b] ? r + u : 0;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int c = D::SWZ ? 4 * v : 0;
          roa[b][v] = D::at(bi[b] * 8 + m, kq + c) - c * D::PITCH;
          rob[b][v] = D::at(bj[b] * 8 + m, kq + c) - c * D::PITCH;
        }
      }
      double cr[MAXB][2], ci[MAXB][2];
#pragma unroll
      for (int b = 0; b < MAXB; ++b) cr[b][0] = cr[b][1] = ci[b][0] = ci[b][1] = 0.0;
#pragma unroll
      for (int kb = 0; kb < D::DB_PAD; kb += 4) {
        if constexpr (SPEC) spec_stage(kb / 4);
        const int v = D::SWZ ? (((kb >> 2) ^ (kb >> 4)) & 3) : 0;
        const int ko = kb * D::PITCH;
#pragma unroll
        for (int b = 0; b < MAXB; ++b) {
          if (!on[b]) continue;
          const double xa = X[roa[b][v] + ko], ya = Y[roa[b][v] + ko];
          const double xb = X[rob[b][v] + ko], yb = Y[rob[b][v] + ko];
          dmma(cr[b][0], cr[b][1], xa, xb);
          dmma(cr[b][0], cr[b][1], ya, yb);
          dmma(ci[b][0], ci[b][1], ya, xb);
          dmma(ci[b][0], ci[b][1], -xa, yb);
        }
      }
      if constexpr (SPEC) {
        spec_stage(KI);
        spec_stage(KI + 1);
        spec_stage(KI + 2);
      }
#pragma unroll
      for (int b = 0; b < MAXB; ++b)
        if (on[b] && bi[b] == bj[b]) {
          if (m == 2 * kq) trace += cr[b][0];
          if (m == 2 * kq + 1) trace += cr[b][1];
        }
      if (fault && warp == 0 && lane == 0) cr[0][0] -= 2.0 * (X[0] * X[0] + Y[0] * Y[0]);  // block (0,0)
      double pd[4] = {0.0, 0.0, 0.0, 0.0}, po[4] = {0.0, 0.0, 0.0, 0.0};  // diagonal / off-diagonal chains
#pragma unroll
      for (int b = 0; b < MAXB; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (!on[b]) continue;
          double& a = bi[b] == bj[b] ? pd[(b * 2 + e) & 3] : po[(b * 2 + e) & 3];
          a = fma(cr[b][e], cr[b][e], a);
          a = fma(ci[b][e], ci[b][e], a);
        }
      const double off = (po[0] + po[1]) + (po[2] + po[3]);
      rho2 = ((pd[0] + pd[1]) + (pd[2] + pd[3])) + (off + off);
    }
  } else if (warp < T::WR * T::WC) {
    const int wr = warp / T::WC, wc = warp % T::WC;
    const int m = lane >> 2, kq = lane & 3;
    double cr[T::TM][T::TN][2], ci[T::TM][T::TN][2];
#pragma unroll
    for (int i = 0; i < T::TM; ++i)
#pragma unroll
      for (int j = 0; j < T::TN; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
    // Fragment offsets: at(row, kb + kq) = kb * PITCH + ro[f(kb)] with f(kb) in 0..3 (the
    // swizzle term of column kb + kq, kb a multiple of 4), so each load is a per-lane base
    // register plus an immediate.
    constexpr int NV = D::SWZ ? 4 : 1;
    int roa[T::TM][NV], rob[T::TN][NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int c = D::SWZ ? 4 * v : 0;  // a column with f(c) = v
#pragma unroll
      for (int i = 0; i < T::TM; ++i) roa[i][v] = D::at((wr * T::TM + i) * 8 + m, kq + c) - c * D::PITCH;
#pragma unroll
      for (int j = 0; j < T::TN; ++j) rob[j][v] = D::at((wc * T::TN + j) * 8 + m, kq + c) - c * D::PITCH;
    }
#pragma unroll
    for (int kb = 0; kb < D::DB_PAD; kb += 4) {
      if constexpr (SPEC) spec_stage(kb / 4);
      const int v = D::SWZ ? (((kb >> 2) ^ (kb >> 4)) & 3) : 0;
      const int ko = kb * D::PITCH;
      double xa[T::TM], ya[T::TM], xn[T::TM], xb[T::TN], yb[T::TN];
#pragma unroll
      for (int i = 0; i < T::TM; ++i) {
        xa[i] = X[roa[i][v] + ko];
        ya[i] = Y[roa[i][v] + ko];
        xn[i] = -xa[i];
      }
#pragma unroll
      for (int j = 0; j < T::TN; ++j) {
        xb[j] = X[rob[j][v] + ko];
        yb[j] = Y[rob[j][v] + ko];
      }
#pragma unroll
      for (int i = 0; i < T::TM; ++i)
#pragma unroll
        for (int j = 0; j < T::TN; ++j) {
          dmma(cr[i][j][0], cr[i][j][1], xa[i], xb[j]);
          dmma(cr[i][j][0], cr[i][j][1], ya[i], yb[j]);
          dmma(ci[i][j][0], ci[i][j][1], ya[i], xb[j]);
          dmma(ci[i][j][0], ci[i][j][1], xn[i], yb[j]);
        }
    }
    if constexpr (SPEC) {
      spec_stage(KI);
      spec_stage(KI + 1);
      spec_stage(KI + 2);
    }
#pragma unroll
    for (int i = 0; i < T::TM; ++i)
#pragma unroll
      for (int j = 0; j < T::TN; ++j)
        if (wr * T::TM + i == wc * T::TN + j) {
          if (m == 2 * kq) trace += cr[i][j][0];
          if (m == 2 * kq + 1) trace += cr[i][j][1];
        }
    if (fault && wr == 0 && wc == 0 && lane == 0)
      cr[0][0][0] -= 2.0 * (X[0] * X[0] + Y[0] * Y[0]);
    double part[4] = {0.0, 0.0, 0.0, 0.0};  // four chains: the fold is not one 32-deep DFMA chain
#pragma unroll
    for (int i = 0; i < T::TM; ++i)
#pragma unroll
      for (int j = 0; j < T::TN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double& a = part[((i * T::TN + j) * 2 + e) & 3];
          a = fma(cr[i][j][e], cr[i][j][e], a);
          a = fma(ci[i][j][e], ci[i][j][e], a);
          if constexpr (STORE) {
            const int o = (wr * T::TM + i) * 8 + m + ((wc * T::TN + j) * 8 + 2 * kq + e) * RP;
            Rr[o] = cr[i][j][e];
            Ri[o] = ci[i][j][e];
          }
        }
    rho2 = (part[0] + part[1]) + (part[2] + part[3]);
  }
  rho2 = warp_sum(rho2);
  trace = warp_sum(trace);
}

// Renyi-2 finalisation (spinmc.cpp:171-175): f = sqrt(sum); e = -log(f*f); max(e, 0)
// keeping -0.0 exactly as std::max does.
__device__ __forceinline__ double renyi2(double rho2) {
  const double f = __dsqrt_rn(rho2);
  const double e = -log(__dmul_rn(f, f));
  return (e < 0.0) ? 0.0 : e;
}

// Metropolis decision of spinmc.cpp:201-207 on rho2 = ||rho||_F^2 (entropy = -log rho2,
// clamped at 0 <=> rho2 clamped at 1): accept <=> u < exp(clamp(delta/T))
// <=> delta > T log u <=> rho2' < rho2_cur * exp(-T log u) (maximize) or
// rho2' > rho2_cur * exp(T log u) (minimize); emul is that factor. Relative margins below
// 1e-12 are re-decided with the reference formula (entropies and exp), so the outcome is
// the reference's wherever FP64 rounding cannot tie.
// The window is the record's tie_tol (>= 1e-12, gate_stream.cu make_gate): wide enough that
// every decision with |u - p| < 1e-9 takes the reference formula and can be audited.
// Verdict.flags: bit 0 = re-decided with the reference formula, bit 1 = near tie
// (|u - p| < 1e-9); p is valid when flags != 0.
struct Verdict {
  int acc;
  int flags;
  double p;
};
// The part of the decision that does not depend on the new rho2 (the bound and the tie
// window), so a caller can form it before the partials barrier.
struct DecPre {
  double bound, tol;
};
template <class R>
__device__ __forceinline__ DecPre decide_prep(double rho2_cur, const R& g) {
  return {fmin(rho2_cur, 1.0) * g.emul, static_cast<double>(g.tie_tol)};
}
template <class R>
__device__ __forceinline__ Verdict decide_audit(double rho2_new, double rho2_cur, const DecPre& d, const R& g,
                                                int objective, double eps = 1e-9) {
  const double r_new = fmin(rho2_new, 1.0);
  if (fabs(r_new - d.bound) > d.tol * r_new)
    return {objective == 0 ? (r_new < d.bound) : (r_new > d.bound), 0, 0.0};
  const double proposed = renyi2(rho2_new), current = renyi2(rho2_cur);
  const double delta = objective == 0 ? proposed - current : current - proposed;
  const double p = acceptance(delta, g.temp);
  return {g.u < p, 1 | (fabs(g.u - p) < eps ? 2 : 0), p};
}
template <class R>
__device__ __forceinline__ Verdict decide_audit(double rho2_new, double rho2_cur, const R& g, int objective,
                                                double eps = 1e-9) {
  return decide_audit(rho2_new, rho2_cur, decide_prep(rho2_cur, g), g, objective, eps);
}
template <class R>
__device__ __forceinline__ int decide(double rho2_new, double rho2_cur, const R& g, int objective) {
  return decide_audit(rho2_new, rho2_cur, g, objective).acc;
}
// spinmc.cpp:201-207 verbatim on entropies (von Neumann), with the near-tie flag.
template <class R>
__device__ __forceinline__ Verdict decide_reference(double proposed, double current, const R& g, int objective,
                                                    double eps = 1e-9) {
  const double delta = objective == 0 ? proposed - current : current - proposed;
  const double p = acceptance(delta, g.temp);
  return {g.u < p, fabs(g.u - p) < eps ? 2 : 0, p};
}
// Decision audit record (one thread): counts and logs (tg_anneal_device_buffers tie_*).
template <class PP, class R>
__device__ __forceinline__ void audit(const PP& P, uint64_t r, uint64_t s, const R& g, const Verdict& v) {
  if (!v.flags || !P.tie_stats) return;
  if (v.flags & 1) atomicAdd(&P.tie_stats[0], 1ull);
  if (v.flags & 2) {
    const unsigned long long i = atomicAdd(&P.tie_stats[1], 1ull);
    if (P.tie_log && i < P.tie_capacity) {
      tg_near_tie& t = P.tie_log[i];
      t.procedure = P.p_first + r * P.p_stride;
      t.step = s;
      t.u = g.u;
      t.p = v.p;
      t.site = static_cast<uint32_t>(g.site);
      t.accepted = v.acc;
    }
  }
}

// Norm check of spinmc.cpp:152-156 on trace(rho) = ||psi'||^2.
__device__ __forceinline__ bool not_normalized(double trace) {
  return fabs(__dsqrt_rn(trace) - 1.0) > 1e-9;
}

}  // namespace smem
}  // namespace tg
