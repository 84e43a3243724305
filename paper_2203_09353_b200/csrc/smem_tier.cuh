// smem_tier.cuh — SMEM-resident tier (S <= 12): the replica's state psi and proposal
// psi' live in shared memory for the whole trajectory (HBM traffic per step ~ 0).
//
// Layout: each buffer is two planes (X = Re, Y = Im) of a column-major d_a x d_b
// matrix Psi[a][b] = psi[a + b*d_a] (spinmc.cpp:145-148), stored with pitch
// PITCH = DA_PAD + 4 doubles per column b. 2*PITCH == 8 or 24 (mod 32) words, so the
// DMMA fragment pattern (8 consecutive a x 4 consecutive b per warp) is bank-conflict
// free. Rows >= d_a and columns >= d_b (S < 6) are zero padding.
//
// rho = Psi Psi^dagger by real split:
//   Re rho = X X^T + Y Y^T,  Im rho = Y X^T - X Y^T,
// four DMMA.8x8x4 per 8x8 complex block and k-chunk of 4 (2048 flop = 8*8*8*4). rho
// never leaves registers: the epilogue reduces sum |rho_ij|^2 (Renyi-2) and trace(rho)
// (= ||psi'||^2, the norm check of spinmc.cpp:152-156) per warp, fixed order.
#pragma once
#include "tg_device.cuh"

namespace tg {
namespace smem {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;

template <int LA, int LB>
struct Dims {
  static constexpr int DA = 1 << LA, DB = 1 << LB;
  static constexpr int DA_PAD = DA < 8 ? 8 : DA;
  static constexpr int DB_PAD = DB < 4 ? 4 : DB;
  static constexpr int PITCH = DA_PAD + 4;
  static constexpr int PLANE = DB_PAD * PITCH;  // doubles per plane
  static constexpr int N = 1 << (LA + LB);
  static constexpr int NB = DA_PAD / 8;  // 8x8 blocks per rho dimension
  static constexpr int S = LA + LB;
  __device__ static __forceinline__ int phys(int idx) {
    return (idx & (DA - 1)) + (idx >> LA) * PITCH;
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

struct Header {  // HBM tier CTA scratch
  double part_rho[kConsumerWarps];
  double part_tr[kConsumerWarps];
  int32_t decision;
  int32_t error;
};
constexpr int kHeaderBytes = (static_cast<int>(sizeof(Header)) + 127) / 128 * 128;

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

// Per-warp sum |rho_ij|^2 and trace(rho) of rho = Psi Psi^dagger (warp-reduced; valid in
// every lane). inject_fault flips the sign of the first accumulation term of rho(0,0)
// (linalg.cpp:94 testhook) AFTER the trace is taken, so only the entropy is corrupted.
// STORE (von Neumann): rho is also written to planar SMEM Rr/Ri (column-major, pitch RP).
template <class D, bool STORE = false>
__device__ __forceinline__ void rho_partials(const double* __restrict__ X,
                                             const double* __restrict__ Y, int warp, int lane,
                                             bool fault, double& rho2, double& trace,
                                             double* Rr = nullptr, double* Ri = nullptr,
                                             int RP = 0) {
  using T = Tile<D::NB>;
  rho2 = 0.0;
  trace = 0.0;
  if (warp < T::WR * T::WC) {
    const int wr = warp / T::WC, wc = warp % T::WC;
    const int m = lane >> 2, kq = lane & 3;
    double cr[T::TM][T::TN][2], ci[T::TM][T::TN][2];
#pragma unroll
    for (int i = 0; i < T::TM; ++i)
#pragma unroll
      for (int j = 0; j < T::TN; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
#pragma unroll
    for (int kb = 0; kb < D::DB_PAD; kb += 4) {
      const int col = (kb + kq) * D::PITCH;
      double xa[T::TM], ya[T::TM], xn[T::TM], xb[T::TN], yb[T::TN];
#pragma unroll
      for (int i = 0; i < T::TM; ++i) {
        const int row = (wr * T::TM + i) * 8 + m;
        xa[i] = X[row + col];
        ya[i] = Y[row + col];
        xn[i] = -xa[i];
      }
#pragma unroll
      for (int j = 0; j < T::TN; ++j) {
        const int row = (wc * T::TN + j) * 8 + m;
        xb[j] = X[row + col];
        yb[j] = Y[row + col];
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

// Norm check of spinmc.cpp:152-156 on trace(rho) = ||psi'||^2.
__device__ __forceinline__ bool not_normalized(double trace) {
  return fabs(__dsqrt_rn(trace) - 1.0) > 1e-9;
}

}  // namespace smem
}  // namespace tg
