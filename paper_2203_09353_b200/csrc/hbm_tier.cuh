// hbm_tier.cuh — HBM/L2-resident tier (13 <= S <= 24): psi and psi' are per-CTA slabs
// in the workspace (planar X, Y planes of 2^S doubles, column-major Psi[a][b] at
// a + b*d_a = amplitude index, spinmc.cpp:145-148). One CTA owns one replica at a time.
//
// rho = Psi' Psi'^dagger is computed in 64x64 complex output tiles; for each tile the
// K = d_b dimension streams through a 2-stage cp.async pipeline of 32-column chunks of
// the A (rows of tile i) and B (rows of tile j) panels, staged in SMEM with pitch 68
// doubles (conflict-free DMMA fragments, as in the SMEM tier). Each warp computes a
// 16x32 sub-tile (2x4 blocks of 8x8) with the real-split DMMA scheme; the epilogue folds
// sum |rho_ij|^2 and trace(rho) into per-thread running sums — rho is never stored.
#pragma once
#include "smem_tier.cuh"

namespace tg {
namespace hbm {

constexpr int kConsumerWarps = smem::kConsumerWarps;
constexpr int kConsumers = smem::kConsumers;
constexpr int kThreads = smem::kConsumers;  // no producer warp: the stream is pre-generated
constexpr int TB = 64;        // output tile (complex rows/cols)
constexpr int KC = 32;        // K columns per pipeline stage
constexpr int SP = TB + 4;    // SMEM pitch (doubles)
constexpr int kPanel = KC * SP;                 // doubles per (panel, plane)
constexpr int kStage = 4 * kPanel;              // A.X, A.Y, B.X, B.Y
constexpr int kStages = 2;
using T8 = smem::Tile<8>;                       // TM=2, TN=4, warp grid 4x2

using smem::Header;
constexpr int kHeaderBytes = smem::kHeaderBytes;
constexpr int kSmemBytes = kHeaderBytes + kStages * kStage * 8;


struct Geo {
  int spins, la, da, db, n;
  __device__ Geo(int s) : spins(s), la(s / 2), da(1 << (s / 2)), db(1 << (s - s / 2)), n(1 << s) {}
  __device__ int tiles() const { return da / TB; }
  __device__ int kchunks() const { return db / KC; }
};

// Gate application (spinmc.cpp:91-136), global planar -> global planar, reference rounding
// (bitwise the reference's psi' for the same U). R = GateRec (global or SMEM).
template <class R>
__device__ __forceinline__ void gate_pass(const double* __restrict__ sx, const double* __restrict__ sy,
                                          double* __restrict__ dx, double* __restrict__ dy,
                                          int spins, int site, const R& g, int tid,
                                          int nthreads) {
  double ur[16], ui[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    ur[e] = g.ur[e];
    ui[e] = g.ui[e];
  }
  const int groups = 1 << (spins - 2);
  const int lo_mask = (1 << site) - 1;
  for (int gi = tid; gi < groups; gi += nthreads) {
    const int base = ((gi >> site) << (site + 2)) | (gi & lo_mask);
    double vr[4], vi[4];
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      vr[y] = __ldcg(sx + (base | (y << site)));
      vi[y] = __ldcg(sy + (base | (y << site)));
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        re = __dadd_rn(re, __dsub_rn(__dmul_rn(ur[x * 4 + y], vr[y]), __dmul_rn(ui[x * 4 + y], vi[y])));
        im = __dadd_rn(im, __dadd_rn(__dmul_rn(ur[x * 4 + y], vi[y]), __dmul_rn(ui[x * 4 + y], vr[y])));
      }
      __stcg(dx + (base | (x << site)), re);
      __stcg(dy + (base | (x << site)), im);
    }
  }
}

// Issue the cp.async copies of pipeline iteration `it` (tile (ti,tj), chunk kc).
__device__ __forceinline__ void load_stage(const Geo& G, const double* X, const double* Y, int it,
                                           double* stage, int tid) {
  const int nk = G.kchunks(), nt = G.tiles();
  const int tile = it / nk, kc = it % nk;
  const int ti = tile / nt, tj = tile % nt;
  // 4 (panel, plane) pairs x KC columns x 32 row-pairs = 4096 16-byte copies
#pragma unroll 4
  for (int c = tid; c < 4 * KC * 32; c += kConsumers) {
    const int pp = c / (KC * 32);
    const int rem = c % (KC * 32);
    const int col = rem >> 5, rp = rem & 31;
    const double* src = (pp & 1) ? Y : X;
    const int row0 = ((pp >> 1) ? tj : ti) * TB;
    const double* g = src + (row0 + 2 * rp) + static_cast<size_t>(kc * KC + col) * G.da;
    double* s = stage + pp * kPanel + col * SP + 2 * rp;
    cp_async16(s, g);
  }
}

// rho partials over all tiles of Psi' (X, Y planes in global memory).
__device__ __forceinline__ void rho_partials(const Geo& G, const double* X, const double* Y,
                                             double* stages, int tid, int warp, int lane,
                                             bool fault, double& rho2_out, double& tr_out) {
  const int wr = warp / T8::WC, wc = warp % T8::WC;
  const int m = lane >> 2, kq = lane & 3;
  const int nk = G.kchunks(), nt = G.tiles();
  const int total = nt * nt * nk;
  double cr[2][4][2], ci[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
  double rho2 = 0.0, tr = 0.0;

  load_stage(G, X, Y, 0, stages, tid);
  cp_async_commit();
  for (int it = 0; it < total; ++it) {
    if (it + 1 < total) {
      load_stage(G, X, Y, it + 1, stages + ((it + 1) & 1) * kStage, tid);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    consumer_sync(kConsumers);
    const double* st = stages + (it & 1) * kStage;
    const double *AX = st, *AY = st + kPanel, *BX = st + 2 * kPanel, *BY = st + 3 * kPanel;
#pragma unroll
    for (int kb = 0; kb < KC; kb += 4) {
      const int col = (kb + kq) * SP;
      double xa[2], ya[2], xn[2], xb[4], yb[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int row = (wr * 2 + i) * 8 + m;
        xa[i] = AX[row + col];
        ya[i] = AY[row + col];
        xn[i] = -xa[i];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int row = (wc * 4 + j) * 8 + m;
        xb[j] = BX[row + col];
        yb[j] = BY[row + col];
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma(cr[i][j][0], cr[i][j][1], xa[i], xb[j]);
          dmma(cr[i][j][0], cr[i][j][1], ya[i], yb[j]);
          dmma(ci[i][j][0], ci[i][j][1], ya[i], xb[j]);
          dmma(ci[i][j][0], ci[i][j][1], xn[i], yb[j]);
        }
    }
    const int kc = it % nk;
    if (kc == nk - 1) {  // tile epilogue
      const int tile = it / nk, ti = tile / nt, tj = tile % nt;
      if (ti == tj) {
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (wr * 2 + i == wc * 4 + j) {
              if (m == 2 * kq) tr += cr[i][j][0];
              if (m == 2 * kq + 1) tr += cr[i][j][1];
            }
      }
      if (fault && tile == 0 && wr == 0 && wc == 0 && lane == 0)
        cr[0][0][0] -= 2.0 * (X[0] * X[0] + Y[0] * Y[0]);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            rho2 = fma(cr[i][j][e], cr[i][j][e], rho2);
            rho2 = fma(ci[i][j][e], ci[i][j][e], rho2);
            cr[i][j][e] = 0.0;
            ci[i][j][e] = 0.0;
          }
    }
    consumer_sync(kConsumers);  // stage (it&1) free for iteration it+2
  }
  rho2_out = warp_sum(rho2);
  tr_out = warp_sum(tr);
}

cudaError_t probe_apply_gate(uint32_t spins, const double* psi, int site, const double* u,
                             double* out, cudaStream_t s);
cudaError_t probe_entropy(uint32_t spins, uint64_t count, const double* psi, double* e,
                          double* n, bool fault, cudaStream_t s);

}  // namespace hbm
}  // namespace tg
