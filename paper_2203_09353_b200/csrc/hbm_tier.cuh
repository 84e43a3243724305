// hbm_tier.cuh — HBM/L2-resident tier (13 <= S <= 24): psi and psi' are slabs in the
// workspace (planar X, Y planes of 2^S doubles, column-major Psi[a][b] at a + b*d_a =
// amplitude index, spinmc.cpp:145-148). One replica is owned by a cluster of CS CTAs
// (CS = 1, 2 or 4; anneal_hbm.cu, ctas_per_replica).
//
// rho = Psi' Psi'^dagger is computed in 64x64 complex output tiles (row-major tile order
// t = ti*nt + tj); for each tile K = d_b streams through a 3-stage pipeline of 32-column
// chunks of the A (rows of tile i) and B (rows of tile j) panels: TMA tensor copies into
// 128-B swizzled boxes (rho_partials_tma, Renyi-2) or per-thread cp.async into panels of
// pitch 68 doubles (rho_partials; von Neumann, probes). Both layouts give conflict-free
// DMMA fragments and feed the DMMAs identical operands in identical order. Each warp computes a 16x32
// sub-tile (2x4 blocks of 8x8) with the real-split DMMA scheme; the epilogue folds
// sum |rho_ij|^2 and trace(rho) into four canonical chains (tile t -> chain t mod 4), and
// rho is never stored. Rank k of a CS-CTA cluster (CS = 1, 2, 4) takes the tiles
// t = k (mod CS), i.e. whole chains, so the result is bitwise the same whatever CS is.
#pragma once
#include "smem_tier.cuh"

namespace tg {
namespace hbm {

constexpr int kWarps = 8;
constexpr int kChains = 4;    // canonical reduction chains (tile t -> chain t % 4)
constexpr int kThreads = kWarps * 32;
constexpr int TB = 64;        // output tile (complex rows/cols)
constexpr int KC = 32;        // K columns per pipeline stage
constexpr int SP = TB + 4;    // SMEM pitch (doubles)
constexpr int kPanel = KC * SP;                 // doubles per (panel, plane)
constexpr int kStage = 4 * kPanel;              // A.X, A.Y, B.X, B.Y
constexpr int kStages = 3;
using T8 = smem::Tile<8>;                       // TM=2, TN=4, warp grid 4x2

struct Geo {
  int spins, la, da, db, n;
  __device__ Geo(int s) : spins(s), la(s / 2), da(1 << (s / 2)), db(1 << (s - s / 2)), n(1 << s) {}
  __device__ int tiles() const { return da / TB; }
  __device__ int kchunks() const { return db / KC; }
};

// ------------------------------------------------------------------------- clusters
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// Cluster-wide barrier with release/acquire at cluster scope (orders the global-memory
// slab writes of one CTA before the other CTA's reads).
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}
// Store v at the same SMEM offset as `local` in CTA `rank` of the cluster (DSMEM).
__device__ __forceinline__ void st_cluster_f64(double* local, uint32_t rank, double v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(v) : "memory");
}

// Gate application (spinmc.cpp:91-136) on groups [g0, g1), global planar -> global planar,
// reference rounding (bitwise the reference's psi' for the same U). R: GateRec.
// A thread takes a pair of groups {2q, 2q+1}: for site >= 1 their four amplitude pairs are
// adjacent (base(2q+1) = base(2q) + 1), for site 0 the pair is 8 consecutive amplitudes, so
// every access is a 16-byte ld/st.cg and a thread has 16 loads in flight before it
// computes (the pass is HBM/L2 latency bound, not FP64 bound).
__device__ __forceinline__ void gate_apply(const double* ur, const double* ui, const double vr[4],
                                           const double vi[4], double re_out[4], double im_out[4]) {
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    double re = 0.0, im = 0.0;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      re = __dadd_rn(re, __dsub_rn(__dmul_rn(ur[x * 4 + y], vr[y]), __dmul_rn(ui[x * 4 + y], vi[y])));
      im = __dadd_rn(im, __dadd_rn(__dmul_rn(ur[x * 4 + y], vi[y]), __dmul_rn(ui[x * 4 + y], vr[y])));
    }
    re_out[x] = re;
    im_out[x] = im;
  }
}
template <class R>
__device__ __forceinline__ void gate_pass(const double* __restrict__ sx, const double* __restrict__ sy,
                                          double* __restrict__ dx, double* __restrict__ dy,
                                          int site, const R& g, int g0, int g1, int tid,
                                          int nthreads) {
  double ur[16], ui[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    ur[e] = g.ur[e];
    ui[e] = g.ui[e];
  }
  const int lo_mask = (1 << site) - 1;
  auto offset = [&](int q, int y) {  // amplitude offset of load/store y of pair q
    const int gi = 2 * q;
    const int base = ((gi >> site) << (site + 2)) | (gi & lo_mask);
    return site == 0 ? base + 2 * y : base + (y << site);
  };
  // software-pipelined: the loads of the thread's next pair are issued before the current
  // pair is computed and stored (stores would otherwise fence the next loads: one L2/HBM
  // round trip per pair)
  double2 lr[4], li[4], nr[4], ni[4];
  const int q1 = g1 >> 1;
  int q = (g0 >> 1) + tid;
  if (q < q1) {
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      lr[y] = __ldcg(reinterpret_cast<const double2*>(sx + offset(q, y)));
      li[y] = __ldcg(reinterpret_cast<const double2*>(sy + offset(q, y)));
    }
  }
  for (; q < q1; q += nthreads) {
    const int qn = q + nthreads;
    if (qn < q1) {
#pragma unroll
      for (int y = 0; y < 4; ++y) {
        nr[y] = __ldcg(reinterpret_cast<const double2*>(sx + offset(qn, y)));
        ni[y] = __ldcg(reinterpret_cast<const double2*>(sy + offset(qn, y)));
      }
    }
    double vr[2][4], vi[2][4];
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      if (site == 0) {  // group 2q: amplitudes base..base+3, group 2q+1: base+4..base+7
        vr[y >> 1][2 * (y & 1)] = lr[y].x;
        vr[y >> 1][2 * (y & 1) + 1] = lr[y].y;
        vi[y >> 1][2 * (y & 1)] = li[y].x;
        vi[y >> 1][2 * (y & 1) + 1] = li[y].y;
      } else {
        vr[0][y] = lr[y].x;
        vr[1][y] = lr[y].y;
        vi[0][y] = li[y].x;
        vi[1][y] = li[y].y;
      }
    }
    double ro[2][4], io[2][4];
    gate_apply(ur, ui, vr[0], vi[0], ro[0], io[0]);
    gate_apply(ur, ui, vr[1], vi[1], ro[1], io[1]);
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      double2 a, b;
      if (site == 0) {
        a = make_double2(ro[x >> 1][2 * (x & 1)], ro[x >> 1][2 * (x & 1) + 1]);
        b = make_double2(io[x >> 1][2 * (x & 1)], io[x >> 1][2 * (x & 1) + 1]);
      } else {
        a = make_double2(ro[0][x], ro[1][x]);
        b = make_double2(io[0][x], io[1][x]);
      }
      __stcg(reinterpret_cast<double2*>(dx + offset(q, x)), a);
      __stcg(reinterpret_cast<double2*>(dy + offset(q, x)), b);
    }
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      lr[y] = nr[y];
      li[y] = ni[y];
    }
  }
}

// Gate pass for an HBM-resident state (S >= 16, one CTA per replica), staged through the
// drained GEMM stage buffers: the TMA engine copies chunks of kGateChunk groups (their four
// amplitude slices, or one contiguous range when the groups span whole 2^(site+2) blocks)
// into a 3-buffer ring (1-D bulk copies, mbarrier completion), the CTA applies the gate in
// shared memory with gate_apply (the reference rounding: bitwise gate_pass) and bulk stores
// write the chunk back. Per-SM bytes in flight are then bounded by the ring (128 KB) instead
// of the threads' registers. gpar: the ring's mbarrier parities (kept across passes).
constexpr int kGateChunk = 1024;  // default groups per chunk: 4096 amplitudes = 32 KB per plane
constexpr int kGateRingBytes = 3 * 8 * kGateChunk * 8;  // 192 KB: the ring's share of the stage buffers
static_assert(kGateRingBytes <= kStages * kStage * 8, "gate ring fits the stage buffers");
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// C: groups per chunk (a power of two dividing g1 - g0); the ring holds NB = min(8, 192 KB /
// chunk bytes) chunks, NB - 1 of them in flight.
template <class R>
__device__ void gate_pass_bulk(const double* __restrict__ sx, const double* __restrict__ sy,
                               double* __restrict__ dx, double* __restrict__ dy, int site, const R& g,
                               int g0, int g1, int tid, double* ring, uint64_t* bars, uint32_t& gpar,
                               int C = kGateChunk) {
  const int A = 4 * C;  // amplitudes per plane of one chunk
  const int NB = min(8, kGateRingBytes / (64 * C));
  double ur[16], ui[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    ur[e] = g.ur[e];
    ui[e] = g.ui[e];
  }
  const int lo_mask = (1 << site) - 1;
  auto base = [&](int gi) { return ((gi >> site) << (site + 2)) | (gi & lo_mask); };
  const bool sliced = C <= (1 << site);  // a chunk's groups share their high bits: 4 slices
  const int nch = (g1 - g0) / C;
  auto buf = [&](int j) { return ring + (j % NB) * 2 * A; };  // [X: A][Y: A]
  auto issue = [&](int j) {  // thread 0
    double* b = buf(j);
    uint64_t* bar = &bars[j % NB];
    mbar_expect_tx(bar, 2 * A * 8);
    const int gs = g0 + j * C, a0 = base(gs);
    if (sliced) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        bulk_g2s(b + t * C, sx + a0 + (t << site), C * 8, bar);
        bulk_g2s(b + A + t * C, sy + a0 + (t << site), C * 8, bar);
      }
    } else {
      bulk_g2s(b, sx + a0, A * 8, bar);
      bulk_g2s(b + A, sy + a0, A * 8, bar);
    }
  };
  auto store = [&](int j) {  // thread 0
    const double* b = buf(j);
    const int gs = g0 + j * C, a0 = base(gs);
    if (sliced) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        bulk_s2g(dx + a0 + (t << site), b + t * C, C * 8);
        bulk_s2g(dy + a0 + (t << site), b + A + t * C, C * 8);
      }
    } else {
      bulk_s2g(dx + a0, b, A * 8);
      bulk_s2g(dy + a0, b + A, A * 8);
    }
    bulk_commit();
  };
  fence_proxy_async_smem();  // the GEMM's generic reads of the stage buffers come first
  __syncthreads();
  if (tid == 0)
    for (int j = 0; j < NB - 1 && j < nch; ++j) issue(j);
  for (int j = 0; j < nch; ++j) {
    double* b = buf(j);
    const int q = j % NB;
    mbar_wait(&bars[q], (gpar >> q) & 1u);
    gpar ^= 1u << q;
    const int gs = g0 + j * C, a0 = base(gs);
#pragma unroll 2
    for (int i = tid; i < C; i += kThreads) {
      int off[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) off[t] = sliced ? t * C + i : base(gs + i) + (t << site) - a0;
      double vr[4], vi[4], ro[4], io[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        vr[t] = b[off[t]];
        vi[t] = b[A + off[t]];
      }
      gate_apply(ur, ui, vr, vi, ro, io);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        b[off[t]] = ro[t];
        b[A + off[t]] = io[t];
      }
    }
    fence_proxy_async_smem();  // generic writes of the chunk before the bulk store reads them
    __syncthreads();
    if (tid == 0) {
      store(j);
      if (j + NB - 1 < nch) {
        bulk_wait_read<1>();  // chunk j-1's store has read buffer (j+NB-1) % NB
        issue(j + NB - 1);
      }
    }
  }
  if (tid == 0) {
    bulk_wait_all();  // psi' complete in global memory before the GEMM reads it
    __threadfence();
    fence_proxy_async_global();
  }
}

// Issue the cp.async copies of one pipeline stage: panels of tile (ti, tj), chunk kc.
// 4 (panel, plane) x 32 columns x 32 row-pairs = 4096 16-byte copies, 16 per thread;
// thread tid copies row-pair rp = tid & 31 of columns 8*(i & 3) + (tid >> 5), plane-panel
// i >> 2 (i = 0..15), so all index math is per-thread constants plus one chunk offset.
__device__ __forceinline__ void load_stage(const double* X, const double* Y, int da, int ti, int tj,
                                           int kc, double* stage, int tid, int i0 = 0, int i1 = 16) {
  const int rp = tid & 31, c0 = tid >> 5;
#pragma unroll
  for (int i = i0; i < i1; ++i) {
    const int pp = i >> 2, col = 8 * (i & 3) + c0;
    const double* src = (pp & 1) ? Y : X;
    const int row0 = ((pp >> 1) ? tj : ti) * TB;
    const double* g = src + (row0 + 2 * rp) + static_cast<size_t>(kc * KC + col) * da;
    cp_async16(stage + pp * kPanel + col * SP + 2 * rp, g);
  }
}

// inject_fault: flip the sign of the first accumulation term of rho(0,0) (linalg.cpp:94).
// One definition for every schedule (cluster and queue), so their rounding is the same.
__device__ __forceinline__ void fault_term(double& c, double x0, double y0) { c -= 2.0 * (x0 * x0 + y0 * y0); }

// Tile epilogue, part 1: the diagonal tile's trace into chain ch; the fault injection.
__device__ __forceinline__ void tile_trace_fault(double (&cr)[2][4][2], double (&tr)[kChains], int ch, bool diag,
                                                 bool fault, const double* X, const double* Y, int wr, int wc,
                                                 int m, int kq, int lane) {
  if (diag) {
    double tsum = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) tsum = c == ch ? tr[c] : tsum;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (wr * 2 + i == wc * 4 + j) {
          if (m == 2 * kq) tsum += cr[i][j][0];
          if (m == 2 * kq + 1) tsum += cr[i][j][1];
        }
#pragma unroll
    for (int c = 0; c < kChains; ++c) tr[c] = c == ch ? tsum : tr[c];
  }
  if (fault && wr == 0 && wc == 0 && lane == 0) fault_term(cr[0][0][0], X[0], Y[0]);
}

// Tile epilogue, part 2: the tile's sum |rho_ij|^2 into chain ch, in four interleaved
// sub-chains (the fold is 8 DFMA deep instead of 32: it runs next to other warps' DMMA
// streams, which starve FP64 latency chains); zero the accumulators for the next tile.
__device__ __forceinline__ void tile_fold(double (&cr)[2][4][2], double (&ci)[2][4][2], double (&rho)[kChains],
                                          int ch, bool zero) {
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double& a = acc[((i * 4 + j) * 2 + e) & 3];
        a = fma(cr[i][j][e], cr[i][j][e], a);
        a = fma(ci[i][j][e], ci[i][j][e], a);
        if (zero) {
          cr[i][j][e] = 0.0;
          ci[i][j][e] = 0.0;
        }
      }
  const double tv = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
  for (int c = 0; c < kChains; ++c) rho[c] = c == ch ? rho[c] + tv : rho[c];
}

// rho partials of the tiles t = first, first + stride, ... (rank's share), as kChains chains
// by t mod 4: out = {rho2 chain 0..3, trace chain 0..3}, warp-reduced (all lanes).
// inject_fault flips the sign of the first accumulation term of rho(0,0) (linalg.cpp:94)
// after the trace is taken.
// STORE (von Neumann, single tile d_a = TB only): after the pipeline drains, rho is also
// written to planar SMEM Rr/Ri (pitch RP), which may alias the (then free) stage buffers.
template <bool STORE = false>
__device__ __forceinline__ void rho_partials(const Geo& G, const double* X, const double* Y,
                                             double* stages, int tid, int warp, int lane,
                                             int first, int stride, bool fault, double out[2 * kChains],
                                             double* Rr = nullptr, double* Ri = nullptr, int RP = 0,
                                             int64_t* prof = nullptr, double* Rg = nullptr) {
  // STORE with Rg (von Neumann, d_a > TB): every finished tile is written to the global
  // column-major planes Rg (Re) and Rg + d_a^2 (Im) instead of SMEM.
  // prof (profiling probe only, thread 0): [0] clk in the chunk waits + barriers,
  // [1] clk in tile epilogues, [2] the largest per-warp wait.
  int64_t t_wait = 0, t_epi = 0;
  const int wr = warp / T8::WC, wc = warp % T8::WC;
  const int m = lane >> 2, kq = lane & 3;
  const int nk = G.kchunks(), nt = G.tiles();
  const int mine = (nt * nt - first + stride - 1) / stride;
  const int lnt = G.la - 6, lnk = (G.spins - G.la) - 5;  // log2 of nt = d_a/64, nk = d_b/32
  const int total = mine * nk;
  double cr[2][4][2], ci[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
  double rho[kChains] = {0.0, 0.0, 0.0, 0.0}, tr[kChains] = {0.0, 0.0, 0.0, 0.0};
  auto issue = [&](int it) {
    if (it < total) {
      const int t = first + (it / nk) * stride, kc = it % nk;
      load_stage(X, Y, G.da, t / nt, t % nt, kc, stages + (it % kStages) * kStage, tid);
    }
    cp_async_commit();  // (possibly empty) group per iteration keeps the wait counts uniform
  };
  issue(0);
  issue(1);
  for (int it = 0; it < total; ++it) {
    const int64_t tw0 = prof ? clock64() : 0;
    cp_async_wait<1>();       // this thread's copies of stage `it` landed
    consumer_sync(kThreads);  // everyone's did; stage (it-1) % 3 is free
    if (prof) t_wait += clock64() - tw0;
    // stage it+2 is issued 2 copies per k-step, spread over the chunk's 8 k-steps (keeps
    // the LSU queue short). Its addresses are set up here, once per chunk, as 32-bit
    // offsets from X (Y = X + n): an address computation inside the k-steps sits on the
    // warps' issue path right after their DMMAs and, with both warps of an SMSP in step
    // after the barrier, leaves the DMMA pipe idle (measured: ~15% of the GEMM).
    const int nx = it + 2;
    const bool has_next = nx < total;
    uint32_t soff[4];
    uint32_t doff;
    {
      const int tn = first + (nx >> lnk) * stride, kcn = nx & (nk - 1);
      const int ti = tn >> lnt, tj = tn & (nt - 1);
      const int rp = tid & 31, c0 = tid >> 5;
#pragma unroll
      for (int pp = 0; pp < 4; ++pp)
        soff[pp] = static_cast<uint32_t>((pp & 1) * G.n + ((pp >> 1) ? tj : ti) * TB + 2 * rp) +
                   static_cast<uint32_t>(kcn * KC + c0) * static_cast<uint32_t>(G.da);
      doff = static_cast<uint32_t>((nx % kStages) * kStage + c0 * SP + 2 * rp);
    }
    const uint32_t col8 = 8u * static_cast<uint32_t>(G.da);
    const double* st = stages + (it % kStages) * kStage;
    const double *AX = st, *AY = st + kPanel, *BX = st + 2 * kPanel, *BY = st + 3 * kPanel;
#pragma unroll
    for (int kb = 0; kb < KC; kb += 4) {
      if (has_next) {
#pragma unroll
        for (int i = kb / 2; i < kb / 2 + 2; ++i) {  // copy i: panel-plane i >> 2, column 8 * (i & 3) + c0
          const int pp = i >> 2, j = i & 3;
          cp_async16(stages + doff + pp * kPanel + 8 * j * SP, X + (soff[pp] + j * col8));
        }
      }
      if (kb == KC - 4) cp_async_commit();
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
    if (it % nk == nk - 1) {  // tile epilogue
      const int64_t te0 = prof ? clock64() : 0;
      const int t = first + (it / nk) * stride, ti = t / nt, tj = t % nt;
      const int ch = t & (kChains - 1);  // chain (selects below, not a dynamic index: no local memory)
      tile_trace_fault(cr, tr, ch, ti == tj, fault && t == 0, X, Y, wr, wc, m, kq, lane);
      if (STORE && Rg) {
        const size_t pl = static_cast<size_t>(G.da) * G.da;
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const size_t o = static_cast<size_t>(ti * TB + (wr * 2 + i) * 8 + m) +
                               static_cast<size_t>(tj * TB + (wc * 4 + j) * 8 + 2 * kq + e) * G.da;
              __stcg(Rg + o, cr[i][j][e]);
              __stcg(Rg + pl + o, ci[i][j][e]);
            }
      }
      tile_fold(cr, ci, rho, ch, !STORE || Rg);
      if (prof) t_epi += clock64() - te0;
    }
  }
  if (prof) {  // [2]: the largest per-warp wait (thread 0's is [0])
    __shared__ int64_t wwait[kWarps];
    if (lane == 0) wwait[warp] = t_wait;
    consumer_sync(kThreads);
    if (tid == 0) {
      int64_t mx = 0;
      for (int w = 0; w < kWarps; ++w) mx = wwait[w] > mx ? wwait[w] : mx;
      prof[0] = t_wait;
      prof[1] = t_epi;
      prof[2] = mx;
    }
  }
  cp_async_wait<0>();
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    out[c] = warp_sum(rho[c]);
    out[kChains + c] = warp_sum(tr[c]);
  }
  consumer_sync(kThreads);  // all warps done with the stages before they are reused
  if (STORE && !Rg) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int o = (wr * 2 + i) * 8 + m + ((wc * 4 + j) * 8 + 2 * kq + e) * RP;
          Rr[o] = cr[i][j][e];
          Ri[o] = ci[i][j][e];
        }
    consumer_sync(kThreads);
  }
}

// ------------------------------------------------------------------ TMA-staged variant
// The same GEMM with the stages filled by the TMA engine instead of per-thread cp.async
// (Renyi-2 only). One 5-D tensor map covers every cluster's slab (anneal_hbm.cu,
// hbm_tensor_map): dim0 16 rows (one 128-B line), dim1 16-row block (stride 16 rows), dim2
// column b (stride d_a), dim3 plane 2*buffer + {X, Y} (stride n), dim4 cluster slot. One box
// (16, 2, 32, 2, 1) is 32 rows x 32 columns of both planes; a stage is 4 boxes (A and B
// panels, two row halves h each) issued by thread 0. With CU_TENSOR_MAP_SWIZZLE_128B row r
// of column k, plane p of a panel lands at (doubles)
//   h * 2048 + p * 1024 + k * 32 + b * 16 + 2 * (((r >> 1) & 7) ^ (b + 2 * (k & 3))) + (r & 1)
// with h = r >> 5, b = (r >> 4) & 1: 128-B line L = 2k + b has its 16-B chunks permuted by
// L & 7. A DMMA fragment's half-warp (4 rows x 4 k) then reads 16 distinct 8-B slots of
// one 128-B bank window: conflict-free.
// Stage reuse is tracked by mbarriers instead of a CTA barrier per chunk: full[s] (one
// arrival + 64 KB of transactions), empty[s] (one arrival per warp after its last read).
constexpr int kTmaBox = 16 * 2 * KC * 2;          // doubles per box (32 rows, both planes)
constexpr int kTmaPanel = 2 * kTmaBox;            // 64 rows
constexpr uint32_t kTmaStageBytes = 2 * kTmaPanel * 8;
static_assert(2 * kTmaPanel <= kStage, "TMA stage fits the cp.async stage stride");

struct TmaPipe {
  uint64_t* full;   // [kStages]
  uint64_t* empty;  // [kStages]
  uint64_t seq;     // chunks consumed so far by this CTA (identical in every thread; 64-bit:
                    // stage q % 3 and parity (q / 3) & 1 must not wrap within a launch)
};

__device__ __forceinline__ void rho_partials_tma(const Geo& G, const void* tmap, int buf, int slot, double* stages,
                                                 TmaPipe& pipe, int tid, int warp, int lane, int first, int stride,
                                                 bool fault, const double* X, const double* Y,
                                                 double out[2 * kChains], int64_t* prof = nullptr) {
  int64_t t_wait = 0, t_epi = 0;
  const int wr = warp / T8::WC, wc = warp % T8::WC;
  const int m = lane >> 2, kq = lane & 3;
  const int nk = G.kchunks(), nt = G.tiles();
  const int mine = (nt * nt - first + stride - 1) / stride;
  const int lnt = G.la - 6, lnk = (G.spins - G.la) - 5;
  const int total = mine * nk;
  // fragment offsets within a panel (X plane) of 8-row block q, for k = kq (+ kb * 32)
  auto frag = [&](int q) {
    const int r = q * 8 + m, b = (r >> 4) & 1;
    return (r >> 5) * 2048 + kq * 32 + b * 16 + 2 * (((r >> 1) & 7) ^ (b + 2 * kq)) + (r & 1);
  };
  int fa[2], fb[4];
#pragma unroll
  for (int i = 0; i < 2; ++i) fa[i] = frag(wr * 2 + i);
#pragma unroll
  for (int j = 0; j < 4; ++j) fb[j] = frag(wc * 4 + j);
  double cr[2][4][2], ci[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
  double rho[kChains] = {0.0, 0.0, 0.0, 0.0}, tr[kChains] = {0.0, 0.0, 0.0, 0.0};
  const uint64_t seq0 = pipe.seq;
  auto issue = [&](int it) {  // thread 0: chunk it into stage (seq0 + it) % kStages
    const uint64_t q = seq0 + static_cast<uint64_t>(it);
    const int s = static_cast<int>(q % kStages);
    if (q >= static_cast<uint64_t>(kStages)) mbar_wait(&pipe.empty[s], static_cast<uint32_t>(q / kStages - 1) & 1);
    const int t = first + (it >> lnk) * stride, kc = it & (nk - 1);
    const int ti = t >> lnt, tj = t & (nt - 1);
    double* st = stages + s * kStage;
    const bool diag = ti == tj;  // diagonal tile: the B panel is the A panel (half the copy)
    mbar_expect_tx(&pipe.full[s], diag ? kTmaStageBytes / 2 : kTmaStageBytes);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      tma_load_5d(st + h * kTmaBox, tmap, 0, ti * 4 + 2 * h, kc * KC, 2 * buf, slot, &pipe.full[s]);
      if (!diag)
        tma_load_5d(st + kTmaPanel + h * kTmaBox, tmap, 0, tj * 4 + 2 * h, kc * KC, 2 * buf, slot, &pipe.full[s]);
    }
  };
  if (tid == 0) {
    if (total > 0) issue(0);
    if (total > 1) issue(1);
  }
  for (int it = 0; it < total; ++it) {
    const uint64_t q = seq0 + static_cast<uint64_t>(it);
    const int s = static_cast<int>(q % kStages);
    if (tid == 0 && it + 2 < total) issue(it + 2);
    const int64_t tw0 = prof ? clock64() : 0;
    mbar_wait(&pipe.full[s], static_cast<uint32_t>(q / kStages) & 1);
    if (prof) t_wait += clock64() - tw0;
    const double* st = stages + s * kStage;
    const int tcur = first + (it >> lnk) * stride;
    const bool dcur = (tcur >> lnt) == (tcur & (nt - 1));
    const double *AX = st, *AY = st + 1024;
    const double *BX = dcur ? AX : st + kTmaPanel, *BY = dcur ? AY : st + kTmaPanel + 1024;
#pragma unroll
    for (int kb = 0; kb < KC; kb += 4) {
      double xa[2], ya[2], xn[2], xb[4], yb[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        xa[i] = AX[fa[i] + kb * 32];
        ya[i] = AY[fa[i] + kb * 32];
        xn[i] = -xa[i];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        xb[j] = BX[fb[j] + kb * 32];
        yb[j] = BY[fb[j] + kb * 32];
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&pipe.empty[s]);  // this warp is done reading stage s
    if (it % nk == nk - 1) {                      // tile epilogue
      const int64_t te0 = prof ? clock64() : 0;
      const int t = first + (it / nk) * stride, ti = t / nt, tj = t % nt;
      const int ch = t & (kChains - 1);
      tile_trace_fault(cr, tr, ch, ti == tj, fault && t == 0, X, Y, wr, wc, m, kq, lane);
      tile_fold(cr, ci, rho, ch, true);
      if (prof) t_epi += clock64() - te0;
    }
  }
  pipe.seq = seq0 + static_cast<uint64_t>(total);
  if (prof) {
    __shared__ int64_t wwait_t[kWarps];
    if (lane == 0) wwait_t[warp] = t_wait;
    __syncthreads();
    if (tid == 0) {
      int64_t mx = 0;
      for (int w = 0; w < kWarps; ++w) mx = wwait_t[w] > mx ? wwait_t[w] : mx;
      prof[0] = t_wait;
      prof[1] = t_epi;
      prof[2] = mx;
    }
  }
#pragma unroll
  for (int c = 0; c < kChains; ++c) {
    out[c] = warp_sum(rho[c]);
    out[kChains + c] = warp_sum(tr[c]);
  }
}

// ------------------------------------------------- per-CTA header, shared helpers
constexpr int kMaxCS = 4;
struct HHeader {
  GateRec rec[2];                    // proposal records of steps s, s + 1 (prefetched)
  double part[kWarps][2 * kChains];  // per-warp chain values {rho chain 0..3, tr chain 0..3}
  double val[kMaxCS][2 * kChains];   // per-rank chain sums (other ranks' arrive by DSMEM)
  double norm_q[4];                  // renormalisation: sums over the four quarters of psi
  uint64_t full[kStages];            // TMA pipeline (rho_partials_tma)
  uint64_t empty[kStages];
  uint64_t gfull[8];                 // staged gate pass (gate_pass_bulk): one per chunk buffer
  int32_t decision;
  int32_t error;
};
constexpr int kHHeaderBytes = (static_cast<int>(sizeof(HHeader)) + 127) / 128 * 128;
// + 1 KB: the anneal kernel aligns its stages to 1 KB (the TMA swizzle is a function of the
// SMEM address bits)
constexpr int kSmemBytes = kHHeaderBytes + kStages * kStage * 8 + 1024;

template <int CS>
__device__ __forceinline__ void sync_all() {
  if constexpr (CS == 1) {
    __syncthreads();
  } else {
    cluster_sync();
  }
}

// Per-rank values (sum of the per-warp chain values in warp order) published to every rank.
template <int CS>
__device__ __forceinline__ void publish_vals(HHeader& H, int tid, uint32_t rank) {
  __syncthreads();  // per-warp parts written
  if (tid < 2 * kChains) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) v += H.part[w][tid];
    H.val[rank][tid] = v;
#pragma unroll
    for (uint32_t d = 1; d < static_cast<uint32_t>(CS); ++d) st_cluster_f64(&H.val[rank][tid], (rank + d) % CS, v);
  }
  sync_all<CS>();
}

// Totals in the canonical order ((c0 + c1) + (c2 + c3)); chain c was summed by rank c % CS.
template <int CS>
__device__ __forceinline__ void totals(const HHeader& H, double& rho2, double& tr) {
  auto v = [&](int k) { return H.val[(k % kChains) % CS][k]; };
  rho2 = (v(0) + v(1)) + (v(2) + v(3));
  tr = (v(4) + v(5)) + (v(6) + v(7));
}

// renormalize (spinmc.cpp:56-59) over the four quarters of psi (rank k owns quarters
// q = k mod CS); the total is ((q0 + q1) + (q2 + q3)) whatever CS is, so every CS agrees
// bitwise.
template <int CS>
__device__ void renormalize(const Geo& G, double* X, double* Y, int tid, int warp, int lane,
                            uint32_t rank, HHeader& H) {
  const int quarter = G.n / 4;
  for (int q = static_cast<int>(rank); q < 4; q += CS) {
    double s = 0.0;
    for (int i = q * quarter + tid; i < (q + 1) * quarter; i += kThreads) {
      const double x = __ldcg(X + i), y = __ldcg(Y + i);
      s = fma(x, x, s);
      s = fma(y, y, s);
    }
    s = warp_sum(s);
    if (lane == 0) H.part[warp][0] = s;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) t += H.part[w][0];
      H.norm_q[q] = t;
      for (uint32_t d = 1; d < static_cast<uint32_t>(CS); ++d) st_cluster_f64(&H.norm_q[q], (rank + d) % CS, t);
    }
    __syncthreads();
  }
  sync_all<CS>();
  const double inv = __ddiv_rn(1.0, __dsqrt_rn((H.norm_q[0] + H.norm_q[1]) + (H.norm_q[2] + H.norm_q[3])));
  const int part = G.n / CS, i0 = static_cast<int>(rank) * part, i1 = i0 + part;
  for (int i = i0 + tid; i < i1; i += kThreads) {
    __stcg(X + i, __dmul_rn(__ldcg(X + i), inv));
    __stcg(Y + i, __dmul_rn(__ldcg(Y + i), inv));
  }
  __threadfence();
  fence_proxy_async_global();  // the next GEMM may read psi through the TMA engine
  sync_all<CS>();
}

cudaError_t probe_apply_gate(uint32_t spins, const double* psi, int site, const double* u,
                             double* out, cudaStream_t s);
cudaError_t probe_entropy(uint32_t spins, uint64_t count, const double* psi, double* e,
                          double* n, bool fault, cudaStream_t s, bool von_neumann = false);

}  // namespace hbm
}  // namespace tg
