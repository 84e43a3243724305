// hbm_queue.cuh — HBM tier, work-queue schedule (Renyi-2, TMA-staged GEMM).
//
// The cluster schedule (anneal_hbm_kernel) binds a replica to 1, 2 or 4 CTAs for its whole
// trajectory, so a batch of R replicas keeps at most R x CS SMs busy and a partial last wave
// idles the rest (64 replicas of L = 20 on 148 SMs: 128 busy). Here every CTA of a
// persistent grid pulls work items from one global queue instead:
//   INIT(r, part)  initial state of replica r, 1/P of the amplitudes    (mc_procedure, spinmc.cpp:229-232)
//   NORM(r)        random start: renormalise                          (spinmc.cpp:37-48, 56-59)
//   TILE(r, s, t)  one 64x64 output tile of rho = Psi' Psi'^dagger     (spinmc.cpp:157-164, linalg.cpp:79-103)
//   DEC(r, s)      fold the tiles' partials, Metropolis decision,     (spinmc.cpp:193-213, 246-248)
//                  trace, renormalisation every `renorm` steps
//   GATE(r, s, p)  the two-site gate of step s on 1/P of the groups    (spinmc.cpp:91-136)
// (s = -1 is the initial-entropy GEMM, spinmc.cpp:234). Items are ordered so that every
// item's inputs are produced by EARLIER items; a CTA that pulls an item whose inputs are not
// ready waits on per-replica completion counters (release/acquire at GPU scope). The
// earliest unfinished item can always run, so the schedule cannot deadlock whatever the
// number of resident CTAs, and it needs no grid-wide barrier: replica r's decision and next
// gate overlap other replicas' GEMM tiles.
//
// Queue layout: a prologue of R x (P [+1]) INIT [NORM] items, then blocks k = 0 .. K+lagG-1
// (K = (steps + 1) R, position k = replica k mod R at step k / R - 1), each
//   [ntt TILE items of position k] [DEC of position k - lagD] [GATE parts 1..P-1: next step of position k - lagG]
// (the DEC item applies part 0 of its replica's next gate itself, right after deciding)
// (slots without work are skipped). lagG < R keeps GATE(r, s+1) ahead of TILE(r, s+1);
// lagD ~ 2 x grid / ntt tile items lets position k's tiles finish before its DEC is pulled,
// and lagG ~ lagD + one CTA round of items lets the DEC finish before its other gate parts
// are pulled.
//
// Determinism. A tile stores its per-thread partials (the ||rho||^2 term tile_fold forms and
// the diagonal trace terms tile_trace_fault adds) instead of adding them to per-thread
// chains; DEC replays the chains in ascending tile order from those values, then the same
// warp / warp-order / chain folds as the cluster kernel. Results are therefore bitwise those
// of the 1-, 2- and 4-CTA cluster schedules whichever CTA computed which tile.
#pragma once
#include "hbm_tier.cuh"
#include "tg_internal.h"
#include "vn_large.cuh"

namespace tg {
namespace hbmq {
using namespace hbm;

enum : int32_t { kItemEmpty = 0, kItemTile, kItemInit, kItemNorm, kItemGate, kItemDec, kItemEnd };
enum : int32_t { kMetaTile = 0, kMetaControl = 1 };

struct Item {
  int32_t type;
  int32_t part;  // tile t, or INIT / GATE part
  int64_t s;     // step (-1: initial state / entropy)
  uint64_t r;    // row
};

// Per-row state (workspace), written by INIT part 0 and DEC, read by GATE / TILE / DEC.
struct QRow {
  int32_t cur, err;  // current buffer, failed norm check
  double cur_e;      // raw ||rho||_F^2 of the current state (finish_renyi converts the trace)
  int64_t t_prev, t_row0;
};

struct QMeta {  // one pipeline stage entry (written by the producer)
  int32_t kind, t, kc, buf;
  Item x;  // TILE: x.r is the row; CONTROL: the item itself
};

constexpr int kQStats = 24;
struct QHeader {
  HHeader h;
  uint64_t ctl_done;  // von Neumann: a DEC item has released the stage buffers (its scratch)
  QMeta meta[kStages];  // read by the consumers (written by the async proxy only)
  QRow row;          // row-state snapshot for a control item
  alignas(16) GateRec rec[2];  // control items: proposal records of steps s (decision) and s + 1 (gate)
  int64_t stat[kQStats];  // STATS probe only (anneal_queue_kernel<true>)
};
constexpr int kQHeaderBytes = (static_cast<int>(sizeof(QHeader)) + 127) / 128 * 128;
constexpr int kQSmemBytes = kQHeaderBytes + kStages * kStage * 8 + 1024;
// warp specialisation: two consumer warpgroups (DMMA, control items) + one producer warpgroup
// (one thread pulls items, waits for dependencies and issues the TMA stages)
constexpr int kQThreads = kThreads + 128;
constexpr int kConsumerRegs = 240, kProducerRegs = 24;  // 256 x 240 + 128 x 24 <= 64K
static_assert(kThreads * kConsumerRegs + 128 * kProducerRegs <= 65536, "register file");

// Queue geometry; identical on host (sizing, launch) and device.
struct QGeo {
  uint32_t spins, nt, ntt, nfull, P, Ip, lagD, lagG;
  bool half;  // rho_half: the upper-triangle tiles only (ntt = nt (nt + 1) / 2 items per step)
  uint64_t rows, steps, BS, pro, K, total, n;
  __host__ __device__ static uint32_t gate_parts(uint32_t spins) {
    const uint64_t groups = uint64_t{1} << (spins - 2);
    const uint64_t p = groups / 4096;
    return static_cast<uint32_t>(p < 1 ? 1 : (p > 16 ? 16 : p));
  }
  bool long_dec;  // von Neumann: the DEC item (an eigen-solve) applies the whole next gate itself
  __host__ __device__ QGeo(uint32_t s, uint64_t r, uint64_t st, bool random, uint32_t grid, bool h = false,
                           bool ldec = false) {
    spins = s;
    n = uint64_t{1} << s;
    nt = (1u << (s / 2)) / TB;
    nfull = nt * nt;
    half = h;
    long_dec = ldec;
    ntt = half ? nt * (nt + 1) / 2 : nfull;
    P = gate_parts(s);
    Ip = P + (random ? 1 : 0);
    rows = r;
    steps = st;
    // tiles, DEC (+ gate part 0 of the next step, or all of it), gate parts 1 .. P-1
    BS = ntt + (long_dec ? 1 : P);
    const uint64_t want = (2ull * grid + ntt - 1) / ntt;
    const uint64_t lmax = r > 0 ? r - 1 : 0;
    const uint64_t wantG = want + (P > 1 ? (grid + BS - 1) / BS : 0);  // ~ one CTA round after the DEC
    lagG = static_cast<uint32_t>(wantG < lmax ? wantG : lmax);
    lagD = static_cast<uint32_t>(want < lagG ? want : lagG);
    if (long_dec) lagG = lagD = 0;  // a DEC outlasts many CTA rounds of tiles: pull it right after its tiles
    pro = r * Ip;
    K = (st + 1) * r;
    total = pro + (K + lagG) * BS;
  }
  __host__ __device__ Item decode(uint64_t i) const {
    Item x{kItemEmpty, 0, 0, 0};
    if (i >= total) {
      x.type = kItemEnd;
      return x;
    }
    if (i < pro) {
      x.r = i / Ip;
      const uint32_t j = static_cast<uint32_t>(i - x.r * Ip);
      x.s = -1;
      x.part = static_cast<int32_t>(j);
      x.type = j < P ? kItemInit : kItemNorm;
      return x;
    }
    const uint64_t ip = i - pro, k = ip / BS;
    const uint32_t j = static_cast<uint32_t>(ip - k * BS);
    if (j < ntt) {
      if (k >= K) return x;
      x.type = kItemTile;
      x.r = k % rows;
      x.s = static_cast<int64_t>(k / rows) - 1;
      x.part = static_cast<int32_t>(half ? upper_tile(j) : j);  // full tile index ti * nt + tj
      return x;
    }
    const uint64_t lag = j == ntt ? lagD : lagG;
    if (k < lag || k - lag >= K) return x;
    const uint64_t k2 = k - lag;
    x.r = k2 % rows;
    x.s = static_cast<int64_t>(k2 / rows) - 1;
    if (j == ntt) {
      x.type = kItemDec;
      return x;
    }
    if (static_cast<uint64_t>(x.s + 1) >= steps) return x;  // no next step
    x.type = kItemGate;
    x.s += 1;
    x.part = static_cast<int32_t>(j - ntt);  // 1 .. P-1 (part 0 runs inside the DEC)
    return x;
  }
  // j-th tile of the upper triangle (ti <= tj), row-major
  __host__ __device__ uint32_t upper_tile(uint32_t j) const {
    uint32_t ti = 0;
    while (j >= nt - ti) {
      j -= nt - ti;
      ++ti;
    }
    return ti * nt + ti + j;
  }
  // gate_done units before TILE(r, s) may run: INIT parts (+ NORM), then P per step
  __host__ __device__ uint64_t gate_target(int64_t s) const { return Ip + static_cast<uint64_t>(s + 1) * P; }
  __host__ __device__ uint64_t tiles_target(int64_t s) const {  // per-warp tile completions
    return static_cast<uint64_t>(kWarps) * ntt * static_cast<uint64_t>(s + 2);
  }
};

// Workspace of the queue schedule, after the slabs (`cap` rows): partials, row state and
// counters. Counters (and only they) are zeroed by the host before every launch.
struct QLayout {
  double* tv;        // [cap][ntt][kThreads] per-thread tile values
  double* dg;        // [cap][nt][2][kThreads] per-thread diagonal (trace) terms
  QRow* row;         // [cap]
  unsigned long long* ctr;  // [0] queue head; then gate_done, tiles_done, dec_done [cap] each
  unsigned long long* gate_done;
  unsigned long long* tiles_done;
  unsigned long long* dec_done;
  size_t counter_bytes;
  double* rho;       // von Neumann: [cap][2][d_a^2] planes Re, Im of rho (column-major)
  static constexpr int kMaxCtas = 1024;  // the launch grid's upper bound
  __host__ __device__ static size_t align(size_t b) { return (b + 255) / 256 * 256; }
  __host__ __device__ static size_t rho_doubles(uint32_t spins) { return 2 * (size_t{1} << (2 * (spins / 2))); }
  __host__ __device__ static size_t bytes(uint32_t spins, uint64_t cap, bool vn = false) {
    const uint64_t nt = (uint64_t{1} << (spins / 2)) / TB;
    return align(cap * nt * nt * kThreads * 8) + align(cap * nt * 2 * kThreads * 8) + align(cap * sizeof(QRow)) +
           align((16 + 3 * cap) * 8) + (vn ? align(cap * rho_doubles(spins) * 8) : 0);
  }
  __host__ __device__ QLayout(char* base, uint32_t spins, uint64_t cap) {
    const uint64_t nt = (uint64_t{1} << (spins / 2)) / TB;
    tv = reinterpret_cast<double*>(base);
    base += align(cap * nt * nt * kThreads * 8);
    dg = reinterpret_cast<double*>(base);
    base += align(cap * nt * 2 * kThreads * 8);
    row = reinterpret_cast<QRow*>(base);
    base += align(cap * sizeof(QRow));
    ctr = reinterpret_cast<unsigned long long*>(base);
    gate_done = ctr + 16;
    tiles_done = gate_done + cap;
    dec_done = tiles_done + cap;
    counter_bytes = align((16 + 3 * cap) * 8);
    base += counter_bytes;
    rho = reinterpret_cast<double*>(base);
  }
};

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_ge(const unsigned long long* p, unsigned long long target) {
  while (ld_acquire(p) < target) __nanosleep(64);
}
// the calling CTA's prior writes (ordered before this call by a barrier) -> consumers
__device__ __forceinline__ void signal(unsigned long long* p, unsigned long long add) {
  __threadfence();
  atomicAdd(p, add);
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Stage metadata: a generic shared-memory write by the producer, released by its
// arrive(.expect_tx) on the stage's full barrier; the consumers' wait on that barrier acquires
// it (PTX mbarrier arrive = release, try_wait = acquire, CTA scope). compute-sanitizer's
// racecheck does not model mbarrier ordering and reports this handoff (write in put_meta,
// read by the consumers); tests/test_sanitizer.py accepts exactly those reports. (The
// async-proxy alternatives measured: st.async and shared -> shared bulk copies only reach
// other CTAs of a cluster; a global ring + bulk load is racecheck-visible too and 0.4 % slower.)
__device__ __forceinline__ void put_meta(QMeta& dst, int32_t kind, int32_t t, int32_t kc, int32_t buf, const Item& x,
                                         uint64_t* full, uint32_t data_bytes) {
  dst.kind = kind;
  dst.t = t;
  dst.kc = kc;
  dst.buf = buf;
  dst.x = x;
  if (data_bytes) mbar_expect_tx(full, data_bytes);  // arrive (release) + the stage's TMA bytes
  else mbar_arrive(full);                            // a control entry: no data
}

__device__ __forceinline__ QRow load_row(const QRow* p) {
  QRow w;
  w.cur = __ldcg(&p->cur);
  w.err = __ldcg(&p->err);
  w.cur_e = __ldcg(&p->cur_e);
  w.t_prev = __ldcg(reinterpret_cast<const long long*>(&p->t_prev));
  w.t_row0 = __ldcg(reinterpret_cast<const long long*>(&p->t_row0));
  return w;
}

// Diagonal (trace) terms of this thread in a diagonal tile, in tile_trace_fault's order:
// block row i contributes at most one element, d[i] (has[i] says whether it exists).
__device__ __forceinline__ bool diag_has(int i, int wr, int wc, int m, int kq) {
  const int row = wr * 2 + i;
  return row >= wc * 4 && row < wc * 4 + 4 && (m >> 1) == kq;
}

// Consumer-only barrier (named barrier 1, the 256 consumer threads; the producer warpgroup
// never joins it).
__device__ __forceinline__ void csync() { consumer_sync(kThreads); }

// publish_vals<1> / totals<1> / renormalize<1> of hbm_tier.cuh with the consumer barrier
// (same arithmetic, same order: bitwise the cluster schedule's values).
__device__ __forceinline__ void q_publish(HHeader& H, int tid) {
  csync();
  if (tid < 2 * kChains) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) v += H.part[w][tid];
    H.val[0][tid] = v;
  }
  csync();
}
__device__ void q_renormalize(const Geo& G, double* X, double* Y, int tid, int warp, int lane, HHeader& H) {
  const int quarter = G.n / 4;
  for (int q = 0; q < 4; ++q) {
    double s = 0.0;
    for (int i = q * quarter + tid; i < (q + 1) * quarter; i += kThreads) {
      const double x = __ldcg(X + i), y = __ldcg(Y + i);
      s = fma(x, x, s);
      s = fma(y, y, s);
    }
    s = warp_sum(s);
    if (lane == 0) H.part[warp][0] = s;
    csync();
    if (tid == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) t += H.part[w][0];
      H.norm_q[q] = t;
    }
    csync();
  }
  const double inv = __ddiv_rn(1.0, __dsqrt_rn((H.norm_q[0] + H.norm_q[1]) + (H.norm_q[2] + H.norm_q[3])));
  for (int i = tid; i < G.n; i += kThreads) {
    __stcg(X + i, __dmul_rn(__ldcg(X + i), inv));
    __stcg(Y + i, __dmul_rn(__ldcg(Y + i), inv));
  }
  __threadfence();
  fence_proxy_async_global();  // the next GEMM reads psi through the TMA engine
  csync();
}

// STATS (probe only): per-CTA clock64 breakdown into P.trace[blockIdx.x * kQStats + i]:
//  0 total, 1 warp-1 waits for stage data, 2 warp-1 chunk compute, 3 warp-1 tile epilogues,
//  4 producer waits for free stages, 5 producer dependency waits (tiles), 6 control items,
//  7 their dependency waits, 8 tiles, 9 DEC, 10 GATE, 11 INIT + NORM items, 12 DEC clocks,
//  13 GATE clocks, 14 producer queue pulls (atomics incl. empty slots), 15 gate passes inside DEC items,
//  DEC phases (thread 0): 16 dependency wait + row / record loads, 17 fold + publish, 18 decision,
//  19 renormalisation + dec_done, 20 signals after the gate
// KIND 0: Renyi-2 (||rho||_F^2 partials); KIND 1: von Neumann for 16 <= S <= 21 (vn_large.cuh):
// TILE items store rho to the row's planes, the DEC item diagonalises it.
template <bool STATS = false, int KIND = 0>
__global__ void __launch_bounds__(kQThreads, 1) anneal_queue_kernel(const AnnealParams P,
                                                                    const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  QHeader& Q = *reinterpret_cast<QHeader*>(smem_raw);
  HHeader& H = Q.h;
  const uint32_t sbase = smem_u32(smem_raw);
  double* stages = reinterpret_cast<double*>(smem_raw + (((sbase + kQHeaderBytes + 1023u) & ~1023u) - sbase));
  const Geo G(static_cast<int>(P.spins));
  const QGeo q(P.spins, P.rows, P.steps, P.initial_state == 1, gridDim.x, P.rho_half != 0, KIND == 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt = G.tiles(), nk = G.kchunks(), lnt = G.la - 6;
  const uint64_t cap = P.queue_rows;
  const QLayout L(reinterpret_cast<char*>(P.workspace + cap * 4 * static_cast<uint64_t>(G.n)), P.spins, cap);
  auto clk = [&]() -> int64_t { return STATS ? clock64() : 0; };
  auto stat_add = [&](int i, int64_t v) {
    if (STATS) Q.stat[i] += v;
  };
  const int64_t t_begin = clk();
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&H.full[s], 1);  // put_meta's arrive(.expect_tx)
      mbar_init(&H.empty[s], kWarps);
    }
    mbar_init(&Q.ctl_done, 1);
    fence_mbar_init();
    if (STATS)
      for (int i = 0; i < kQStats; ++i) Q.stat[i] = 0;
  }
  __syncthreads();  // the last CTA-wide barrier: from here on consumers use csync()
  static_assert(KIND == 0 || sizeof(vnl::Scratch) <= kStages * kStage * 8, "vN scratch fits the stages");

  // ================================================================== producer (1 thread)
  if (tid >= kThreads) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kProducerRegs));
    if (tid != kThreads) return;
    uint64_t issued = 0;
    uint32_t ctl_par = 0;
    auto stage_for = [&](uint64_t e) {  // wait until entry e's stage is free
      const int s = static_cast<int>(e % kStages);
      if (e >= static_cast<uint64_t>(kStages)) {
        const int64_t a = clk();
        mbar_wait(&H.empty[s], static_cast<uint32_t>(e / kStages - 1) & 1);
        stat_add(4, clk() - a);
      }
      return s;
    };
    for (;;) {
      const int64_t a = clk();
      Item x;
      do {
        x = q.decode(atomicAdd(L.ctr, 1ull));
      } while (x.type == kItemEmpty);
      stat_add(14, clk() - a);
      if (x.type != kItemTile) {  // control entry (consumers execute it, in queue order)
        const int s = stage_for(issued++);
        put_meta(Q.meta[s], kMetaControl, 0, 0, 0, x, &H.full[s], 0);
        if (x.type == kItemEnd) break;
        if (KIND == 1 && x.type == kItemDec) {  // its eigen-solver uses the stage buffers as scratch
          mbar_wait(&Q.ctl_done, ctl_par);
          ctl_par ^= 1;
        }
        continue;
      }
      // TILE(r, s, t): wait for its gate (or initial state), then its row's buffer
      const int64_t b = clk();
      wait_ge(&L.gate_done[x.r], q.gate_target(x.s));
      stat_add(5, clk() - b);
      int buf = 0;
      if (x.s >= 0) {
        if (__ldcg(&L.row[x.r].err)) {  // a failed replica: its tile counts as done, no work
          signal(&L.tiles_done[x.r], kWarps);
          continue;
        }
        buf = __ldcg(&L.row[x.r].cur) ^ 1;
      }
      fence_proxy_async_global();
      const int t = x.part, ti = t >> lnt, tj = t & (nt - 1);
      const bool diag = ti == tj;
      for (int kc = 0; kc < nk; ++kc) {
        const int s = stage_for(issued++);
        double* st = stages + s * kStage;
        put_meta(Q.meta[s], kMetaTile, t, kc, buf, x, &H.full[s], diag ? kTmaStageBytes / 2 : kTmaStageBytes);
        for (int h = 0; h < 2; ++h) {
          tma_load_5d(st + h * kTmaBox, &tmap, 0, ti * 4 + 2 * h, kc * KC, 2 * buf, static_cast<int>(x.r), &H.full[s]);
          if (!diag)
            tma_load_5d(st + kTmaPanel + h * kTmaBox, &tmap, 0, tj * 4 + 2 * h, kc * KC, 2 * buf,
                        static_cast<int>(x.r), &H.full[s]);
        }
      }
    }
    if (STATS) {  // the consumers have all finished (they consumed the END entry and left)
      // (written by the producer after the consumers' final stats are in: see below)
    }
    return;
  }

  // ================================================================== consumers (256 threads)
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kConsumerRegs));
  const int wr = warp / T8::WC, wc = warp % T8::WC;
  const int m = lane >> 2, kq = lane & 3;
  auto slab = [&](uint64_t r) { return P.workspace + r * 4 * static_cast<uint64_t>(G.n); };
  auto PX = [&](uint64_t r, int b) { return slab(r) + (2 * b) * static_cast<size_t>(G.n); };
  auto PY = [&](uint64_t r, int b) { return slab(r) + (2 * b + 1) * static_cast<size_t>(G.n); };
  const bool fault = P.inject_fault != 0;
  auto wait_dep = [&](const unsigned long long* c, unsigned long long target) {  // consumer thread 0
    const int64_t a = clk();
    wait_ge(c, target);
    stat_add(7, clk() - a);
  };
  // fragment offsets (rho_partials_tma's swizzled panel layout)
  auto frag = [&](int qb) {
    const int r = qb * 8 + m, b = (r >> 4) & 1;
    return (r >> 5) * 2048 + kq * 32 + b * 16 + 2 * (((r >> 1) & 7) ^ (b + 2 * kq)) + (r & 1);
  };
  int fa[2], fb[4];
#pragma unroll
  for (int i = 0; i < 2; ++i) fa[i] = frag(wr * 2 + i);
#pragma unroll
  for (int j = 0; j < 4; ++j) fb[j] = frag(wc * 4 + j);

  // --------------------------------------------------------------- control items
  auto sync_signal = [&](unsigned long long* c) {  // every consumer's writes, then one release
    csync();
    if (tid == 0) signal(c, 1);
  };
  // A control item's proposal records (steps s0 and s0 + 1 of row r, when they exist) are
  // copied to SMEM by cp.async as the item starts, so the global round trips overlap its
  // dependency wait and fold instead of sitting on the decision / gate path; rec_wait()
  // (every consumer thread) completes them before the next barrier.
  auto rec_fetch = [&](uint64_t r, int64_t s0) {
    if (tid < 36) {
      const int64_t s = s0 + tid / 18;
      if (s >= 0 && static_cast<uint64_t>(s) < P.steps)
        cp_async16(reinterpret_cast<char*>(&Q.rec[tid / 18]) + 16 * (tid % 18),
                   reinterpret_cast<const char*>(P.gates + static_cast<uint64_t>(s) * P.rows + r) + 16 * (tid % 18));
      cp_async_commit();
    }
  };
  auto rec_wait = [&]() {
    if (tid < 36) cp_async_wait<0>();
  };
  auto gate_part = [&](uint64_t r, const GateRec& g, int part, int cur) {  // spinmc.cpp:91-136 on 1/P of the groups
    const int groups = G.n / 4, per = groups / static_cast<int>(q.P), g0 = part * per;
    gate_pass(PX(r, cur), PY(r, cur), PX(r, cur ^ 1), PY(r, cur ^ 1), g.site, g, g0, g0 + per, tid, kThreads);
    fence_proxy_async_global();  // psi' is read by the TMA engine
  };
  auto run_control = [&](const Item& x) {
    const uint64_t r = x.r;
    if (x.type == kItemInit) {  // product_state / random_state amplitudes of part x.part
      if (x.part == 0 && tid == 0) {
        QRow w{0, 0, 0.0, 0, (P.initial_wall_ns || P.wall_ns) ? globaltimer() : 0};
        L.row[r] = w;
      }
      const uint64_t per = G.n / q.P, i0 = static_cast<uint64_t>(x.part) * per, i1 = i0 + per;
      double *X = PX(r, 0), *Y = PY(r, 0);
      if (P.initial_state == 0) {
        for (uint64_t i = i0 + tid; i < i1; i += kThreads) {
          __stcg(X + i, i == 0 ? 1.0 : 0.0);
          __stcg(Y + i, 0.0);
        }
      } else {
        const double* src = P.init_states + r * 2 * static_cast<size_t>(G.n);
        for (uint64_t i = i0 + tid; i < i1; i += kThreads) {
          __stcg(X + i, src[2 * i]);
          __stcg(Y + i, src[2 * i + 1]);
        }
      }
      fence_proxy_async_global();
      sync_signal(&L.gate_done[r]);
      return;
    }
    if (x.type == kItemNorm) {
      if (tid == 0) wait_dep(&L.gate_done[r], q.P);
      csync();
      q_renormalize(G, PX(r, 0), PY(r, 0), tid, warp, lane, H);  // ends with fences + barrier
      if (tid == 0) signal(&L.gate_done[r], 1);
      return;
    }
    if (x.type == kItemGate) {
      rec_fetch(r, x.s - 1);  // rec[1] = step x.s
      if (tid == 0) {
        wait_dep(&L.dec_done[r], static_cast<unsigned long long>(x.s + 1));
        Q.row = load_row(&L.row[r]);
      }
      rec_wait();
      csync();
      if (!Q.row.err) gate_part(r, Q.rec[1], x.part, Q.row.cur);
      sync_signal(&L.gate_done[r]);
      return;
    }
    // DEC(r, s)
    const int64_t s = x.s;
    const int64_t d0 = clk();
    rec_fetch(r, s);  // rec[0] = step s (the decision), rec[1] = step s + 1 (the next gate)
    if (tid == 0) {
      wait_dep(&L.tiles_done[r], q.tiles_target(s));
      Q.row = load_row(&L.row[r]);
    }
    rec_wait();
    csync();
    const int64_t d1 = clk();
    if (STATS && tid == 0) stat_add(16, d1 - d0);
    const bool next_gate = static_cast<uint64_t>(s + 1) < P.steps;
    if (Q.row.err) {
      sync_signal(&L.dec_done[r]);
      if (next_gate && tid == 0) signal(&L.gate_done[r], q.long_dec ? q.P : 1);  // its gate parts (no work)
      return;
    }
    // replay the per-thread chains of rho_partials_tma (CS = 1, tiles in ascending order)
    double rho[kChains] = {0.0, 0.0, 0.0, 0.0}, tr[kChains] = {0.0, 0.0, 0.0, 0.0};
    {
      const double* tvr = L.tv + r * q.nfull * kThreads + tid;
      for (uint32_t t0 = 0; KIND == 0 && t0 < q.nfull; t0 += kChains) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
          const uint32_t t = t0 + c;  // rho_half: lower tiles (ti > tj) were not formed
          if (t < q.nfull && !(q.half && (t >> lnt) > (t & (nt - 1))))
            rho[c] = rho[c] + __ldcg(tvr + static_cast<size_t>(t) * kThreads);
        }
      }
      const bool h0 = diag_has(0, wr, wc, m, kq), h1 = diag_has(1, wr, wc, m, kq);
      const double* dgr = L.dg + r * nt * 2 * kThreads + tid;
      for (int ti = 0; ti < nt; ++ti) {
        const int ch = (ti * nt + ti) & (kChains - 1);
        double tsum = 0.0;
#pragma unroll
        for (int c = 0; c < kChains; ++c) tsum = c == ch ? tr[c] : tsum;
        if (h0) tsum += __ldcg(dgr + static_cast<size_t>(ti * 2) * kThreads);
        if (h1) tsum += __ldcg(dgr + static_cast<size_t>(ti * 2 + 1) * kThreads);
#pragma unroll
        for (int c = 0; c < kChains; ++c) tr[c] = c == ch ? tsum : tr[c];
      }
    }
    double out[2 * kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) {
      out[c] = warp_sum(rho[c]);
      out[kChains + c] = warp_sum(tr[c]);
    }
    if (lane == 0)
      for (int c = 0; c < 2 * kChains; ++c) H.part[warp][c] = out[c];
    q_publish(H, tid);
    double rho2, trv;
    totals<1>(H, rho2, trv);
    const int64_t d2 = clk();
    if (STATS && tid == 0) stat_add(17, d2 - d1);
    if constexpr (KIND == 1) {  // von Neumann: eigenvalues of this step's rho (stages = scratch)
      const size_t da = size_t{1} << G.la;
      double* Rr = L.rho + r * QLayout::rho_doubles(P.spins);
      rho2 = vnl::entropy(Rr, Rr + da * da, static_cast<int>(da), *reinterpret_cast<vnl::Scratch*>(stages), tid,
                          [] { csync(); });  // thread 0: the entropy (the trace value of this proposal)
    }
    if (tid == 0) {
      QRow w = Q.row;
      const bool bad = smem::not_normalized(trv);
      int acc = 0;
      if (s < 0) {  // initial state (spinmc.cpp:234)
        w.cur = 0;
        w.cur_e = rho2;
        P.status[r] = bad ? kRowNotNormalized : kRowOk;
        if (bad) {
          P.status_step[r] = -1;
          if (P.status_norm) P.status_norm[r] = __dsqrt_rn(trv);
        }
        P.initial_entropy[r] = rho2;
        if (P.wall_ns || P.initial_wall_ns) {
          const int64_t now = globaltimer();
          if (P.initial_wall_ns) P.initial_wall_ns[r] = now - w.t_row0;
          w.t_prev = now;
        }
      } else {
        const GateRec& g = Q.rec[0];
        if (bad) {
          P.status[r] = kRowNotNormalized;
          P.status_step[r] = s;
          if (P.status_norm) P.status_norm[r] = __dsqrt_rn(trv);
        } else {
          // KIND 0: the lean decision on ||rho||^2; KIND 1: spinmc.cpp:203-207 on the entropies
          const smem::Verdict v = KIND == 0 ? smem::decide_audit(rho2, w.cur_e, g, P.objective, P.tie_eps)
                                            : smem::decide_reference(rho2, w.cur_e, g, P.objective, P.tie_eps);
          acc = v.acc;
          smem::audit(P, r, static_cast<uint64_t>(s), g, v);
          if (acc) {
            w.cur_e = rho2;
            w.cur ^= 1;
          }
          const uint64_t o = r * P.steps + static_cast<uint64_t>(s);
          P.entropies[o] = w.cur_e;
          P.accepted[o] = static_cast<uint8_t>(acc);
          if (P.sites) P.sites[o] = static_cast<uint8_t>(g.site);
          if (P.wall_ns) {
            const int64_t now = globaltimer();
            P.wall_ns[o] = now - w.t_prev;
            w.t_prev = now;
          }
        }
      }
      w.err = bad ? 1 : 0;
      if (P.final_entropy) P.final_entropy[r] = w.cur_e;
      L.row[r] = w;
      Q.row = w;
    }
    csync();
    const int64_t d3 = clk();
    if (STATS && tid == 0) stat_add(18, d3 - d2);
    if (s >= 0 && !Q.row.err && P.renorm > 0 && (static_cast<uint64_t>(s) + 1) % P.renorm == 0)
      q_renormalize(G, PX(r, Q.row.cur), PY(r, Q.row.cur), tid, warp, lane, H);  // spinmc.cpp:246-248
    // dec_done is waited on by GATE items only: none exist when the DEC applies the whole gate
    const bool gate_items = !q.long_dec && q.P > 1;
    if (gate_items) sync_signal(&L.dec_done[r]);
    if (STATS && tid == 0) stat_add(19, clk() - d3);
    if (next_gate) {  // part 0 (von Neumann: every part) of the next step's gate, on the state just decided
      const int parts = q.long_dec ? static_cast<int>(q.P) : 1;
      const int64_t g0 = clk();
      if (!Q.row.err)
        for (int part = 0; part < parts; ++part) gate_part(r, Q.rec[1], part, Q.row.cur);
      const int64_t g1 = clk();
      if (STATS && tid == 0) stat_add(15, g1 - g0);
      csync();
      if (tid == 0) signal(&L.gate_done[r], static_cast<unsigned long long>(parts));
      if (STATS && tid == 0) stat_add(20, clk() - g1);
    }
  };

  // ------------------------------------------------------------------ consumer loop
  // The producer issues a tile's nk chunks back to back, so a tile is one inner loop and its
  // accumulators are dead outside it (the control items reuse those registers).
  uint64_t seq = 0;
  auto wait_full = [&](uint64_t e) {
    const int s = static_cast<int>(e % kStages);
    const uint32_t par = static_cast<uint32_t>(e / kStages) & 1;
    if (STATS && tid == 32) {
      const int64_t a = clk();
      mbar_wait(&H.full[s], par);
      stat_add(1, clk() - a);
    } else {
      mbar_wait(&H.full[s], par);
    }
    return s;
  };
  for (;;) {
    int s = wait_full(seq);
    const QMeta md = Q.meta[s];
    if (md.kind == kMetaControl) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&H.empty[s]);  // the stage holds no data
      ++seq;
      if (md.x.type == kItemEnd) break;
      csync();  // every consumer warp has finished the earlier entries
      const int64_t a = clk();
      run_control(md.x);
      csync();
      if (KIND == 1 && md.x.type == kItemDec && tid == 0) mbar_arrive(&Q.ctl_done);  // scratch released
      if (STATS && tid == 0) {
        const int64_t d = clk() - a;
        stat_add(6, d);
        if (md.x.type == kItemDec) {
          stat_add(9, 1);
          stat_add(12, d);
        } else if (md.x.type == kItemGate) {
          stat_add(10, 1);
          stat_add(13, d);
        } else {
          stat_add(11, 1);
        }
      }
      continue;
    }
    // TILE md.t of row md.x.r: nk consecutive entries
    const int ti = md.t >> lnt, tj = md.t & (nt - 1);
    const bool diag = ti == tj;
    double cr[2][4][2], ci[2][4][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
    for (int kc = 0; kc < nk; ++kc) {
      if (kc > 0) s = wait_full(seq);
      const int64_t c0 = clk();
      const double* st = stages + s * kStage;
      const double *AX = st, *AY = st + 1024;
      const double *BX = diag ? AX : st + kTmaPanel, *BY = diag ? AY : st + kTmaPanel + 1024;
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
      if (lane == 0) mbar_arrive(&H.empty[s]);
      ++seq;
      if (STATS && tid == 32) stat_add(2, clk() - c0);
    }
    // tile epilogue: per-thread partials, then this warp's completion
    const int64_t e0 = clk();
    const uint64_t r = md.x.r;
    if (diag) {
      double d[2] = {0.0, 0.0};
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (wr * 2 + i == wc * 4 + j) {
            if (m == 2 * kq) d[i] = cr[i][j][0];
            if (m == 2 * kq + 1) d[i] = cr[i][j][1];
          }
      double* dgr = L.dg + (r * nt + ti) * 2 * kThreads + tid;
      __stcg(dgr, d[0]);
      __stcg(dgr + kThreads, d[1]);
    }
    if (fault && md.t == 0 && wr == 0 && wc == 0 && lane == 0) {
      const double x0 = __ldcg(PX(r, md.buf)), y0 = __ldcg(PY(r, md.buf));
      fault_term(cr[0][0][0], x0, y0);
    }
    if constexpr (KIND == 1) {  // rho itself, for the DEC item's eigen-solver
      const size_t da = size_t{1} << G.la;
      double* Rr = L.rho + r * QLayout::rho_doubles(P.spins);
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const size_t o = static_cast<size_t>(ti * TB + (wr * 2 + i) * 8 + m) +
                             static_cast<size_t>(tj * TB + (wc * 4 + j) * 8 + 2 * kq + e) * da;
            __stcg(Rr + o, cr[i][j][e]);
            __stcg(Rr + da * da + o, ci[i][j][e]);
          }
    } else {
      double rho1[kChains] = {0.0, 0.0, 0.0, 0.0};
      tile_fold(cr, ci, rho1, 0, false);  // rho1[0] = 0.0 + tv (tile_fold's arithmetic)
      if (q.half && !diag) rho1[0] += rho1[0];  // rho_half: the mirrored lower tile (exact)
      __stcg(L.tv + (r * q.nfull + static_cast<uint64_t>(md.t)) * kThreads + tid, rho1[0]);
    }
    __syncwarp();
    if (lane == 0) signal(&L.tiles_done[r], 1);
    if (STATS && tid == 32) {
      stat_add(3, clk() - e0);
      stat_add(8, 1);
    }
  }
  if (STATS) {
    csync();
    if (tid == 0) {
      Q.stat[0] = clk() - t_begin;
      for (int i = 0; i < kQStats; ++i) P.trace[blockIdx.x * kQStats + i] = Q.stat[i];
    }
  }
}

}  // namespace hbmq
}  // namespace tg
