// zgemm.cu — fixed-size batched complex GEMM on DMMA.8x8x4: the device side of the GEMM
// batcher (VirtualDevice::batched_gemm, exec.cpp:144-221; per-entry math linalg.cpp:79-113:
// out = alpha*A*B + beta*C, column-major interleaved complex128).
//
// Persistent: one CTA per SM walks the work items (entry e, 64x64 output tile)
// w = blockIdx.x, blockIdx.x + gridDim.x, ...; K streams in chunks of 32 through a 3-stage
// pipeline that runs on across work items (the next item's first chunks load during the
// current item's last ones), the HBM tier's scheme (hbm_tier.cuh). Two stagings:
// zgemm_tma_kernel (m, k multiples of 8: TMA tensor copies, mbarriers; 8 warps of 16x32 or,
// for K >= 128, 16 warps of 16x16) and zgemm_kernel below (any shape: per-thread cp.async,
// 8 warps of 16x32 = 2x4 blocks of 8x8). Both give every output element the same DMMA
// sequence, so they agree bitwise. Operands stay interleaved complex in SMEM
// (cp.async copies one 16-byte element, no de-interleave pass): A as [k][i] with pitch 66
// elements, B as [j][k] with pitch 36; a fragment is one LDS.128 (re, im), and the pitches
// (2 and 4 mod 8 elements) make every quarter-warp of 8 such loads bank-conflict free.
// Complex product by real split: Re = Ar Br - Ai Bi, Im = Ar Bi + Ai Br (4 DMMA per block
// per k-step of 4). Edges (m, n, k not multiples of the tile) are zero-filled by the copy.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "smem_tier.cuh"
#include "tg_internal.h"

namespace tg {
namespace {

constexpr int ZT = 64, ZK = 32;
constexpr int PA = ZT + 2;  // A stage [k][i]: pitch 66 elements (16 B each)
constexpr int PB = ZK + 4;  // B stage [j][k]: pitch 36
constexpr int ZThreads = 256, ZStages = 3;
constexpr int StageA = ZK * PA, StageB = ZT * PB;  // elements
constexpr int StageElems = StageA + StageB;

__device__ __forceinline__ void cp_async16_zfill(void* s, const void* g, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(s)), "l"(g), "r"(valid ? 16 : 0)
               : "memory");
}

struct ZArgs {
  int m, n, k, tm, tn, nk;
  double ar, ai, br, bi;
  const double* A;
  int64_t sA;
  const double* B;
  int64_t sB;
  const double* C;
  int64_t sC;
  double* out;
  int64_t sO;
  int fault;
  int64_t items;
};

__global__ void __launch_bounds__(ZThreads, 1) zgemm_kernel(const ZArgs P) {
  extern __shared__ __align__(16) double2 zsm[];  // ZStages x {A [k][i], B [j][k]}
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp >> 1, wc = warp & 1;  // warp grid 4 x 2
  const int mm = lane >> 2, kq = lane & 3;
  const int64_t mine = P.items > blockIdx.x ? (P.items - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t total = mine * P.nk;
  // Work-item cursors (the producer runs two chunks ahead of the consumer): item w -> entry
  // e = w / (tm*tn), tile t = w % (tm*tn); decomposed once per item, never per chunk (64-bit
  // divisions per chunk would sit on every warp's issue path between the DMMA phases).
  struct Cursor {
    int64_t w;
    int kc, i0, j0;
    const double *a, *b;
  };
  auto set_item = [&](Cursor& q, int64_t w) {
    q.w = w;
    q.kc = 0;
    if (w < P.items) {
      const int64_t e = w / (P.tm * P.tn);
      const int t = static_cast<int>(w - e * P.tm * P.tn);
      q.i0 = (t / P.tn) * ZT;
      q.j0 = (t % P.tn) * ZT;
      q.a = P.A + 2 * P.sA * e;
      q.b = P.B + 2 * P.sB * e;
    }
  };
  auto advance = [&](Cursor& q) {
    if (++q.kc == P.nk) set_item(q, q.w + gridDim.x);
  };
  Cursor prod, cons;
  set_item(prod, blockIdx.x);
  set_item(cons, blockIdx.x);
  int pslot = 0, cslot = 0;  // stage slots (it % ZStages) of producer and consumer, in 32 bits
  // Stage copies of the producer's (item, chunk): thread tid copies A elements
  // (i0 + ii, k0 + kk0 + 4u) and B elements (k0 + kb, j0 + jb0 + 8u), u = 0..7 (coalesced:
  // consecutive threads take consecutive rows of one column). Addresses are set up once per
  // chunk; in the main loop the 16 copies are spread 2 per k-step.
  const int ii = tid & (ZT - 1), kk0 = tid >> 6;   // A
  const int kb_ = tid & (ZK - 1), jb0 = tid >> 5;  // B
  struct Stage {
    const double *a, *b;
    int64_t astep, bstep;
    double2* st;
    bool arow_ok, bk_ok;
    int k0, j0;
  } ps{};
  auto prepare = [&]() {  // the producer's next stage
    ps.k0 = prod.kc * ZK;
    ps.j0 = prod.j0;
    const int gi = prod.i0 + ii, gka = ps.k0 + kk0, gkb = ps.k0 + kb_;
    ps.arow_ok = gi < P.m;
    ps.bk_ok = gkb < P.k;
    ps.a = prod.a + 2 * (static_cast<int64_t>(gi) + static_cast<int64_t>(gka) * P.m);
    ps.b = prod.b + 2 * (static_cast<int64_t>(gkb) + static_cast<int64_t>(prod.j0 + jb0) * P.k);
    ps.astep = 2 * 4 * static_cast<int64_t>(P.m);
    ps.bstep = 2 * 8 * static_cast<int64_t>(P.k);
    ps.st = zsm + pslot * StageElems;
  };
  auto copy_part = [&](int u) {  // copies u of the prepared stage
    const bool oka = ps.arow_ok && ps.k0 + kk0 + 4 * u < P.k;
    const bool okb = ps.bk_ok && ps.j0 + jb0 + 8 * u < P.n;
    cp_async16_zfill(ps.st + (kk0 + 4 * u) * PA + ii, oka ? ps.a + u * ps.astep : P.A, oka);
    cp_async16_zfill(ps.st + StageA + (jb0 + 8 * u) * PB + kb_, okb ? ps.b + u * ps.bstep : P.B, okb);
  };
  auto finish = [&]() {
    advance(prod);
    pslot = pslot == ZStages - 1 ? 0 : pslot + 1;
  };
  auto issue_all = [&](int64_t it) {  // prologue: a whole stage at once
    if (it < total) {
      prepare();
#pragma unroll
      for (int u = 0; u < 8; ++u) copy_part(u);
      finish();
    }
    cp_async_commit();
  };
  double cr[2][4][2], ci[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
  issue_all(0);
  issue_all(1);
  for (int64_t it = 0; it < total; ++it) {
    cp_async_wait<1>();          // this thread's copies of stage `it` landed
    __syncthreads();             // everyone's did; stage (it-1) % 3 is free
    const bool has_next = it + 2 < total;
    if (has_next) prepare();
    const double2* st = zsm + cslot * StageElems;
    cslot = cslot == ZStages - 1 ? 0 : cslot + 1;
    const double2* sa = st;
    const double2* sb = st + StageA;
#pragma unroll
    for (int kb = 0; kb < ZK; kb += 4) {
      if (has_next) copy_part(kb / 4);
      double xa[2], ya[2], yn[2], xb[4], yb[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double2 v = sa[(kb + kq) * PA + (wr * 2 + i) * 8 + mm];
        xa[i] = v.x;
        ya[i] = v.y;
        yn[i] = -v.y;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 v = sb[((wc * 4 + j) * 8 + mm) * PB + kb + kq];
        xb[j] = v.x;
        yb[j] = v.y;
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma(cr[i][j][0], cr[i][j][1], xa[i], xb[j]);
          dmma(cr[i][j][0], cr[i][j][1], yn[i], yb[j]);
          dmma(ci[i][j][0], ci[i][j][1], xa[i], yb[j]);
          dmma(ci[i][j][0], ci[i][j][1], ya[i], xb[j]);
        }
    }
    if (has_next) finish();
    cp_async_commit();
    if (cons.kc == P.nk - 1) {  // item epilogue
      const int64_t e = cons.w / (P.tm * P.tn);
      const int i0 = cons.i0, j0 = cons.j0;
      const double* a = cons.a;
      const double* b = cons.b;
      // fault hook (linalg.cpp:94): sign of the first term of element (0,0) flipped
      if (P.fault && i0 == 0 && j0 == 0 && wr == 0 && wc == 0 && lane == 0) {
        const double2 a00 = *reinterpret_cast<const double2*>(a);
        const double2 b00 = *reinterpret_cast<const double2*>(b);
        const double tr = __dsub_rn(__dmul_rn(a00.x, b00.x), __dmul_rn(a00.y, b00.y));
        cr[0][0][0] -= 2.0 * tr;
      }
      // out = alpha*sum + beta*C (linalg.cpp:98-101), reference operation order
      const double* c = P.C ? P.C + 2 * P.sC * e : nullptr;
      double* o = P.out + 2 * P.sO * e;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gi = i0 + (wr * 2 + i) * 8 + mm;
            const int gj = j0 + (wc * 4 + j) * 8 + 2 * kq + h;
            if (gi < P.m && gj < P.n) {
              const size_t idx = gi + static_cast<size_t>(gj) * P.m;
              double cvr = 0.0, cvi = 0.0;
              if (c) {
                const double2 v = *reinterpret_cast<const double2*>(c + 2 * idx);
                cvr = v.x;
                cvi = v.y;
              }
              const double sr = cr[i][j][h], si = ci[i][j][h];
              const double re = __dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(P.ar, sr), __dmul_rn(P.ai, si)),
                                                    __dmul_rn(P.br, cvr)),
                                          __dmul_rn(P.bi, cvi));
              const double im = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(P.ar, si), __dmul_rn(P.ai, sr)),
                                                    __dmul_rn(P.br, cvi)),
                                          __dmul_rn(P.bi, cvr));
              *reinterpret_cast<double2*>(o + 2 * idx) = make_double2(re, im);
            }
            cr[i][j][h] = 0.0;
            ci[i][j][h] = 0.0;
          }
    }
    advance(cons);
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------- TMA-staged variant
// Same items, warp tiling, DMMA order and epilogue; the stages are filled by TMA tensor
// copies (thread 0, two chunks ahead) with mbarrier full/empty tracking instead of
// per-thread cp.async + a CTA barrier per chunk. Requires m % 8 == 0 and k % 8 == 0 (a
// 128-B line is 8 complex elements of a column); tile edges are TMA out-of-bounds zeros.
//   A map: (16 doubles = 8 rows, m/8 row blocks, k columns, batch), box (16, 2, 32, 1): a
//          16-row x 32-k box; line L = 2k + b (b: 8-row block in the box), 128-B swizzle
//          permutes the 16-B elements of a line by L & 7. Panel = 4 boxes.
//   B map: (16 doubles = 8 k, k/8 blocks, n columns, batch), box (16, 4, 64, 1): the whole
//          32-k x 64-j panel; line L = 4j + kb8, elements permuted by L & 7.
// Every quarter-warp of fragment LDS.128 then reads 8 distinct 16-B slots of one 128-B
// bank window (A: row bit 0 ^ b and (row bits 1-2) ^ k; B: k bits 0-1 ^ kb8 and k bit 2 ^ j).
constexpr int TBoxA = 16 * 2 * ZK;                  // doubles per A box (16 rows)
constexpr int TPanel = 4 * TBoxA;                   // doubles per panel (64 rows / columns)
constexpr int TStage = 2 * TPanel;                  // A panel + B panel
constexpr uint32_t TStageBytes = TStage * 8;
static_assert(16 * 4 * ZT == TPanel, "B box = one panel");

// Warp grid WR x WC, each warp 16 rows x NB*8 columns: CTA tile (16 WR) x (8 NB WC).
//  <4, 2, 4, 3, 1>: 8 warps, 64x64 tiles, 1 CTA per SM (192 KB of stages);
//  <4, 4, 2, 3, 1>: 16 warps of 16x16: twice the warps per SMSP to hide the DMMA accumulator
//                   latency;
//  <2, 2, 2, 2, 3>: 4 warps, 32x32 tiles, 2 stages of 32 KB, 3 CTAs per SM — the shape of
//                   cuBLAS's z884 32x32x16 kernel: a CTA's epilogue overlaps the other CTAs'
//                   main loops (small K, where the epilogue weighs most).
// Every 8x8 output block sees the same DMMA sequence in all three (and in zgemm_kernel):
// results are bitwise equal.
// PROD: one extra warpgroup whose first thread issues the TMA stages (the consumer warps
// never leave the DMMA loop to issue).
// CREGS > 0 (with PROD): setmaxnreg rebalancing, consumers up to CREGS registers and the
// producer warpgroup 40, for shapes whose launch bound would otherwise cap the consumers.
template <int WR, int WC, int NB, int STAGES, int MINB, bool PROD = false, int CREGS = 0>
__global__ void __launch_bounds__(32 * WR * WC + (PROD ? 128 : 0), MINB) zgemm_tma_kernel(const ZArgs P, const __grid_constant__ CUtensorMap mapA,
                                                                      const __grid_constant__ CUtensorMap mapB) {
  constexpr int TM = 16 * WR, TN = 8 * NB * WC;
  constexpr int PanelA = WR * TBoxA, Stage = PanelA + 64 * TN;  // doubles
  constexpr uint32_t StageBytes = Stage * 8;
  extern __shared__ __align__(1024) unsigned char zraw[];
  const uint32_t sbase = smem_u32(zraw);
  double* stages = reinterpret_cast<double*>(zraw + (((sbase + 1023u) & ~1023u) - sbase));
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int wr = warp / WC, wc = warp % WC;
  const int mm = lane >> 2, kq = lane & 3;
  const int64_t mine = P.items > blockIdx.x ? (P.items - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int64_t total = mine * P.nk;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], WR * WC);  // one arrival per warp
    }
    fence_mbar_init();
  }
  __syncthreads();
  // fragment offsets: A block i of the warp (rows (2 wr + i) * 8 + mm: box wr, b = i),
  // B for k-steps kb (k block kb >> 3, bit 2 of k = (kb >> 2) & 1)
  int fa[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) fa[i] = wr * TBoxA + (2 * kq + i) * 16 + 2 * (mm ^ (i + 2 * kq));
  const int fb0 = (wc * NB * 8 + mm) * 64;  // column j = (wc * NB + jj) * 8 + mm, + jj * 512
  // epilogue fast path: (1*sr - 0*si + 0*0) - 0*0 == sr + 0.0 bit for bit (the sum maps -0 to
  // +0 as the full formula does); skips 13 FP64 ops per element that contend with the DMMAs
  // (+0.0 exactly: a -0.0 alpha.im or beta would keep a -0 result)
  const bool unit = P.ar == 1.0 && __double_as_longlong(P.ai) == 0 && __double_as_longlong(P.br) == 0 &&
                    __double_as_longlong(P.bi) == 0 && P.C == nullptr;
  struct Cursor {
    int64_t w, e;
    int kc, i0, j0;
  };
  auto set_item = [&](Cursor& q, int64_t w) {
    q.w = w;
    q.kc = 0;
    if (w < P.items) {
      q.e = w / (P.tm * P.tn);
      const int t = static_cast<int>(w - q.e * P.tm * P.tn);
      q.i0 = (t / P.tn) * TM;
      q.j0 = (t % P.tn) * TN;
    }
  };
  auto advance = [&](Cursor& q) {
    if (++q.kc == P.nk) set_item(q, q.w + gridDim.x);
  };
  Cursor prod, cons;
  set_item(prod, blockIdx.x);
  set_item(cons, blockIdx.x);
  auto issue = [&](int64_t it) {  // thread 0: chunk it (= prod's) into stage it % STAGES
    const int s = static_cast<int>(it % STAGES);
    if (it >= STAGES) mbar_wait(&empty[s], static_cast<uint32_t>(it / STAGES - 1) & 1);
    double* st = stages + s * Stage;
    mbar_expect_tx(&full[s], StageBytes);
    const int e = static_cast<int>(prod.e), k0 = prod.kc * ZK;
#pragma unroll
    for (int h = 0; h < WR; ++h) tma_load_4d(st + h * TBoxA, &mapA, 0, prod.i0 / 8 + 2 * h, k0, e, &full[s]);
    tma_load_4d(st + PanelA, &mapB, 0, k0 / 8, prod.j0, e, &full[s]);
    advance(prod);
  };
  double cr[2][NB][2], ci[2][NB][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) cr[i][j][0] = cr[i][j][1] = ci[i][j][0] = ci[i][j][1] = 0.0;
  if constexpr (PROD) {
    if (tid >= 32 * WR * WC) {
      if constexpr (CREGS > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
      if (tid == 32 * WR * WC)
        for (int64_t it = 0; it < total; ++it) issue(it);
      return;
    }
    if constexpr (CREGS > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(CREGS));
  } else if (tid == 0) {
    for (int64_t it = 0; it < STAGES - 1 && it < total; ++it) issue(it);
  }
  for (int64_t it = 0; it < total; ++it) {
    const int s = static_cast<int>(it % STAGES);
    if (!PROD && tid == 0 && it + STAGES - 1 < total) issue(it + STAGES - 1);
    mbar_wait(&full[s], static_cast<uint32_t>(it / STAGES) & 1);
    const double* sa = stages + s * Stage;
    const double* sb = sa + PanelA;
#pragma unroll
    for (int kb = 0; kb < ZK; kb += 4) {
      double xa[2], ya[2], yn[2], xb[NB], yb[NB];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double2 v = *reinterpret_cast<const double2*>(sa + fa[i] + kb * 32);
        xa[i] = v.x;
        ya[i] = v.y;
        yn[i] = -v.y;
      }
      const int kblk = kb >> 3, hb = (kb >> 2) & 1;
      const int fbk = fb0 + kblk * 16 + 2 * ((kq ^ kblk) + 4 * (hb ^ (mm & 1)));
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const double2 v = *reinterpret_cast<const double2*>(sb + fbk + j * 512);
        xb[j] = v.x;
        yb[j] = v.y;
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          dmma(cr[i][j][0], cr[i][j][1], xa[i], xb[j]);
          dmma(cr[i][j][0], cr[i][j][1], yn[i], yb[j]);
          dmma(ci[i][j][0], ci[i][j][1], xa[i], yb[j]);
          dmma(ci[i][j][0], ci[i][j][1], ya[i], xb[j]);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (cons.kc == P.nk - 1) {  // item epilogue (as zgemm_kernel)
      const int64_t e = cons.e;
      const int i0 = cons.i0, j0 = cons.j0;
      if (P.fault && i0 == 0 && j0 == 0 && wr == 0 && wc == 0 && lane == 0) {
        const double2 a00 = *reinterpret_cast<const double2*>(P.A + 2 * P.sA * e);
        const double2 b00 = *reinterpret_cast<const double2*>(P.B + 2 * P.sB * e);
        const double tr = __dsub_rn(__dmul_rn(a00.x, b00.x), __dmul_rn(a00.y, b00.y));
        cr[0][0][0] -= 2.0 * tr;
      }
      const double* c = P.C ? P.C + 2 * P.sC * e : nullptr;
      double* o = P.out + 2 * P.sO * e;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int gi = i0 + (wr * 2 + i) * 8 + mm;
            const int gj = j0 + (wc * NB + j) * 8 + 2 * kq + h;
            if (gi < P.m && gj < P.n) {
              const size_t idx = gi + static_cast<size_t>(gj) * P.m;
              double cvr = 0.0, cvi = 0.0;
              if (c) {
                const double2 v = *reinterpret_cast<const double2*>(c + 2 * idx);
                cvr = v.x;
                cvi = v.y;
              }
              const double sr = cr[i][j][h], si = ci[i][j][h];
              double re, im;
              if (unit) {  // alpha = 1, beta = 0, no C: the formula below reduces to x + 0.0 exactly
                re = __dadd_rn(sr, 0.0);
                im = __dadd_rn(si, 0.0);
              } else {
                re = __dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(P.ar, sr), __dmul_rn(P.ai, si)), __dmul_rn(P.br, cvr)),
                               __dmul_rn(P.bi, cvi));
                im = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(P.ar, si), __dmul_rn(P.ai, sr)), __dmul_rn(P.br, cvi)),
                               __dmul_rn(P.bi, cvr));
              }
              *reinterpret_cast<double2*>(o + 2 * idx) = make_double2(re, im);
            }
            cr[i][j][h] = 0.0;
            ci[i][j][h] = 0.0;
          }
    }
    advance(cons);
  }
}

using EncodeTiled = PFN_cuTensorMapEncodeTiled_v12000;
EncodeTiled tensor_map_encoder() {
  static const EncodeTiled fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiled>(nullptr);
    return reinterpret_cast<EncodeTiled>(f);
  }();
  return fn;
}

// 4-D FP64 map (16 doubles, rows / 8, cols, batch) of a column-major complex operand with
// `rows` rows (multiple of 8), entry stride `stride` complex elements; box (16, b1, b2, 1).
bool encode_operand(CUtensorMap* map, const double* base, int rows, int cols, int batch, int64_t stride,
                    int b1, int b2) {
  const EncodeTiled enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[4] = {16, static_cast<cuuint64_t>(rows / 8), static_cast<cuuint64_t>(cols),
                        static_cast<cuuint64_t>(batch)};
  cuuint64_t strides[3] = {128, static_cast<cuuint64_t>(rows) * 16, static_cast<cuuint64_t>(stride) * 16};
  cuuint32_t box[4] = {16, static_cast<cuuint32_t>(b1), static_cast<cuuint32_t>(b2), 1};
  cuuint32_t elem[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, elem,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t launch_zgemm_strided(int batch, int m, int n, int k, double ar, double ai,
                                 const double* A, int64_t sA, const double* B, int64_t sB,
                                 double br, double bi, const double* C, int64_t sC, double* out,
                                 int64_t sO, int inject_fault, cudaStream_t stream) {
  if (batch < 1 || m < 1 || n < 1 || k < 1) return cudaErrorInvalidValue;
  ZArgs P{};
  P.m = m;
  P.n = n;
  P.k = k;
  P.tm = (m + ZT - 1) / ZT;
  P.tn = (n + ZT - 1) / ZT;
  P.nk = (k + ZK - 1) / ZK;
  P.ar = ar;
  P.ai = ai;
  P.br = br;
  P.bi = bi;
  P.A = A;
  P.sA = sA;
  P.B = B;
  P.sB = sB;
  P.C = C;
  P.sC = sC;
  P.out = out;
  P.sO = sO;
  P.fault = inject_fault;
  P.items = static_cast<int64_t>(batch) * P.tm * P.tn;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = static_cast<int>(std::min<int64_t>(P.items, sms));
  // TMA staging when the shapes allow it (TG_ZGEMM_TMA=0: the cp.async pipeline)
  const char* env = std::getenv("TG_ZGEMM_TMA");
  if (!(env && env[0] == '0') && m % 8 == 0 && k % 8 == 0) {
    // kernel shape (TG_ZGEMM_WARPS=4|5|8|9|16 overrides; profiles/r02_zgemm_vs_cublas.txt): the
    // 32x32-tile kernel (3 CTAs per SM; 4 consumer warps + a producer warpgroup, "5") when
    // 64x64 tiles would pad m x n noticeably more (96^3: 31.9 vs 18.5 TF/s), else 8 warps of 16x32 plus a producer warp that issues
    // the TMA stages ("9": best or within 0.3 % of the best at every measured size)
    auto fill = [&](int t) {
      const double mp = static_cast<double>((m + t - 1) / t * t), np_ = static_cast<double>((n + t - 1) / t * t);
      return static_cast<double>(m) * n / (mp * np_);
    };
    const char* w = std::getenv("TG_ZGEMM_WARPS");
    const int warps = w ? std::atoi(w) : (fill(32) > 1.05 * fill(64) ? 5 : 9);
    auto run = [&](auto kern, int wr, int tn, int stages, int minb, int extra = 0) -> cudaError_t {
      ZArgs Q = P;
      Q.tm = (m + 16 * wr - 1) / (16 * wr);
      Q.tn = (n + tn - 1) / tn;
      Q.items = static_cast<int64_t>(batch) * Q.tm * Q.tn;
      CUtensorMap mapA, mapB;
      if (!encode_operand(&mapA, A, m, k, batch, sA, 2, ZK) || !encode_operand(&mapB, B, k, n, batch, sB, 4, tn))
        return cudaErrorNotSupported;
      const int stage_bytes = (wr * TBoxA + 64 * tn) * 8;
      const int tbytes = stages * stage_bytes + 1024;
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, tbytes);
      if (e != cudaSuccess) return e;
      const int g = static_cast<int>(std::min<int64_t>(Q.items, static_cast<int64_t>(sms) * minb));
      kern<<<g, 32 * wr * (warps == 4 || warps == 5 ? 2 : warps / wr) + extra, tbytes, stream>>>(Q, mapA, mapB);
      return cudaGetLastError();
    };
    cudaError_t e = cudaErrorNotSupported;
    if (warps == 4) e = run(zgemm_tma_kernel<2, 2, 2, 2, 3>, 2, 32, 2, 3);
    else if (warps == 5) e = run(zgemm_tma_kernel<2, 2, 2, 2, 3, true, 120>, 2, 32, 2, 3, 128);  // 4 + producer
    else if (warps == 16) e = run(zgemm_tma_kernel<4, 4, 2, 3, 1>, 4, 64, 3, 1);
    else if (warps == 9) e = run(zgemm_tma_kernel<4, 2, 4, 3, 1, true>, 4, 64, 3, 1, 128);  // + producer
    else e = run(zgemm_tma_kernel<4, 2, 4, 3, 1>, 4, 64, 3, 1);
    if (e != cudaErrorNotSupported) return e;
  }
  constexpr int bytes = ZStages * StageElems * 16;
  cudaError_t e = cudaFuncSetAttribute(zgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  zgemm_kernel<<<grid, ZThreads, bytes, stream>>>(P);
  return cudaGetLastError();
}

}  // namespace tg
