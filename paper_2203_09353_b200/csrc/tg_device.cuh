// tg_device.cuh — device building blocks of the persistent annealing kernels (sm_100a).
//
//  * xoshiro256++ / splitmix64 seeding: bit-exact port of rng.cpp:12-59 (integer work).
//  * Box-Muller (rng.cpp:61-67) with CUDA libm log/sqrt/sincos (<= 2 ulp vs glibc).
//  * GateRec: one pre-generated proposal (gate_stream.cu builds the stream).
//  * mbarrier / cp.async helpers.
//  * FP64 tensor op: mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4 (the only FP64 MMA shape on
//    sm_100a; there is no tcgen05 kind for f64).
#pragma once
#include <cstdint>

namespace tg {

// ------------------------------------------------------------------------------ RNG
struct Xoshiro {
  uint64_t s0, s1, s2, s3;
};

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// rng.cpp:23-33
__host__ __device__ __forceinline__ Xoshiro stream_init(uint64_t global_seed, uint64_t p) {
  uint64_t s = global_seed ^ mix64(p + 1);
  uint64_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    s += 0x9E3779B97F4A7C15ULL;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    w[i] = z ^ (z >> 31);
  }
  if ((w[0] | w[1] | w[2] | w[3]) == 0) w[0] = 1;
  return Xoshiro{w[0], w[1], w[2], w[3]};
}

__host__ __device__ __forceinline__ uint64_t rotl64(uint64_t x, int k) {
  return (x << k) | (x >> (64 - k));
}

// rng.cpp:35-45
__host__ __device__ __forceinline__ uint64_t next_u64(Xoshiro& st) {
  const uint64_t result = rotl64(st.s0 + st.s3, 23) + st.s0;
  const uint64_t t = st.s1 << 17;
  st.s2 ^= st.s0;
  st.s3 ^= st.s1;
  st.s1 ^= st.s2;
  st.s0 ^= st.s3;
  st.s2 ^= t;
  st.s3 = rotl64(st.s3, 45);
  return result;
}

// rng.cpp:47-49 (exact: a 53-bit integer converts exactly)
__device__ __forceinline__ double u01(uint64_t x) {
  return __dmul_rn(__ull2double_rn(x >> 11), 0x1.0p-53);
}

// rng.cpp:51-59: reject x < 2^64 mod n, return x mod n. Warp-uniform when all lanes
// hold the same state.
__device__ __forceinline__ uint32_t uniform_index(Xoshiro& st, uint64_t n) {
  const uint64_t reject_below = (0 - n) % n;
  for (;;) {
    const uint64_t x = next_u64(st);
    if (x >= reject_below) return static_cast<uint32_t>(x % n);
  }
}

// rng.cpp:61-67 for the two draws (x1 -> u1, x2 -> u2).
__device__ __forceinline__ void box_muller(uint64_t x1, uint64_t x2, double& a, double& b) {
  const double u1 = __dsub_rn(1.0, u01(x1));
  const double u2 = u01(x2);
  const double r = sqrt(__dmul_rn(-2.0, log(u1)));
  const double angle = __dmul_rn(6.283185307179586, u2);  // (2.0 * std::numbers::pi) * u2
  double s, c;
  sincos(angle, &s, &c);
  a = __dmul_rn(r, c);
  b = __dmul_rn(r, s);
}

// -------------------------------------------------------------- gate stream record
// One proposal of one replica, produced by the pre-pass (gate_stream.cu). 288 bytes.
struct GateRec {
  double ur[16];  // U(x,y).re at x*4+y (row-major: x = output basis index)
  double ui[16];
  double u;       // uniform01 acceptance draw (spinmc.cpp:207)
  double temp;    // temperature(step) (spinmc.cpp:178-184)
  double emul;    // decision factor: exp(-T log u) (maximize) / exp(T log u) (minimize)
  int32_t site;   // uniform_index(S-1) (spinmc.cpp:198)
  float tie_tol;  // lean-decision window: relative margins <= tie_tol are re-decided with the
                  // reference formula (covers every |u - p| < 1e-9, smem::decide_audit)
};
static_assert(sizeof(GateRec) == 288, "GateRec layout");

// spinmc.cpp:178-184 (the schedule is data-independent: computed by the pre-pass)
__device__ __forceinline__ double temperature(double t0, double t_min, uint64_t step,
                                              uint64_t total) {
  const double frac = __ddiv_rn(static_cast<double>(step), static_cast<double>(total));
  return __dmul_rn(t0, pow(__ddiv_rn(t_min, t0), frac));
}

// spinmc.cpp:186-191
__device__ __forceinline__ double acceptance(double delta, double t) {
  double x = __ddiv_rn(delta, t);
  x = (0.0 < x) ? 0.0 : x;
  x = (x < -745.0) ? -745.0 : x;
  return exp(x);
}

// ---------------------------------------------------------------------- mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Generic-proxy global writes made visible to later async-proxy (bulk copy) reads.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Prior generic-proxy shared-memory accesses ordered before later async-proxy writes.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// TMA-engine bulk copy global -> shared (cp.async.bulk, SASS UBLKCP), completion counted
// in bytes on an mbarrier of the executing CTA.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMA tensor copy global -> shared of one box of a 5-D tensor map (SASS UTMALDG), completion
// counted in bytes on an mbarrier of the executing CTA. `map` is the generic address of a
// __grid_constant__ CUtensorMap kernel parameter.
__device__ __forceinline__ void tma_load_5d(void* dst, const void* map, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const void* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// Named barrier over the consumer warps only (id 1; the producer warp never joins).
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// -------------------------------------------------------------------------- DMMA
// D = A*B + C, m8n8k4 f64. Lane l: A[l>>2][l&3], B[l&3][l>>2], C/D[l>>2][2(l&3)+{0,1}].
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int64_t globaltimer() {
  int64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace tg
