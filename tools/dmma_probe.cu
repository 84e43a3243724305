// dmma_probe.cu — DMMA.8x8x4 latency / issue characterisation on B200 (sm_100a).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe tools/dmma_probe.cu
// Prints, for one CTA per SM on every SM:
//   chains: W warps x C independent accumulator chains (register-only) -> DMMA/clk/SM
//   tile  : the anneal GEMM inner pattern (per k4: 12 LDS.64 fragment loads, 32 DMMA into
//           16 accumulators, two dependent DMMAs per accumulator) for W warps, with the
//           fragment loads software-pipelined one k4 ahead (PIPE=1) or not (PIPE=0).
// Peak = 0.25 DMMA/clk/SM (128 FP64 flop/clk/SM, profiles/r01_fp64_peak.json).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int C>
__global__ void chains(int iters, long long* cyc, double* sink) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[C][2];
#pragma unroll
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  __syncthreads();
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) sink[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// GEMM-tile pattern: SMEM panel 4 planes x 32 cols x 68 pitch (like hbm_tier.cuh), warp
// grid 4x2 of 16x32 sub-tiles (TM=2, TN=4) — only the first 8 warps' roles, repeated.
template <int PIPE, bool RANDOM = false>
__global__ void tile(int iters, long long* cyc, double* sink) {
  extern __shared__ double sm[];
  constexpr int SP = 68, KP = 32 * SP;
  for (int i = threadIdx.x; i < 6 * KP; i += blockDim.x) {
    if (RANDOM) {  // state-like data: random signs/mantissas, magnitudes ~2^-6 (|psi| ~ 1/64)
      unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      sm[i] = (static_cast<double>(z >> 11) * 0x1.0p-53 - 0.5) * 0.03;
    } else {
      sm[i] = 1.0 + i * 1e-12;
    }
  }
  double* gout = sm + 4 * KP;  // PIPE 2: gate-chunk stores (another buffer)
  double g_vr = 0, g_vi = 0, r0 = 0, r1 = 0;
  const double ga1 = 0.5 + threadIdx.x * 1e-6, ga2 = 0.25 - threadIdx.x * 1e-6;
  __syncthreads();
  const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
  const int wr = warp / 2, wc = warp % 2, m = lane >> 2, kq = lane & 3;
  const double *AX = sm, *AY = sm + KP, *BX = sm + 2 * KP, *BY = sm + 3 * KP;
  double cr[2][4][2] = {}, ci[2][4][2] = {};
  double xa[2], ya[2], xb[4], yb[4];
  auto load = [&](int kb) {
    const int col = (kb + kq) * SP;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      xa[i] = AX[(wr * 2 + i) * 8 + m + col];
      ya[i] = AY[(wr * 2 + i) * 8 + m + col];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      xb[j] = BX[(wc * 4 + j) * 8 + m + col];
      yb[j] = BY[(wc * 4 + j) * 8 + m + col];
    }
  };
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kb = 0; kb < 32; kb += 4) {
      load(kb);
      double xn[2] = {-xa[0], -xa[1]};
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (PIPE != 1) {
            dmma(cr[i][j][0], cr[i][j][1], xa[i], xb[j]);
            dmma(cr[i][j][0], cr[i][j][1], ya[i], yb[j]);
            dmma(ci[i][j][0], ci[i][j][1], ya[i], xb[j]);
            dmma(ci[i][j][0], ci[i][j][1], xn[i], yb[j]);
          } else {
            dmma(cr[i][j][0], cr[i][j][1], xa[i], xb[j]);
            dmma(ci[i][j][0], ci[i][j][1], ya[i], xb[j]);
          }
        }
      if (PIPE == 5) {  // + 2 cp.async (16 B, L2-resident global) per k4 per thread, like the HBM tier
        const double* g = sink + 64 + ((blockIdx.x * 8192 + it * 512 + kb * 64 + threadIdx.x * 2) & ((1 << 21) - 1));
        double* d = gout + ((threadIdx.x * 2 + kb * 128) & 2047);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(d)), "l"(g) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(d + 512)), "l"(g + 512) : "memory");
        if (kb == 28) {
          asm volatile("cp.async.commit_group;\n" ::: "memory");
          asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        }
      }
      if (PIPE == 3) {  // gate-chunk DMMAs only (no SMEM traffic)
        r0 = 0; r1 = 0;
        dmma(r0, r1, ga1, g_vr);
        dmma(r0, r1, ga2, g_vi);
        g_vr += r0;
        g_vi += r1;
      }
      if (PIPE == 4) {  // gate-chunk SMEM traffic only (no DMMA)
        const int o = ((threadIdx.x * 8 + kb * 67 + it) & 2047);
        gout[o] = g_vr;
        gout[o ^ 1024] = g_vi;
        g_vr = AX[o & 1023];
        g_vi = AY[o & 1023];
      }
      if (PIPE == 2) {  // one software-pipelined gate chunk per k4 (anneal SPEC pattern)
        const int o = ((threadIdx.x * 8 + kb * 67 + it) & 2047);
        gout[o] = r0;
        gout[o ^ 1024] = r1;
        r0 = 0; r1 = 0;
        dmma(r0, r1, ga1, g_vr);
        dmma(r0, r1, ga2, g_vi);
        g_vr = AX[o & 1023];
        g_vi = AY[o & 1023];
      }
      if (PIPE == 1) {  // second half: dependent partners 8 DMMAs later
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            dmma(cr[i][j][0], cr[i][j][1], ya[i], yb[j]);
            dmma(ci[i][j][0], ci[i][j][1], xn[i], yb[j]);
          }
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) s += cr[i][j][0] + cr[i][j][1] + ci[i][j][0] + ci[i][j][1];
  if (s == 12345.678 || g_vr + r0 == 12345.678) sink[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <class K>
double run(K kern, int warps, int iters, int dmma_per_warp_iter, int smem) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc;
  double* sink;
  cudaMalloc(&cyc, sms * sizeof(long long));
  cudaMalloc(&sink, (64 + (1 << 21) + 4096) * sizeof(double));
  cudaMemset(sink, 0, (64 + (1 << 21) + 4096) * sizeof(double));
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kern<<<sms, warps * 32, smem>>>(iters / 4, cyc, sink);
  kern<<<sms, warps * 32, smem>>>(iters, cyc, sink);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  cudaFree(cyc);
  cudaFree(sink);
  return static_cast<double>(warps) * iters * dmma_per_warp_iter / mx;  // DMMA/clk/SM
}

int main() {
  const int it = 20000;
  printf("latency (1 warp, 1 chain): %.1f clk per dependent DMMA\n", 1.0 / run(chains<1>, 1, it, 1, 0));
  const int Ws[] = {1, 2, 4, 8, 12, 16};
  for (int w : Ws) {
    printf("W=%2d warps:", w);
    printf("  C=1 %.3f", run(chains<1>, w, it, 1, 0));
    printf("  C=2 %.3f", run(chains<2>, w, it, 2, 0));
    printf("  C=4 %.3f", run(chains<4>, w, it / 2, 4, 0));
    printf("  C=8 %.3f", run(chains<8>, w, it / 4, 8, 0));
    printf("  C=16 %.3f DMMA/clk/SM (peak 0.25)\n", run(chains<16>, w, it / 8, 16, 0));
  }
  const int smem = 6 * 32 * 68 * 8;
  const int Wt[] = {4, 8, 16};
  for (int w : Wt)
    printf("tile W=%2d: adjacent pairs %.3f  split pairs %.3f  +gate chunk %.3f  +gate DMMA only %.3f  +gate SMEM only %.3f DMMA/clk/SM\n", w,
           run(tile<0>, w, 500, 256, smem), run(tile<1>, w, 500, 256, smem), run(tile<2>, w, 500, 272, smem),
           run(tile<3>, w, 500, 272, smem), run(tile<4>, w, 500, 256, smem));
  for (int w : Wt) printf("tile W=%2d: + 2 cp.async/k4/thread %.3f DMMA/clk/SM\n", w, run(tile<5>, w, 500, 256, smem));
  for (int w : Wt)
    printf("tile W=%2d, random state-like data: adjacent pairs %.3f  (1.0-ish data %.3f) DMMA/clk/SM\n", w,
           run(tile<0, true>, w, 500, 256, smem), run(tile<0, false>, w, 500, 256, smem));
  return 0;
}
