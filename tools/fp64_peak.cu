// FP64 peak microbenchmark for B200 (sm_100a): DMMA.8x8x4 (mma.sync f64) vs DFMA.
// Measures the roofline denominator used by bench.py (no FP64 entry exists in MEASURED_PEAKS.json).
// Each warp runs NCHAIN independent accumulator chains in a register-resident loop.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int NCHAIN>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NCHAIN][2];
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCHAIN; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NCHAIN>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NCHAIN];
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCHAIN; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
double timeit(K kern, int blocks, int threads, int iters, double* d) {
  kern<<<blocks, threads>>>(d, iters / 10);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main(int argc, char** argv) {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* d; CK(cudaMalloc(&d, 64));
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;
  printf("{\"sms\": %d, \"results\": [\n", sms);
  bool first = true;
  for (int wpb : {4, 8, 16}) {
    for (int bps : {1, 2}) {
      int threads = wpb * 32, blocks = sms * bps;
      double ms = timeit(dmma_loop<8>, blocks, threads, iters, d);
      double flops = 512.0 * 8 * iters * (double)blocks * wpb;
      printf("%s {\"kind\": \"dmma_m8n8k4\", \"warps_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
             first ? "" : ",", wpb * bps, ms, flops / ms / 1e9);
      first = false;
      ms = timeit(dfma_loop<8>, blocks, threads, iters, d);
      flops = 2.0 * 8 * iters * (double)blocks * threads;
      printf(", {\"kind\": \"dfma\", \"warps_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
             wpb * bps, ms, flops / ms / 1e9);
    }
  }
  printf("]}\n");
  return 0;
}
