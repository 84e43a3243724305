// fp64_contention.cu — latency of a dependent FP64 chain (DADD/DFMA) on an SMSP whose FP64
// pipe is saturated by DMMA.8x8x4 from other warps (sm_100a). Also measures the chain
// with FP32 ops and integer ops as controls, and DMMA throughput with/without the chain.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// warps 0..7: DMMA streams (if dmma_on); warp 8 lane 0: dependent chain of `kind` ops.
__global__ void contention(int dmma_on, int kind, int iters, long long* out, double* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp < 8) {
    if (!dmma_on) return;
    double a = 1.0 + lane * 1e-9, b = 1.0 - lane * 1e-9;
    double c[8][2] = {};
    long long n = 0;
    while (!stop) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
      ++n;
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) sink[0] = s;
    if (lane == 0) atomicAdd((unsigned long long*)&out[2], (unsigned long long)n);
    return;
  }
  if (lane != 0) return;
  // let the DMMA warps ramp up
  long long t = clock64();
  while (clock64() - t < 20000) {}
  long long t0 = clock64();
  if (kind == 0) {  // dependent DADD chain
    double x = 1.0 + sink[1];
    for (int i = 0; i < iters; ++i) x = x + 1e-30;
    sink[2] = x;
  } else if (kind == 1) {  // dependent FP32 chain
    float x = 1.0f + (float)sink[1];
    for (int i = 0; i < iters; ++i) x = x + 1e-30f;
    sink[2] = x;
  } else {  // dependent integer chain
    long long x = (long long)sink[1];
    for (int i = 0; i < iters; ++i) x = x * 3 + 1;
    sink[2] = (double)x;
  }
  long long t1 = clock64();
  out[0] = t1 - t0;
  stop = 1;
}

int main() {
  long long* d;
  double* sink;
  cudaMalloc(&d, 64);
  cudaMalloc(&sink, 64);
  cudaMemset(sink, 0, 64);
  const char* names[] = {"DADD chain", "FADD chain", "IMAD chain"};
  for (int kind = 0; kind < 3; ++kind)
    for (int on = 0; on < 2; ++on) {
      cudaMemset(d, 0, 64);
      const int iters = 2000;
      contention<<<1, 9 * 32>>>(on, kind, iters, d, sink);
      cudaDeviceSynchronize();
      long long h[3];
      cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
      printf("%s, DMMA warps %s: %.1f clk per dependent op (dmma iterations %lld)\n", names[kind],
             on ? "ON " : "OFF", (double)h[0] / iters, h[2]);
    }
  return 0;
}
