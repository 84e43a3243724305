// vn_bench.cu — clock64 phase timing of the device von Neumann solver (vn.cuh) on
// rho = Psi Psi^dagger of random states, one CTA of 256 threads per SM (the anneal kernel's
// configuration). Prints per-phase clocks (CTA 0, averaged over repetitions).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2203_09353_b200/csrc \
//        vn_bench.cu -o vn_bench && ./vn_bench [n=64] [reps=20]
#include <cstdio>
#include <cstdlib>

#include "vn.cuh"

using namespace tg;

__device__ double hash01(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return (x >> 11) * 0x1.0p-53;
}

__global__ void __launch_bounds__(256, 1) bench(int n, int reps, long long* clk, double* ent) {
  extern __shared__ __align__(16) double sm[];
  const int P = n + 4;
  double* Ar = sm;
  double* Ai = Ar + n * P;
  vn::Scratch& W = *reinterpret_cast<vn::Scratch*>(Ai + n * P);
  double* psr = reinterpret_cast<double*>(&W + 1);
  double* psi = psr + n * n;
  const int tid = threadIdx.x;
  auto sync = [] { __syncthreads(); };
  long long acc[3] = {0, 0, 0};
  for (int r = 0; r < reps; ++r) {
    // random Psi (n x n) and rho = Psi Psi^H / tr
    for (int i = tid; i < n * n; i += 256) {
      psr[i] = hash01(blockIdx.x * 1000003ull + r * 7919ull + 2 * i) - 0.5;
      psi[i] = hash01(blockIdx.x * 1000003ull + r * 7919ull + 2 * i + 1) - 0.5;
    }
    __syncthreads();
    for (int idx = tid; idx < n * n; idx += 256) {
      const int i = idx % n, j = idx / n;
      double sr = 0, si = 0;
      for (int k = 0; k < n; ++k) {
        const double ar = psr[i + k * n], ai = psi[i + k * n], br = psr[j + k * n], bi = psi[j + k * n];
        sr += ar * br + ai * bi;
        si += ai * br - ar * bi;
      }
      Ar[i + j * P] = sr / (n * n / 6.0);
      Ai[i + j * P] = si / (n * n / 6.0);
    }
    __syncthreads();
    const long long t0 = clock64();
    vn::tridiagonalize(Ar, Ai, n, P, W, tid, sync);
    const long long t1 = clock64();
    vn::eigenvalues(n, W, tid, sync);
    const long long t2 = clock64();
    double e = 0.0;
    if (tid < 32) {
      for (int i = tid; i < n; i += 32) {
        const double l = W.lam[i];
        W.pr[0][i] = l > 1e-15 ? l * log(l) : 0.0;
      }
      __syncwarp();
      if (tid == 0)
        for (int i = 0; i < n; ++i) e -= W.pr[0][i];
    }
    __syncthreads();
    const long long t3 = clock64();
    acc[0] += t1 - t0;
    acc[1] += t2 - t1;
    acc[2] += t3 - t2;
    if (tid == 0) ent[blockIdx.x * reps + r] = e;
  }
  if (tid == 0 && blockIdx.x == 0)
    for (int k = 0; k < 3; ++k) clk[k] = acc[k] / reps;
}

// Isolated pieces of one Householder step at k = 0 (m = n-1), each repeated `reps` times.
__global__ void __launch_bounds__(256, 1) pieces(int n, int reps, long long* clk) {
  extern __shared__ __align__(16) double sm[];
  const int P = n + 4;
  double* Ar = sm;
  double* Ai = Ar + n * P;
  vn::Scratch& W = *reinterpret_cast<vn::Scratch*>(Ai + n * P);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < n * P; i += 256) {
    Ar[i] = hash01(i) * 1e-3;
    Ai[i] = hash01(i + 99999) * 1e-3;
  }
  for (int i = tid; i < 64; i += 256) {
    W.vr[0][i] = W.vr[1][i] = hash01(i + 7) * 1e-3;
    W.vi[0][i] = W.vi[1][i] = hash01(i + 8) * 1e-3;
    W.pr[0][i] = W.pr[1][i] = hash01(i + 9) * 1e-3;
    W.pi[0][i] = W.pi[1][i] = hash01(i + 10) * 1e-3;
  }
  if (tid < 8) W.part[0][tid] = W.part[1][tid] = 1e-3;
  if (tid == 0) W.tau[0] = W.tau[1] = 1.0;
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    vn::update(Ar, Ai, n, P, 0, W, warp, lane);
    __syncthreads();
  }
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) {
    vn::matvec(Ar, Ai, n, P, 0, W, warp, lane);
    __syncthreads();
  }
  long long t2 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (warp == 0) vn::reflector(Ar, Ai, n, P, 0, W, lane);
    __syncthreads();
  }
  long long t3 = clock64();
  for (int r = 0; r < reps; ++r) __syncthreads();
  long long t4 = clock64();
  if (tid == 0 && blockIdx.x == 0) {
    clk[0] = (t1 - t0) / reps;
    clk[1] = (t2 - t1) / reps;
    clk[2] = (t3 - t2) / reps;
    clk[3] = (t4 - t3) / reps;
  }
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 64, reps = argc > 2 ? atoi(argv[2]) : 20;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* clk;
  double* ent;
  cudaMalloc(&clk, 3 * sizeof(long long));
  cudaMalloc(&ent, sizeof(double) * sms * reps);
  const int bytes = 2 * n * (n + 4) * 8 + sizeof(vn::Scratch) + 2 * n * n * 8;
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  bench<<<sms, 256, bytes>>>(n, 1, clk, ent);  // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<<<sms, 256, bytes>>>(n, reps, clk, ent);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  long long h[3];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double e0;
  cudaMemcpy(&e0, ent, 8, cudaMemcpyDeviceToHost);
  printf("{\"n\": %d, \"reps\": %d, \"tridiag_clk\": %lld, \"eig_clk\": %lld, \"sum_clk\": %lld, "
         "\"kernel_ms\": %.3f, \"entropy0\": %.17g}\n", n, reps, h[0], h[1], h[2], ms, e0);
  {
    long long* c4;
    cudaMalloc(&c4, 4 * sizeof(long long));
    const int pb = 2 * n * (n + 4) * 8 + sizeof(vn::Scratch);
    cudaFuncSetAttribute(pieces, cudaFuncAttributeMaxDynamicSharedMemorySize, pb);
    pieces<<<sms, 256, pb>>>(n, 50, c4);
    cudaDeviceSynchronize();
    long long h4[4];
    cudaMemcpy(h4, c4, sizeof(h4), cudaMemcpyDeviceToHost);
    printf("{\"n\": %d, \"update_clk\": %lld, \"matvec_clk\": %lld, \"reflector_clk\": %lld, \"sync_clk\": %lld}\n",
           n, h4[0], h4[1], h4[2], h4[3]);
  }
  return 0;
}
