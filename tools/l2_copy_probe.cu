// l2_copy_probe.cu — per-SM bandwidth of an L2-resident read+write pass shaped like the
// HBM tier's S = 14 gate (one CTA of 256 threads per SM, each CTA owning a 256 KB source
// and a 256 KB destination, 16-byte ld.cg/st.cg, 8 loads in flight per thread).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2_copy_probe tools/l2_copy_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int INFLIGHT>
__global__ void copy_pass(const double2* src, double2* dst, int n2, int reps, long long* cyc) {
  const double2* s = src + static_cast<size_t>(blockIdx.x) * n2;
  double2* d = dst + static_cast<size_t>(blockIdx.x) * n2;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int i = threadIdx.x; i < n2; i += blockDim.x * INFLIGHT) {
      double2 v[INFLIGHT];
#pragma unroll
      for (int k = 0; k < INFLIGHT; ++k) {
        const int j = i + k * blockDim.x;
        v[k] = j < n2 ? __ldcg(s + j) : make_double2(0, 0);
      }
#pragma unroll
      for (int k = 0; k < INFLIGHT; ++k) {
        const int j = i + k * blockDim.x;
        if (j < n2) __stcg(d + j, make_double2(v[k].x * 1.0000001, v[k].y));
      }
    }
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0) / reps;
}

template <int INFLIGHT>
void run(int sms, int kb) {
  const int n2 = kb * 1024 / 16;  // double2 per CTA
  double2 *a, *b;
  long long* cyc;
  cudaMalloc(&a, static_cast<size_t>(sms) * n2 * 16);
  cudaMalloc(&b, static_cast<size_t>(sms) * n2 * 16);
  cudaMalloc(&cyc, sms * 8);
  cudaMemset(a, 0, static_cast<size_t>(sms) * n2 * 16);
  copy_pass<INFLIGHT><<<sms, 256>>>(a, b, n2, 2, cyc);
  copy_pass<INFLIGHT><<<sms, 256>>>(a, b, n2, 20, cyc);
  cudaDeviceSynchronize();
  long long h[1024], mx = 0, sum = 0;
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  for (int i = 0; i < sms; ++i) {
    mx = h[i] > mx ? h[i] : mx;
    sum += h[i];
  }
  printf("in-flight %2d x 16B/thread, %d KB read + %d KB written per SM: %lld clk (mean %lld) = %.1f B/clk/SM\n",
         INFLIGHT, kb, kb, mx, sum / sms, 2.0 * kb * 1024 / (sum / sms));
  cudaFree(a);
  cudaFree(b);
  cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4>(sms, 256);
  run<8>(sms, 256);
  run<16>(sms, 256);
  run<16>(sms, 1024);
  run<1>(1, 256);
  run<16>(1, 256);
  return 0;
}
