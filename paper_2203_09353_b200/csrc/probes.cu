// probes.cu — device-piece entry points used by the parity suite
// and the FP64 DMMA roofline probe. They run the SAME device functions as the anneal
// kernels (tg_device.cuh, smem_tier.cuh, hbm_tier.cuh), on inputs the test supplies.
#include "hbm_tier.cuh"
#include "smem_tier.cuh"
#include "tg_internal.h"
#include "vn.cuh"

namespace tg {
namespace {

__global__ void rng_kernel(uint64_t seed, uint64_t p, uint64_t n, uint64_t* out) {
  Xoshiro st = stream_init(seed, p);
  for (uint64_t i = 0; i < n; ++i) out[i] = next_u64(st);
}

__global__ void probe_unpack_kernel(const GateRec* recs, uint64_t steps, uint8_t* sites, double* u,
                                    double* uacc) {
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (i >= steps) return;
  const GateRec& g = recs[i];
  for (int x = 0; x < 4; ++x)
    for (int y = 0; y < 4; ++y) {  // back to column-major interleaved U(x,y) at 2*(x + 4y)
      u[i * 32 + 2 * (x + 4 * y)] = g.ur[x * 4 + y];
      u[i * 32 + 2 * (x + 4 * y) + 1] = g.ui[x * 4 + y];
    }
  sites[i] = static_cast<uint8_t>(g.site);
  uacc[i] = g.u;
}

// Loads interleaved complex psi (2^S) into the planar padded SMEM layout.
template <class D>
__device__ void load_state(const double* psi, double* X, double* Y, int tid, int nthr) {
  for (int i = tid; i < 2 * D::PLANE; i += nthr) X[i] = 0.0;  // X and Y are contiguous
  __syncthreads();
  for (int idx = tid; idx < D::N; idx += nthr) {
    X[D::phys(idx)] = psi[2 * idx];
    Y[D::phys(idx)] = psi[2 * idx + 1];
  }
  __syncthreads();
}

template <int LA, int LB>
__global__ void apply_gate_smem_kernel(const double* psi, int site, const double* u, double* out) {
  using D = smem::Dims<LA, LB>;
  extern __shared__ __align__(128) unsigned char raw[];
  GateRec& g = *reinterpret_cast<GateRec*>(raw);
  double* planes = reinterpret_cast<double*>(raw + 512);
  const int tid = threadIdx.x;
  if (tid < 16) {
    const int x = tid >> 2, y = tid & 3;
    g.ur[tid] = u[2 * (x + 4 * y)];
    g.ui[tid] = u[2 * (x + 4 * y) + 1];
  }
  load_state<D>(psi, planes, planes + D::PLANE, tid, blockDim.x);
  smem::gate_pass<D>(planes, planes + D::PLANE, planes + 2 * D::PLANE, planes + 3 * D::PLANE,
                     site, g, tid, blockDim.x);
  __syncthreads();
  for (int idx = tid; idx < D::N; idx += blockDim.x) {
    out[2 * idx] = planes[2 * D::PLANE + D::phys(idx)];
    out[2 * idx + 1] = planes[3 * D::PLANE + D::phys(idx)];
  }
}

template <int LA, int LB>
__global__ void entropy_smem_kernel(const double* psi_all, double* e_out, double* n_out, bool fault) {
  using D = smem::Dims<LA, LB>;
  extern __shared__ __align__(128) unsigned char raw[];
  __shared__ double part[2][smem::kConsumerWarps];
  double* planes = reinterpret_cast<double*>(raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* psi = psi_all + 2ull * D::N * blockIdx.x;
  load_state<D>(psi, planes, planes + D::PLANE, tid, blockDim.x);
  double rho2, tr;
  smem::rho_partials<D>(planes, planes + D::PLANE, warp, lane, fault, rho2, tr);
  if (lane == 0) {
    part[0][warp] = rho2;
    part[1][warp] = tr;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, t = 0.0;
    for (int w = 0; w < smem::kConsumerWarps; ++w) {
      a += part[0][w];
      t += part[1][w];
    }
    e_out[blockIdx.x] = smem::renyi2(a);
    if (n_out) n_out[blockIdx.x] = __dsqrt_rn(t);
  }
}

// von Neumann entropy of each state (vn.cuh), same rho path as the anneal kernel.
template <int LA, int LB>
__global__ void entropy_vn_smem_kernel(const double* psi_all, double* e_out, double* n_out, bool fault) {
  using D = smem::Dims<LA, LB>;
  constexpr int RP = D::DA_PAD + 4;
  extern __shared__ __align__(128) unsigned char raw[];
  __shared__ double part[smem::kConsumerWarps];
  double* planes = reinterpret_cast<double*>(raw);
  double* Rr = planes + 2 * D::PLANE;
  double* Ri = Rr + D::DA_PAD * RP;
  vn::Scratch& W = *reinterpret_cast<vn::Scratch*>(Ri + D::DA_PAD * RP);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* psi = psi_all + 2ull * D::N * blockIdx.x;
  load_state<D>(psi, planes, planes + D::PLANE, tid, blockDim.x);
  double rho2, tr;
  smem::rho_partials<D, true>(planes, planes + D::PLANE, warp, lane, fault, rho2, tr, Rr, Ri, RP);
  if (lane == 0) part[warp] = tr;
  __syncthreads();
  const double e = vn::entropy(Rr, Ri, D::DA, RP, W, tid, [] { __syncthreads(); });
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < smem::kConsumerWarps; ++w) t += part[w];
    e_out[blockIdx.x] = e;
    if (n_out) n_out[blockIdx.x] = __dsqrt_rn(t);
  }
}

template <int S>
cudaError_t gate_s(const double* psi, int site, const double* u, double* out, cudaStream_t s) {
  constexpr int LA = S / 2, LB = S - S / 2;
  using D = smem::Dims<LA, LB>;
  const int bytes = 512 + 4 * D::PLANE * 8;
  auto k = apply_gate_smem_kernel<LA, LB>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  k<<<1, smem::kConsumers, bytes, s>>>(psi, site, u, out);
  return cudaGetLastError();
}

template <int S>
cudaError_t entropy_s(uint64_t count, const double* psi, double* e, double* n, bool fault,
                      cudaStream_t s, bool von_neumann) {
  constexpr int LA = S / 2, LB = S - S / 2;
  using D = smem::Dims<LA, LB>;
  if (von_neumann) {
    const int bytes = 2 * D::PLANE * 8 + 2 * D::DA_PAD * (D::DA_PAD + 4) * 8 + static_cast<int>(sizeof(vn::Scratch));
    auto k = entropy_vn_smem_kernel<LA, LB>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    k<<<static_cast<unsigned>(count), smem::kConsumers, bytes, s>>>(psi, e, n, fault);
    return cudaGetLastError();
  }
  const int bytes = 2 * D::PLANE * 8;
  auto k = entropy_smem_kernel<LA, LB>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  k<<<static_cast<unsigned>(count), smem::kConsumers, bytes, s>>>(psi, e, n, fault);
  return cudaGetLastError();
}

template <int NCHAIN>
__global__ void dmma_peak_kernel(double* out, int iters, long long* cycles) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NCHAIN][2];
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) c[i][0] = c[i][1] = 0.0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NCHAIN; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  const long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NCHAIN; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

}  // namespace

cudaError_t probe_rng(uint64_t seed, uint64_t p, uint64_t n, uint64_t* d_out, cudaStream_t s) {
  rng_kernel<<<1, 1, 0, s>>>(seed, p, n, d_out);
  return cudaGetLastError();
}

// The production pre-pass (gate_stream.cu) for one replica; records copied out.
cudaError_t probe_gates(uint32_t spins, uint64_t seed, uint64_t p, uint64_t steps, int initial,
                        uint8_t* d_sites, double* d_u, double* d_uacc, cudaStream_t s) {
  AnnealParams ap{};
  ap.spins = spins;
  ap.initial_state = initial;
  ap.steps = steps;
  ap.seed = seed;
  ap.t0 = 1.0;
  ap.t_min = 1e-3;
  ap.rows = 1;
  ap.p_first = p;
  ap.p_stride = 1;
  const size_t bytes = gate_stream_bytes_per_row(spins, steps, initial);
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, bytes, s);
  if (e != cudaSuccess) return e;
  GateStream gs{};
  e = launch_gate_stream(ap, ws, bytes, &gs, s);
  if (e == cudaSuccess && steps > 0) {
    probe_unpack_kernel<<<static_cast<unsigned>((steps + 127) / 128), 128, 0, s>>>(gs.recs, steps, d_sites, d_u, d_uacc);
    e = cudaGetLastError();
  }
  cudaFreeAsync(ws, s);
  return e;
}

cudaError_t probe_apply_gate(uint32_t spins, const double* psi, int site, const double* u,
                             double* out, cudaStream_t s) {
  switch (spins) {
    case 2: return gate_s<2>(psi, site, u, out, s);
    case 3: return gate_s<3>(psi, site, u, out, s);
    case 4: return gate_s<4>(psi, site, u, out, s);
    case 5: return gate_s<5>(psi, site, u, out, s);
    case 6: return gate_s<6>(psi, site, u, out, s);
    case 7: return gate_s<7>(psi, site, u, out, s);
    case 8: return gate_s<8>(psi, site, u, out, s);
    case 9: return gate_s<9>(psi, site, u, out, s);
    case 10: return gate_s<10>(psi, site, u, out, s);
    case 11: return gate_s<11>(psi, site, u, out, s);
    case 12: return gate_s<12>(psi, site, u, out, s);
    default: return hbm::probe_apply_gate(spins, psi, site, u, out, s);
  }
}

cudaError_t probe_entropy(uint32_t spins, uint64_t count, const double* psi, double* e,
                          double* n, bool fault, cudaStream_t s, bool von_neumann) {
  if (von_neumann && spins > static_cast<uint32_t>(kVnMaxSpins)) return cudaErrorInvalidValue;
  switch (spins) {
    case 2: return entropy_s<2>(count, psi, e, n, fault, s, von_neumann);
    case 3: return entropy_s<3>(count, psi, e, n, fault, s, von_neumann);
    case 4: return entropy_s<4>(count, psi, e, n, fault, s, von_neumann);
    case 5: return entropy_s<5>(count, psi, e, n, fault, s, von_neumann);
    case 6: return entropy_s<6>(count, psi, e, n, fault, s, von_neumann);
    case 7: return entropy_s<7>(count, psi, e, n, fault, s, von_neumann);
    case 8: return entropy_s<8>(count, psi, e, n, fault, s, von_neumann);
    case 9: return entropy_s<9>(count, psi, e, n, fault, s, von_neumann);
    case 10: return entropy_s<10>(count, psi, e, n, fault, s, von_neumann);
    case 11: return entropy_s<11>(count, psi, e, n, fault, s, von_neumann);
    case 12: return entropy_s<12>(count, psi, e, n, fault, s, von_neumann);
    default: return hbm::probe_entropy(spins, count, psi, e, n, fault, s, von_neumann);
  }
}

cudaError_t fp64_dmma_peak(double* tflops, double* clock_ghz) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  long long* cyc = nullptr;
  if (cudaMalloc(&d, 64) != cudaSuccess || cudaMalloc(&cyc, 8) != cudaSuccess)
    return cudaErrorMemoryAllocation;
  const int iters = 20000, warps = 8;
  dmma_peak_kernel<8><<<sms, warps * 32>>>(d, iters / 10, cyc);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  long long cycles = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dmma_peak_kernel<8><<<sms, warps * 32>>>(d, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) {
      best = ms;
      cudaMemcpy(&cycles, cyc, 8, cudaMemcpyDeviceToHost);
    }
  }
  cudaError_t err = cudaGetLastError();
  const double flops = 512.0 * 8 * iters * static_cast<double>(sms) * warps;
  *tflops = flops / (best * 1e-3) / 1e12;
  if (clock_ghz) *clock_ghz = static_cast<double>(cycles) / (best * 1e-3) / 1e9;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  cudaFree(cyc);
  return err;
}

}  // namespace tg
