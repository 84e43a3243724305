// anneal_hbm.cu — persistent annealing kernel, HBM/L2-resident tier (13 <= S <= 24).
// Same warp roles and step protocol as anneal_smem.cu; psi/psi' live in this CTA's
// workspace slab, rho tiles are staged through SMEM (hbm_tier.cuh).
#include "hbm_tier.cuh"
#include "tg_internal.h"

namespace tg {
namespace hbm {

__device__ void renormalize(const Geo& G, double* X, double* Y, int tid, int warp, int lane,
                            Header& H) {
  double s = 0.0;
  for (int i = tid; i < G.n; i += kConsumers) {
    const double x = __ldcg(X + i), y = __ldcg(Y + i);
    s = fma(x, x, s);
    s = fma(y, y, s);
  }
  s = warp_sum(s);
  if (lane == 0) H.part_tr[warp] = s;
  consumer_sync(kConsumers);
  double tot = 0.0;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) tot += H.part_tr[w];
  const double inv = __ddiv_rn(1.0, __dsqrt_rn(tot));
  for (int i = tid; i < G.n; i += kConsumers) {
    __stcg(X + i, __dmul_rn(__ldcg(X + i), inv));
    __stcg(Y + i, __dmul_rn(__ldcg(Y + i), inv));
  }
  __threadfence_block();
  consumer_sync(kConsumers);
}

__global__ void __launch_bounds__(kThreads, 1) anneal_hbm_kernel(const AnnealParams P) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Header& H = *reinterpret_cast<Header*>(smem_raw);
  double* stages = reinterpret_cast<double*>(smem_raw + kHeaderBytes);
  const Geo G(static_cast<int>(P.spins));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  double* slab = P.workspace + static_cast<size_t>(blockIdx.x) * 4 * G.n;
  auto PX = [&](int b) { return slab + (2 * b) * static_cast<size_t>(G.n); };
  auto PY = [&](int b) { return slab + (2 * b + 1) * static_cast<size_t>(G.n); };

  for (uint64_t r = blockIdx.x; r < P.rows; r += gridDim.x) {
    const GateRec* recs = P.gates + r * P.steps;
    if (P.initial_state == 0) {
      for (int i = tid; i < G.n; i += kConsumers) {  // product_state (spinmc.cpp:28-35)
        __stcg(PX(0) + i, i == 0 ? 1.0 : 0.0);
        __stcg(PY(0) + i, 0.0);
      }
    } else {  // random_state (spinmc.cpp:37-48), normals from the pre-pass
      const double* src = P.init_states + r * 2 * static_cast<size_t>(G.n);
      for (int i = tid; i < G.n; i += kConsumers) {
        __stcg(PX(0) + i, src[2 * i]);
        __stcg(PY(0) + i, src[2 * i + 1]);
      }
    }
    __threadfence_block();
    __syncthreads();
    int cur = 0;
    if (P.initial_state == 1) renormalize(G, PX(0), PY(0), tid, warp, lane, H);

    double rho2, tr;
    rho_partials(G, PX(cur), PY(cur), stages, tid, warp, lane, P.inject_fault != 0, rho2, tr);
    if (lane == 0) {
      H.part_rho[warp] = rho2;
      H.part_tr[warp] = tr;
    }
    consumer_sync(kConsumers);
    double cur_e = 0.0;
    if (tid == 0) {
      double a = 0.0, t = 0.0;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) {
        a += H.part_rho[w];
        t += H.part_tr[w];
      }
      H.error = 0;
      if (smem::not_normalized(t)) {
        H.error = 1;
        P.status[r] = kRowNotNormalized;
        P.status_step[r] = -1;
      } else {
        P.status[r] = kRowOk;
      }
      cur_e = smem::renyi2(a);
      P.initial_entropy[r] = cur_e;
    }
    consumer_sync(kConsumers);
    bool err = H.error != 0;

    int64_t t_prev = (tid == 0 && P.wall_ns) ? globaltimer() : 0;
    for (uint64_t s = 0; s < P.steps && !err; ++s) {
      const GateRec& g = recs[s];
      const int site = g.site;
      gate_pass(PX(cur), PY(cur), PX(cur ^ 1), PY(cur ^ 1), G.spins, site, g, tid, kConsumers);
      __threadfence_block();
      consumer_sync(kConsumers);
      rho_partials(G, PX(cur ^ 1), PY(cur ^ 1), stages, tid, warp, lane, P.inject_fault != 0,
                   rho2, tr);
      if (lane == 0) {
        H.part_rho[warp] = rho2;
        H.part_tr[warp] = tr;
      }
      consumer_sync(kConsumers);
      if (tid == 0) {
        double a = 0.0, t = 0.0;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) {
          a += H.part_rho[w];
          t += H.part_tr[w];
        }
        int acc = 0;
        if (smem::not_normalized(t)) {
          H.error = 1;
          P.status[r] = kRowNotNormalized;
          P.status_step[r] = static_cast<int64_t>(s);
        } else {
          const double proposed = smem::renyi2(a);
          const double delta = P.objective == 0 ? proposed - cur_e : cur_e - proposed;
          acc = g.u < acceptance(delta, g.temp);
          if (acc) cur_e = proposed;
        }
        H.decision = acc;
        const uint64_t o = r * P.steps + s;
        P.entropies[o] = cur_e;
        P.accepted[o] = static_cast<uint8_t>(acc);
        if (P.sites) P.sites[o] = static_cast<uint8_t>(site);
        if (P.wall_ns) {
          const int64_t t_now = globaltimer();
          P.wall_ns[o] = t_now - t_prev;
          t_prev = t_now;
        }
      }
      consumer_sync(kConsumers);
      err = H.error != 0;
      if (H.decision) cur ^= 1;
      if (!err && P.renorm > 0 && (s + 1) % P.renorm == 0)
        renormalize(G, PX(cur), PY(cur), tid, warp, lane, H);
    }
    if (tid == 0 && P.final_entropy) P.final_entropy[r] = cur_e;
    __syncthreads();  // the slab is rewritten by the next replica
  }
}

// ----------------------------------------------------------------------------- probes
__global__ void gate_probe_kernel(int spins, const double* psi, int site, const double* u,
                                  double* scratch, double* out) {
  __shared__ GateRec g;
  const int tid = threadIdx.x;
  const int n = 1 << spins;
  if (tid < 16) {
    const int x = tid >> 2, y = tid & 3;
    g.ur[tid] = u[2 * (x + 4 * y)];
    g.ui[tid] = u[2 * (x + 4 * y) + 1];
  }
  for (int i = tid; i < n; i += blockDim.x) {
    scratch[i] = psi[2 * i];
    scratch[n + i] = psi[2 * i + 1];
  }
  __threadfence_block();
  __syncthreads();
  gate_pass(scratch, scratch + n, scratch + 2 * n, scratch + 3 * n, spins, site, g, tid, blockDim.x);
  __threadfence_block();
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) {
    out[2 * i] = scratch[2 * n + i];
    out[2 * i + 1] = scratch[3 * n + i];
  }
}

__global__ void __launch_bounds__(kConsumers, 1) entropy_probe_kernel(int spins, const double* psi_all,
                                                                       double* scratch, double* e_out,
                                                                       double* n_out, bool fault) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ double part[2][kConsumerWarps];
  double* stages = reinterpret_cast<double*>(smem_raw);
  const Geo G(spins);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* psi = psi_all + 2ull * G.n * blockIdx.x;
  double* X = scratch + 2ull * G.n * blockIdx.x;
  double* Y = X + G.n;
  for (int i = tid; i < G.n; i += kConsumers) {
    X[i] = psi[2 * i];
    Y[i] = psi[2 * i + 1];
  }
  __threadfence_block();
  __syncthreads();
  double rho2, tr;
  rho_partials(G, X, Y, stages, tid, warp, lane, fault, rho2, tr);
  if (lane == 0) {
    part[0][warp] = rho2;
    part[1][warp] = tr;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, t = 0.0;
    for (int w = 0; w < kConsumerWarps; ++w) {
      a += part[0][w];
      t += part[1][w];
    }
    e_out[blockIdx.x] = smem::renyi2(a);
    if (n_out) n_out[blockIdx.x] = __dsqrt_rn(t);
  }
}

cudaError_t probe_apply_gate(uint32_t spins, const double* psi, int site, const double* u,
                             double* out, cudaStream_t s) {
  if (spins < 13 || spins > 24) return cudaErrorInvalidValue;
  double* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, sizeof(double) * 4 * (size_t{1} << spins), s);
  if (e != cudaSuccess) return e;
  gate_probe_kernel<<<1, kConsumers, 0, s>>>(static_cast<int>(spins), psi, site, u, scratch, out);
  e = cudaGetLastError();
  cudaFreeAsync(scratch, s);
  return e;
}

cudaError_t probe_entropy(uint32_t spins, uint64_t count, const double* psi, double* e_out,
                          double* n_out, bool fault, cudaStream_t s) {
  if (spins < 13 || spins > 24) return cudaErrorInvalidValue;
  double* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, sizeof(double) * 2 * (size_t{1} << spins) * count, s);
  if (e != cudaSuccess) return e;
  const int bytes = kStages * kStage * 8;
  cudaFuncSetAttribute(entropy_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  entropy_probe_kernel<<<static_cast<unsigned>(count), kConsumers, bytes, s>>>(
      static_cast<int>(spins), psi, scratch, e_out, n_out, fault);
  e = cudaGetLastError();
  cudaFreeAsync(scratch, s);
  return e;
}

}  // namespace hbm

size_t anneal_hbm_workspace_bytes(uint32_t spins, uint64_t rows, int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const uint64_t grid = rows < static_cast<uint64_t>(sms) ? rows : static_cast<uint64_t>(sms);
  return static_cast<size_t>(grid) * 4 * (size_t{1} << spins) * sizeof(double);
}

cudaError_t launch_anneal_hbm(const AnnealParams& p, cudaStream_t stream, int* grid_out) {
  if (p.spins < 13 || p.spins > 24) return cudaErrorInvalidValue;
  if (!p.workspace) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(hbm::anneal_hbm_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, hbm::kSmemBytes);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = static_cast<int>(p.rows < static_cast<uint64_t>(sms) ? p.rows : sms);
  if (grid_out) *grid_out = grid;
  if (grid == 0) return cudaSuccess;
  hbm::anneal_hbm_kernel<<<grid, hbm::kThreads, hbm::kSmemBytes, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace tg
