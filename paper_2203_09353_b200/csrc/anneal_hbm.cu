// anneal_hbm.cu — persistent annealing kernel, HBM/L2-resident tier (13 <= S <= 24).
// Same warp roles and step protocol as anneal_smem.cu; psi/psi' live in this CTA's
// workspace slab, rho tiles are staged through SMEM (hbm_tier.cuh).
#include "hbm_tier.cuh"
#include "tg_internal.h"

namespace tg {
namespace hbm {

__device__ void fill_random(const Geo& G, Xoshiro& st, int lane, double* X, double* Y) {
  for (int c = 0; c < G.n / 16; ++c) {
    uint64_t d1 = 0, d2 = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const uint64_t x = next_u64(st);
      if (j == 2 * lane) d1 = x;
      if (j == 2 * lane + 1) d2 = x;
    }
    if (lane < 16) {
      double a, b;
      box_muller(d1, d2, a, b);
      X[c * 16 + lane] = a;
      Y[c * 16 + lane] = b;
    }
  }
}

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
  const bool producer = warp == kConsumerWarps;
  double* slab = P.workspace + static_cast<size_t>(blockIdx.x) * 4 * G.n;
  auto PX = [&](int b) { return slab + (2 * b) * static_cast<size_t>(G.n); };
  auto PY = [&](int b) { return slab + (2 * b + 1) * static_cast<size_t>(G.n); };

  if (tid == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&H.full[i], 1);
      mbar_init(&H.empty[i], 1);
    }
  }
  __syncthreads();

  uint64_t gseq = 0;
  for (uint64_t r = blockIdx.x; r < P.rows; r += gridDim.x) {
    const uint64_t p = P.p_first + r * P.p_stride;
    if (producer) {
      Xoshiro st = stream_init(P.seed, p);
      __syncthreads();  // A
      if (P.initial_state == 1) {
        fill_random(G, st, lane, PX(0), PY(0));
        __threadfence_block();
      }
      __syncthreads();  // B
      for (uint64_t s = 0; s < P.steps; ++s, ++gseq) {
        const int slot = static_cast<int>(gseq % kRing);
        const uint32_t par = static_cast<uint32_t>((gseq / kRing) & 1);
        mbar_wait(&H.empty[slot], par ^ 1u);
        const double temp = temperature(P.t0, P.t_min, s, P.steps);
        produce_gate(st, lane, G.spins, &H.ring[slot], temp);
        __syncwarp();
        if (lane == 0) mbar_arrive(&H.full[slot]);
      }
      continue;
    }

    if (P.initial_state == 0) {
      for (int i = tid; i < G.n; i += kConsumers) {
        __stcg(PX(0) + i, i == 0 ? 1.0 : 0.0);
        __stcg(PY(0) + i, 0.0);
      }
      __threadfence_block();
    }
    __syncthreads();  // A
    __syncthreads();  // B
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

    for (uint64_t s = 0; s < P.steps; ++s, ++gseq) {
      const int slot = static_cast<int>(gseq % kRing);
      const uint32_t par = static_cast<uint32_t>((gseq / kRing) & 1);
      mbar_wait(&H.full[slot], par);
      const GateSlot& g = H.ring[slot];
      if (err) {
        if (tid == 0) mbar_arrive(&H.empty[slot]);
        continue;
      }
      int64_t t_start = 0;
      if (tid == 0 && P.wall_ns) t_start = globaltimer();
      const int site = g.site;
      const double uacc = g.uacc, temp = g.temp;
      gate_pass(PX(cur), PY(cur), PX(cur ^ 1), PY(cur ^ 1), G.spins, site, g, tid, kConsumers);
      __threadfence_block();
      consumer_sync(kConsumers);
      if (tid == 0) mbar_arrive(&H.empty[slot]);
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
          acc = uacc < acceptance(delta, temp);
          if (acc) cur_e = proposed;
        }
        H.decision = acc;
        const uint64_t o = r * P.steps + s;
        P.entropies[o] = cur_e;
        P.accepted[o] = static_cast<uint8_t>(acc);
        if (P.sites) P.sites[o] = static_cast<uint8_t>(site);
        if (P.wall_ns) P.wall_ns[o] = globaltimer() - t_start;
      }
      consumer_sync(kConsumers);
      err = H.error != 0;
      if (H.decision) cur ^= 1;
      if (!err && P.renorm > 0 && (s + 1) % P.renorm == 0)
        renormalize(G, PX(cur), PY(cur), tid, warp, lane, H);
    }
    if (tid == 0 && P.final_entropy) P.final_entropy[r] = cur_e;
  }
}

// ----------------------------------------------------------------------------- probes
__global__ void gate_probe_kernel(int spins, const double* psi, int site, const double* u,
                                  double* scratch, double* out) {
  __shared__ GateSlot g;
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
                                                                       double* n_out) {
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
  rho_partials(G, X, Y, stages, tid, warp, lane, false, rho2, tr);
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
                          double* n_out, cudaStream_t s) {
  if (spins < 13 || spins > 24) return cudaErrorInvalidValue;
  double* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, sizeof(double) * 2 * (size_t{1} << spins) * count, s);
  if (e != cudaSuccess) return e;
  const int bytes = kStages * kStage * 8;
  cudaFuncSetAttribute(entropy_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  entropy_probe_kernel<<<static_cast<unsigned>(count), kConsumers, bytes, s>>>(
      static_cast<int>(spins), psi, scratch, e_out, n_out);
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
