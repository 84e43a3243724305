// anneal_smem.cu — persistent annealing kernel, SMEM-resident tier (2 <= S <= 12).
//
// One CTA owns one replica at a time for its whole trajectory (replicas never
// communicate); the grid is sized to the resident-CTA count and loops over
// rows. Warp roles:
//   warp 8      producer: owns the replica's xoshiro256++ stream and writes the
//               data-independent proposal stream (site, Haar U, u_accept, T(s)) into an
//               8-slot SMEM ring (mbarrier full/empty), steps ahead of the consumers;
//   warps 0..7  consumers: gate pass psi -> psi' (SMEM), rho = Psi' Psi'^dagger on
//               DMMA.8x8x4 with fused ||rho||_F^2 and trace, Metropolis decision
//               (thread 0), buffer swap, renormalisation every `renorm` steps.
// Per step this replaces metropolis_step (spinmc.cpp:193-213); per replica mc_procedure
// (spinmc.cpp:215-251). No host round trip between steps.
#include "smem_tier.cuh"
#include "tg_internal.h"

namespace tg {
namespace smem {

// Random initial state (spinmc.cpp:37-48): 2^S normal pairs from the replica stream, in
// amplitude order, written into plane pair (X, Y). Producer warp; all lanes share state.
template <class D>
__device__ void fill_random(Xoshiro& st, int lane, double* X, double* Y) {
  constexpr int PPC = D::N < 16 ? D::N : 16;  // pairs per chunk
  for (int c = 0; c < D::N / PPC; ++c) {
    uint64_t d1 = 0, d2 = 0;
    for (int j = 0; j < 2 * PPC; ++j) {
      const uint64_t x = next_u64(st);
      if (j == 2 * lane) d1 = x;
      if (j == 2 * lane + 1) d2 = x;
    }
    if (lane < PPC) {
      double a, b;
      box_muller(d1, d2, a, b);
      const int ph = D::phys(c * PPC + lane);
      X[ph] = a;
      Y[ph] = b;
    }
  }
}

// renormalize (spinmc.cpp:56-59): inv = 1/||psi||; amp *= inv. Consumers only.
template <class D>
__device__ void renormalize(double* X, double* Y, int tid, int warp, int lane, Header& H) {
  double s = 0.0;
  for (int idx = tid; idx < D::N; idx += kConsumers) {
    const int ph = D::phys(idx);
    s = fma(X[ph], X[ph], s);
    s = fma(Y[ph], Y[ph], s);
  }
  s = warp_sum(s);
  if (lane == 0) H.part_tr[warp] = s;
  consumer_sync(kConsumers);
  double tot = 0.0;
#pragma unroll
  for (int w = 0; w < kConsumerWarps; ++w) tot += H.part_tr[w];
  const double inv = __ddiv_rn(1.0, __dsqrt_rn(tot));
  for (int idx = tid; idx < D::N; idx += kConsumers) {
    const int ph = D::phys(idx);
    X[ph] = __dmul_rn(X[ph], inv);
    Y[ph] = __dmul_rn(Y[ph], inv);
  }
  consumer_sync(kConsumers);
}

template <int LA, int LB, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) anneal_smem_kernel(const AnnealParams P) {
  using D = Dims<LA, LB>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  Header& H = *reinterpret_cast<Header*>(smem_raw);
  double* planes = reinterpret_cast<double*>(smem_raw + kHeaderBytes);
  auto PX = [&](int b) { return planes + (2 * b) * D::PLANE; };
  auto PY = [&](int b) { return planes + (2 * b + 1) * D::PLANE; };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool producer = warp == kConsumerWarps;
  if (tid == 0) {
    for (int i = 0; i < kRing; ++i) {
      mbar_init(&H.full[i], 1);
      mbar_init(&H.empty[i], 1);
    }
  }
  __syncthreads();

  uint64_t gseq = 0;  // gates produced/consumed by this CTA (ring phase tracking)
  for (uint64_t r = blockIdx.x; r < P.rows; r += gridDim.x) {
    const uint64_t p = P.p_first + r * P.p_stride;
    if (producer) {
      Xoshiro st = stream_init(P.seed, p);
      __syncthreads();  // A: consumers zeroed both buffers
      if (P.initial_state == 1) fill_random<D>(st, lane, PX(0), PY(0));
      __syncthreads();  // B: initial state in buffer 0
      for (uint64_t s = 0; s < P.steps; ++s, ++gseq) {
        const int slot = static_cast<int>(gseq % kRing);
        const uint32_t par = static_cast<uint32_t>((gseq / kRing) & 1);
        mbar_wait(&H.empty[slot], par ^ 1u);
        const double temp = temperature(P.t0, P.t_min, s, P.steps);
        produce_gate(st, lane, D::S, &H.ring[slot], temp);
        __syncwarp();
        if (lane == 0) mbar_arrive(&H.full[slot]);
      }
      continue;
    }

    // ------------------------------------------------------------------ consumers
    for (int i = tid; i < 4 * D::PLANE; i += kConsumers) planes[i] = 0.0;
    __syncthreads();  // A
    if (P.initial_state == 0 && tid == 0) PX(0)[0] = 1.0;  // product_state (spinmc.cpp:28-35)
    __syncthreads();  // B
    int cur = 0;
    if (P.initial_state == 1) renormalize<D>(PX(0), PY(0), tid, warp, lane, H);

    // initial entropy: one extra GEMM per replica (spinmc.cpp:234)
    double rho2, tr;
    rho_partials<D>(PX(cur), PY(cur), warp, lane, P.inject_fault != 0, rho2, tr);
    if (lane == 0) {
      H.part_rho[warp] = rho2;
      H.part_tr[warp] = tr;
    }
    consumer_sync(kConsumers);
    double cur_e = 0.0;  // meaningful in thread 0 only
    if (tid == 0) {
      double a = 0.0, t = 0.0;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) {
        a += H.part_rho[w];
        t += H.part_tr[w];
      }
      H.error = 0;
      if (not_normalized(t)) {
        H.error = 1;
        P.status[r] = kRowNotNormalized;
        P.status_step[r] = -1;
      } else {
        P.status[r] = kRowOk;
      }
      cur_e = renyi2(a);
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
      gate_pass<D>(PX(cur), PY(cur), PX(cur ^ 1), PY(cur ^ 1), site, g, tid, kConsumers);
      consumer_sync(kConsumers);
      if (tid == 0) mbar_arrive(&H.empty[slot]);  // every consumer has read the slot
      rho_partials<D>(PX(cur ^ 1), PY(cur ^ 1), warp, lane, P.inject_fault != 0, rho2, tr);
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
        if (not_normalized(t)) {
          H.error = 1;
          P.status[r] = kRowNotNormalized;
          P.status_step[r] = static_cast<int64_t>(s);
        } else {
          const double proposed = renyi2(a);
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
        renormalize<D>(PX(cur), PY(cur), tid, warp, lane, H);
    }
    if (tid == 0 && P.final_entropy) P.final_entropy[r] = cur_e;
  }
}

template <int S>
cudaError_t launch_s(const AnnealParams& p, cudaStream_t stream, int* grid_out) {
  constexpr int LA = S / 2, LB = S - S / 2;
  constexpr int MINB = S >= 12 ? 1 : 2;
  constexpr int bytes = smem_bytes<LA, LB>();
  auto kern = anneal_smem_kernel<LA, LB, MINB>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, bytes);
  if (e != cudaSuccess) return e;
  if (occ < 1) return cudaErrorInvalidConfiguration;
  const uint64_t cap = static_cast<uint64_t>(sms) * occ;
  const int grid = static_cast<int>(p.rows < cap ? p.rows : cap);
  if (grid_out) *grid_out = grid;
  if (grid == 0) return cudaSuccess;
  kern<<<grid, kThreads, bytes, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace smem

cudaError_t launch_anneal_smem(const AnnealParams& p, cudaStream_t stream, int* grid_out) {
  switch (p.spins) {
    case 2: return smem::launch_s<2>(p, stream, grid_out);
    case 3: return smem::launch_s<3>(p, stream, grid_out);
    case 4: return smem::launch_s<4>(p, stream, grid_out);
    case 5: return smem::launch_s<5>(p, stream, grid_out);
    case 6: return smem::launch_s<6>(p, stream, grid_out);
    case 7: return smem::launch_s<7>(p, stream, grid_out);
    case 8: return smem::launch_s<8>(p, stream, grid_out);
    case 9: return smem::launch_s<9>(p, stream, grid_out);
    case 10: return smem::launch_s<10>(p, stream, grid_out);
    case 11: return smem::launch_s<11>(p, stream, grid_out);
    case 12: return smem::launch_s<12>(p, stream, grid_out);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tg
