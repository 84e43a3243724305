// anneal_hbm.cu — persistent annealing kernel, HBM/L2-resident tier (13 <= S <= 24).
//
// A cluster of CS CTAs (1, 2 or 4, see hbm_tier.cuh) owns one replica at a time; its psi /
// psi' slabs live in the workspace. Per step (metropolis_step, spinmc.cpp:193-213):
//   gate pass  — rank k applies U to its 1/CS of the groups (reference rounding), global
//                -> global; cluster barrier;
//   GEMM       — rho tiles t = k (mod CS) on DMMA, fused ||rho||_F^2 and trace in four
//                canonical chains; per-rank chain values exchanged through DSMEM; cluster
//                barrier;
//   decision   — thread 0 of every rank evaluates the same reference formula on the same
//                totals (identical results); rank 0 writes the trace.
// Every FP64 op outside the GEMM runs while no DMMA is in flight on the SM (the FP64 pipe
// is shared, profiles/r01_fp64_contention.txt). The proposal stream comes from the
// pre-pass (gate_stream.cu).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "hbm_queue.cuh"
#include "hbm_tier.cuh"
#include "tg_internal.h"
#include "vn.cuh"
#include "vn_packed.cuh"

namespace tg {
namespace hbm {

// von Neumann (KIND 1, S = 13: d_a = 64 = one tile, CS = 1): rho planes (pitch 68) and the
// solver scratch reuse the stage buffers once the GEMM pipeline has drained.
constexpr int kRP = TB + 4;
static_assert(2 * TB * kRP * 8 + static_cast<int>(sizeof(vn::Scratch)) <= kStages * kStage * 8, "vN region");
// von Neumann at S = 14, 15 (d_a = 128): packed lower Hermitian part + solver scratch in the
// drained stages (vn_packed.cuh); rho itself goes through the slab's extra planes.
constexpr int kPackedN = vnp::kMaxN;
constexpr int kPackedPlane = (vnp::packed_size(kPackedN) + 15) / 16 * 16;
static_assert(2 * kPackedPlane * 8 + static_cast<int>(sizeof(vnp::Scratch)) <= kStages * kStage * 8, "vN packed region");

// TRACE: phase stamps (clock64) of the first cluster's first replica into P.trace[steps][8]:
// 0 step start, 1 gate pass done, 2 GEMM done, 3 decision done (profiling probe only).
// KIND: 0 Renyi-2, 1 von Neumann (S = 13, CS = 1; vn.cuh after the GEMM).
// TMA (KIND 0): the GEMM stages are filled by the TMA engine from `tmap` (hbm_tensor_map,
// rho_partials_tma) instead of per-thread cp.async.
template <bool TRACE, int CS, int KIND, bool TMA>
__global__ void __launch_bounds__(kThreads, 1) anneal_hbm_kernel(const AnnealParams P,
                                                                 const __grid_constant__ CUtensorMap tmap) {
  static_assert(KIND == 0 || CS == 1, "von Neumann runs one CTA per replica");
  static_assert(KIND == 0 || !TMA, "the TMA pipeline is the Renyi-2 GEMM");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  HHeader& H = *reinterpret_cast<HHeader*>(smem_raw);
  const uint32_t sbase = smem_u32(smem_raw);
  double* stages = reinterpret_cast<double*>(smem_raw + (((sbase + kHHeaderBytes + 1023u) & ~1023u) - sbase));
  double* Rr = stages;  // KIND 1 only (aliases the drained stages)
  double* Ri = stages + TB * kRP;
  vn::Scratch& VW = *reinterpret_cast<vn::Scratch*>(stages + 2 * TB * kRP);
  const Geo G0(static_cast<int>(P.spins));
  const bool packed = KIND == 1 && G0.da > TB;
  double* Rg = nullptr;  // packed: global rho of the cluster (after its slab)
  if (packed) Rg = P.workspace + static_cast<size_t>(blockIdx.x) * (4 * static_cast<size_t>(G0.n) +
                                                                    2 * static_cast<size_t>(G0.da) * G0.da) +
                   4 * static_cast<size_t>(G0.n);
  // KIND 0: the trace value of a proposal is its raw ||rho||_F^2 (finish_renyi_kernel turns
  // it into -log(f*f) after the kernel, as in the SMEM tier) and the decision is the lean
  // smem::decide on rho2 (one multiply, reference formula near ties). KIND 1: the entropy
  // of the proposal whose rho the last GEMM produced (valid in thread 0).
  auto entropy_of = [&](double rho2) -> double {
    if constexpr (KIND == 0) {
      return rho2;
    } else {
      if (packed) {
        double* Ar = stages;
        double* Ai = stages + kPackedPlane;
        vnp::Scratch& PW = *reinterpret_cast<vnp::Scratch*>(stages + 2 * kPackedPlane);
        __threadfence_block();
        __syncthreads();  // every tile of rho is in Rg
        vnp::build(Rg, Rg + static_cast<size_t>(G0.da) * G0.da, Ar, Ai, G0.da, threadIdx.x);
        __syncthreads();
        return vnp::entropy(Ar, Ai, G0.da, PW, threadIdx.x, [] { __syncthreads(); });
      }
      return vn::entropy(Rr, Ri, TB, kRP, VW, threadIdx.x, [] { __syncthreads(); });
    }
  };
  const Geo G(static_cast<int>(P.spins));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = CS == 1 ? 0u : cluster_rank();
  const uint64_t cid = blockIdx.x / CS, ncl = gridDim.x / CS;
  double* slab = P.workspace + static_cast<size_t>(cid) * (4 * static_cast<size_t>(G.n) +
                                                         (packed ? 2 * static_cast<size_t>(G.da) * G.da : 0));
  auto PX = [&](int b) { return slab + (2 * b) * static_cast<size_t>(G.n); };
  auto PY = [&](int b) { return slab + (2 * b + 1) * static_cast<size_t>(G.n); };
  TmaPipe pipe{H.full, H.empty, 0};
  if constexpr (TMA) {
    if (tid == 0) {
      for (int s = 0; s < kStages; ++s) {
        mbar_init(&H.full[s], 1);
        mbar_init(&H.empty[s], kWarps);
      }
      for (int s = 0; s < 8; ++s) mbar_init(&H.gfull[s], 1);
      fence_mbar_init();
    }
    __syncthreads();
  }
  int64_t* gprof = nullptr;  // TRACE: GEMM-internal clocks of the current step (slots 4..6)
  auto gemm = [&](int b, int first, int stride, double out[2 * kChains]) {  // rho of buffer b
    if constexpr (TMA) {
      rho_partials_tma(G, &tmap, b, static_cast<int>(cid), stages, pipe, tid, warp, lane, first, stride,
                       P.inject_fault != 0, PX(b), PY(b), out, gprof);
    } else {
      rho_partials<KIND == 1>(G, PX(b), PY(b), stages, tid, warp, lane, first, stride, P.inject_fault != 0, out,
                              Rr, Ri, kRP, gprof, Rg);
    }
  };
  auto mark = [&](uint64_t r, uint64_t s, int k) {
    if (TRACE && tid == 0 && rank == 0 && r == 0 && s < P.steps) P.trace[s * 8 + k] = clock64();
  };
  const int groups = G.n / 4;
  const int g0 = static_cast<int>(rank) * (groups / CS), g1 = g0 + groups / CS;
  const int first = static_cast<int>(rank), stride = CS;
  const bool writer = rank == 0;
  const bool light_fence = P.light_fence != 0;
  // S >= 16: each CTA's share of the gate pass is staged through its stage buffers by the TMA
  // engine (gate_pass_bulk). (Starting the CTAs a quarter step apart, so that their gate passes
  // do not hit HBM together, was measured on top of it and changed nothing.)
  const int gate_chunk = P.gate_chunk > 0 ? P.gate_chunk : kGateChunk;
  const bool bulk_gate = TMA && KIND == 0 && G0.spins >= P.gate_bulk_min && P.gate_bulk != 0 &&
                         (G0.n / 4 / CS) % gate_chunk == 0;
  uint32_t gpar = 0;

  for (uint64_t r = cid; r < P.rows; r += ncl) {
    const int64_t t_row0 = (tid == 0 && writer && P.initial_wall_ns) ? globaltimer() : 0;
    const GateRec* recs = P.gates + r;  // record s at recs[s * rows] (gate_stream.cu layout)
    // record s is copied to H.rec[s & 1] while the previous GEMM runs (an HBM miss on the
    // step's critical path otherwise); 18 threads x 16 B
    auto prefetch_rec = [&](uint64_t s) {
      if (s < P.steps && tid < static_cast<int>(sizeof(GateRec) / 16)) {
        cp_async16(reinterpret_cast<char*>(&H.rec[s & 1]) + 16 * tid,
                   reinterpret_cast<const char*>(recs + s * P.rows) + 16 * tid);
        cp_async_commit();
      }
    };
    {  // initial state, split by halves of the amplitude index
      const int i0 = static_cast<int>(rank) * (G.n / CS), i1 = i0 + G.n / CS;
      if (P.initial_state == 0) {
        for (int i = i0 + tid; i < i1; i += kThreads) {  // product_state (spinmc.cpp:28-35)
          __stcg(PX(0) + i, i == 0 ? 1.0 : 0.0);
          __stcg(PY(0) + i, 0.0);
        }
      } else {  // random_state (spinmc.cpp:37-48), normals from the pre-pass
        const double* src = P.init_states + r * 2 * static_cast<size_t>(G.n);
        for (int i = i0 + tid; i < i1; i += kThreads) {
          __stcg(PX(0) + i, src[2 * i]);
          __stcg(PY(0) + i, src[2 * i + 1]);
        }
      }
      __threadfence();
      fence_proxy_async_global();
      sync_all<CS>();
    }
    int cur = 0;
    if (P.initial_state == 1) renormalize<CS>(G, PX(0), PY(0), tid, warp, lane, rank, H);

    double out[2 * kChains], rho2, tr;
    prefetch_rec(0);
    gemm(cur, first, stride, out);
    cp_async_wait<0>();  // record 0 (visible after publish_vals' barriers)
    if (lane == 0)
      for (int c = 0; c < 2 * kChains; ++c) H.part[warp][c] = out[c];
    publish_vals<CS>(H, tid, rank);
    totals<CS>(H, rho2, tr);
    double cur_e = entropy_of(rho2);  // spinmc.cpp:234 (thread 0)
    bool err = smem::not_normalized(tr);
    if (tid == 0 && writer) {
      P.status[r] = err ? kRowNotNormalized : kRowOk;
      if (err) P.status_step[r] = -1;
      if (err && P.status_norm) P.status_norm[r] = __dsqrt_rn(tr);
      P.initial_entropy[r] = cur_e;
    }

    int64_t t_prev = (tid == 0 && (P.wall_ns || P.initial_wall_ns)) ? globaltimer() : 0;
    if (tid == 0 && writer && P.initial_wall_ns) P.initial_wall_ns[r] = t_prev - t_row0;
    uint64_t renorm_left = P.renorm;  // countdown: no 64-bit modulo per step
    for (uint64_t s = 0; s < P.steps && !err; ++s) {
      const GateRec& g = H.rec[s & 1];
      mark(r, s, 0);
      if (bulk_gate)
        gate_pass_bulk(PX(cur), PY(cur), PX(cur ^ 1), PY(cur ^ 1), g.site, g, g0, g1, tid, stages, H.gfull, gpar,
                       gate_chunk);
      else
        gate_pass(PX(cur), PY(cur), PX(cur ^ 1), PY(cur ^ 1), g.site, g, g0, g1, tid, kThreads);
      // psi' is read by the cluster's CTAs after the barrier (bar.sync / barrier.cluster
      // release-acquire order the generic-proxy writes; no GPU-scope fence needed) and, with
      // TMA, through the async proxy
      if constexpr (TMA) fence_proxy_async_global();
      if (!light_fence) __threadfence();
      sync_all<CS>();
      mark(r, s, 1);
      if (TRACE && rank == 0 && r == 0 && s < P.steps) gprof = P.trace + s * 8 + 4;
      prefetch_rec(s + 1);
      gemm(cur ^ 1, first, stride, out);
      cp_async_wait<0>();
      gprof = nullptr;
      if (lane == 0)
        for (int c = 0; c < 2 * kChains; ++c) H.part[warp][c] = out[c];
      publish_vals<CS>(H, tid, rank);
      totals<CS>(H, rho2, tr);
      const double e_new = entropy_of(rho2);
      mark(r, s, 2);
      if (tid == 0) {  // every rank decides identically; rank 0 writes
        int acc = 0;
        if (smem::not_normalized(tr)) {
          H.error = 1;
          if (writer) {
            P.status[r] = kRowNotNormalized;
            P.status_step[r] = static_cast<int64_t>(s);
            if (P.status_norm) P.status_norm[r] = __dsqrt_rn(tr);
          }
        } else {
          H.error = 0;
          const double proposed = e_new;
          // KIND 0: lean decision on rho2; KIND 1: spinmc.cpp:203-207 verbatim
          const smem::Verdict v = KIND == 0 ? smem::decide_audit(proposed, cur_e, g, P.objective, P.tie_eps)
                                            : smem::decide_reference(proposed, cur_e, g, P.objective, P.tie_eps);
          acc = v.acc;
          if (writer) smem::audit(P, r, s, g, v);
          if (acc) cur_e = proposed;
        }
        H.decision = acc;
        if (writer) {
          const uint64_t o = r * P.steps + s;
          P.entropies[o] = cur_e;
          P.accepted[o] = static_cast<uint8_t>(acc);
          if (P.sites) P.sites[o] = static_cast<uint8_t>(g.site);
          if (P.wall_ns) {
            const int64_t t_now = globaltimer();
            P.wall_ns[o] = t_now - t_prev;
            t_prev = t_now;
          }
        }
        mark(r, s, 3);
      }
      __syncthreads();
      err = H.error != 0;
      if (H.decision) cur ^= 1;
      if (P.renorm > 0 && --renorm_left == 0) {  // (s + 1) % renorm == 0, spinmc.cpp:246-248
        renorm_left = P.renorm;
        if (!err) renormalize<CS>(G, PX(cur), PY(cur), tid, warp, lane, rank, H);
      }
    }
    if (tid == 0 && writer && P.final_entropy) P.final_entropy[r] = cur_e;
    sync_all<CS>();  // the slab is rewritten by the cluster's next replica
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
  gate_pass(scratch, scratch + n, scratch + 2 * n, scratch + 3 * n, site, g, 0, n / 4, tid, blockDim.x);
  __threadfence_block();
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) {
    out[2 * i] = scratch[2 * n + i];
    out[2 * i + 1] = scratch[3 * n + i];
  }
}

template <int KIND>
__global__ void __launch_bounds__(kThreads, 1) entropy_probe_kernel(int spins, const double* psi_all,
                                                                     double* scratch, double* e_out,
                                                                     double* n_out, bool fault) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  HHeader& H = *reinterpret_cast<HHeader*>(smem_raw);
  double* stages = reinterpret_cast<double*>(smem_raw + kHHeaderBytes);
  const Geo G(spins);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const double* psi = psi_all + 2ull * G.n * blockIdx.x;
  double* X = scratch + 2ull * G.n * blockIdx.x;
  double* Y = X + G.n;
  for (int i = tid; i < G.n; i += kThreads) {
    X[i] = psi[2 * i];
    Y[i] = psi[2 * i + 1];
  }
  __threadfence_block();
  __syncthreads();
  double out[2 * kChains];
  double* Rr = stages;
  double* Ri = stages + TB * kRP;
  const bool packed = KIND == 1 && G.da > TB;
  double* Rg = packed ? scratch + 2ull * G.n * gridDim.x + 2ull * G.da * G.da * blockIdx.x : nullptr;
  rho_partials<KIND == 1>(G, X, Y, stages, tid, warp, lane, 0, 1, fault, out, Rr, Ri, kRP, nullptr, Rg);
  if (lane == 0)
    for (int c = 0; c < 2 * kChains; ++c) H.part[warp][c] = out[c];
  publish_vals<1>(H, tid, 0);
  double rho2, tr;
  totals<1>(H, rho2, tr);
  double e = 0.0;
  if constexpr (KIND == 1) {
    if (packed) {
      double* Ar = stages;
      double* Ai = stages + kPackedPlane;
      vnp::Scratch& PW = *reinterpret_cast<vnp::Scratch*>(stages + 2 * kPackedPlane);
      __threadfence_block();
      __syncthreads();
      vnp::build(Rg, Rg + static_cast<size_t>(G.da) * G.da, Ar, Ai, G.da, tid);
      __syncthreads();
      e = vnp::entropy(Ar, Ai, G.da, PW, tid, [] { __syncthreads(); });
    } else {
      vn::Scratch& W = *reinterpret_cast<vn::Scratch*>(stages + 2 * TB * kRP);
      e = vn::entropy(Rr, Ri, TB, kRP, W, tid, [] { __syncthreads(); });
    }
  } else {
    e = smem::renyi2(rho2);
  }
  if (tid == 0) {
    e_out[blockIdx.x] = e;
    if (n_out) n_out[blockIdx.x] = __dsqrt_rn(tr);
  }
}

cudaError_t probe_apply_gate(uint32_t spins, const double* psi, int site, const double* u,
                             double* out, cudaStream_t s) {
  if (spins < 13 || spins > 24) return cudaErrorInvalidValue;
  double* scratch = nullptr;
  cudaError_t e = cudaMallocAsync(&scratch, sizeof(double) * 4 * (size_t{1} << spins), s);
  if (e != cudaSuccess) return e;
  gate_probe_kernel<<<1, kThreads, 0, s>>>(static_cast<int>(spins), psi, site, u, scratch, out);
  e = cudaGetLastError();
  cudaFreeAsync(scratch, s);
  return e;
}

cudaError_t probe_entropy(uint32_t spins, uint64_t count, const double* psi, double* e_out,
                          double* n_out, bool fault, cudaStream_t s, bool von_neumann) {
  if (spins < 13 || spins > 24) return cudaErrorInvalidValue;
  if (von_neumann && spins > static_cast<uint32_t>(kVnMaxSpins)) return cudaErrorInvalidValue;
  double* scratch = nullptr;
  const size_t da = size_t{1} << (spins / 2);
  const size_t per = 2 * (size_t{1} << spins) + (von_neumann && da > TB ? 2 * da * da : 0);
  cudaError_t e = cudaMallocAsync(&scratch, sizeof(double) * per * count, s);
  if (e != cudaSuccess) return e;
  auto k = von_neumann ? entropy_probe_kernel<1> : entropy_probe_kernel<0>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  k<<<static_cast<unsigned>(count), kThreads, kSmemBytes, s>>>(static_cast<int>(spins), psi, scratch, e_out,
                                                              n_out, fault);
  e = cudaGetLastError();
  cudaFreeAsync(scratch, s);
  return e;
}

// CTAs per replica. Small batches (cs * rows <= SMs for some cs > 1): the largest cs in
// {2, 4} (at most the replica's 64x64 tile count, 2 always allowed) that still fits one
// wave, since otherwise SMs idle. Larger batches: 1, or 2 when that removes a partial last
// wave worth >= 2% of the machine (e.g. 512 replicas on 148 SMs: 86.5% -> 98.8%). A
// 4-CTA replica is far less efficient per SM than a 1-CTA one (one 64x64 tile per CTA at
// S = 14: fixed per-step costs dominate), so it is only worth it while SMs would idle.
// TG_HBM_CTAS_PER_REPLICA=1|2|4 overrides (tests check they agree bitwise).
int ctas_per_replica(uint32_t spins, uint64_t rows, int sms, int entropy_kind) {
  if (entropy_kind == 0) return 1;  // von Neumann: the eigen-solver runs in one CTA
  const int tiles = 1 << (2 * (static_cast<int>(spins) / 2 - 6));
  if (const char* env = std::getenv("TG_HBM_CTAS_PER_REPLICA")) {
    const int v = std::atoi(env);
    if (v == 1 || v == 2 || v == 4) return v;
  }
  if (rows == 0) return 1;
  for (int cs = kMaxCS; cs >= 2; cs /= 2)
    if ((cs <= tiles || cs == 2) && static_cast<uint64_t>(cs) * rows <= static_cast<uint64_t>(sms)) return cs;
  auto eff = [&](uint64_t units) {
    const uint64_t waves = (units + sms - 1) / sms;
    return static_cast<double>(units) / static_cast<double>(waves * sms);
  };
  return eff(2 * rows) > eff(rows) + 0.02 ? 2 : 1;
}

}  // namespace hbm

namespace {

using HbmKernel = void (*)(AnnealParams, CUtensorMap);
template <bool TMA>
HbmKernel hbm_kernel_renyi(int cs, bool trace) {
  using namespace hbm;
  if (cs == 1) return trace ? anneal_hbm_kernel<true, 1, 0, TMA> : anneal_hbm_kernel<false, 1, 0, TMA>;
  if (cs == 2) return trace ? anneal_hbm_kernel<true, 2, 0, TMA> : anneal_hbm_kernel<false, 2, 0, TMA>;
  return trace ? anneal_hbm_kernel<true, 4, 0, TMA> : anneal_hbm_kernel<false, 4, 0, TMA>;
}

// Renyi-2 GEMM stages through the TMA engine unless TG_HBM_TMA=0 (the cp.async pipeline).
bool hbm_use_tma() {
  const char* env = std::getenv("TG_HBM_TMA");
  return !(env && env[0] == '0');
}

HbmKernel hbm_kernel(int kind, int cs, bool trace, bool tma) {
  if (kind == 0) return trace ? hbm::anneal_hbm_kernel<true, 1, 1, false> : hbm::anneal_hbm_kernel<false, 1, 1, false>;
  return tma ? hbm_kernel_renyi<true>(cs, trace) : hbm_kernel_renyi<false>(cs, trace);
}

// The TMA view of the workspace (hbm_tier.cuh, rho_partials_tma): 5-D, FP64,
//   dim0 16 rows (contiguous), dim1 16-row block, dim2 column b (stride d_a),
//   dim3 plane 2 * buffer + {X, Y} (stride n), dim4 cluster slot (stride 4n),
// box (16, 2, KC, 2, 1), 128-B swizzle. The encoder comes from the driver at run time (no
// libcuda link dependency).
using EncodeTiled = PFN_cuTensorMapEncodeTiled_v12000;
EncodeTiled tensor_map_encoder() {
  static const EncodeTiled fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiled>(nullptr);
    return reinterpret_cast<EncodeTiled>(f);
  }();
  return fn;
}

cudaError_t hbm_tensor_map(const AnnealParams& p, uint64_t clusters, CUtensorMap* map) {
  const EncodeTiled enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  const uint64_t la = p.spins / 2, da = uint64_t{1} << la, db = uint64_t{1} << (p.spins - la);
  const uint64_t n = uint64_t{1} << p.spins;
  cuuint64_t dims[5] = {16, da / 16, db, 4, clusters};
  cuuint64_t strides[4] = {128, da * 8, n * 8, 4 * n * 8};
  cuuint32_t box[5] = {16, 2, static_cast<cuuint32_t>(hbm::KC), 2, 1};
  cuuint32_t elem[5] = {1, 1, 1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, p.workspace, dims, strides, box, elem,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::fprintf(stderr, "[tg] cuTensorMapEncodeTiled failed (%d): HBM tier stages through cp.async\n",
                 static_cast<int>(r));
    return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

cudaLaunchConfig_t hbm_config(int grid, int cs, cudaStream_t stream, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(hbm::kThreads);
  cfg.dynamicSmemBytes = hbm::kSmemBytes;
  cfg.stream = stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

// CTAs per replica and the number of persistent clusters: at most the clusters that can
// be co-resident (a GPC whose SM count is not a multiple of cs leaves SMs over, so 4-CTA
// clusters do not reach sms / 4: a non-resident cluster would run as a second wave).
cudaError_t hbm_geometry(uint32_t spins, uint64_t rows, int kind, int device, int& cs, uint64_t& clusters) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  auto resident_for = [&](int c, int& resident) -> cudaError_t {
    resident = sms / c;
    if (c == 1) return cudaSuccess;
    HbmKernel kern = hbm_kernel(kind, c, false, false);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, hbm::kSmemBytes);
    if (e != cudaSuccess) return e;
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t cfg = hbm_config(resident * c, c, nullptr, attr);
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    if (e != cudaSuccess) return e;
    if (n > 0 && n < resident) resident = n;
    return cudaSuccess;
  };
  cs = hbm::ctas_per_replica(spins, rows, sms, kind);
  int resident = 0;
  cudaError_t e = resident_for(cs, resident);
  if (e != cudaSuccess) return e;
  // a small batch that does not fit the co-resident 4-CTA clusters drops to 2 CTAs (unless
  // forced by TG_HBM_CTAS_PER_REPLICA)
  if (cs == 4 && rows > static_cast<uint64_t>(resident) && !std::getenv("TG_HBM_CTAS_PER_REPLICA")) {
    cs = 2;
    e = resident_for(cs, resident);
    if (e != cudaSuccess) return e;
  }
  clusters = std::min<uint64_t>(rows, static_cast<uint64_t>(resident));
  if (std::getenv("TG_VERBOSE"))
    std::fprintf(stderr, "[tg] hbm geometry: spins %u rows %llu -> %d CTAs/replica, %llu clusters (resident %d)\n",
                 spins, static_cast<unsigned long long>(rows), cs, static_cast<unsigned long long>(clusters), resident);
  return cudaSuccess;
}

}  // namespace

// Any launch of r <= rows replicas runs min(r, resident clusters) <= min(rows, SMs) clusters
// (hbm_geometry); sizing for that bound keeps a batch tail or a partial launch whose geometry
// has more clusters than the full batch inside the workspace.
uint64_t anneal_hbm_slab_clusters(uint64_t rows, int device) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return std::min<uint64_t>(rows, static_cast<uint64_t>(sms > 0 ? sms : 1));
}

namespace {

// Work-queue schedule (hbm_queue.cuh): Renyi-2 with TMA staging, every row's slab resident at
// once, so the row count is bounded by memory (and the queue only pays where the cluster
// schedule leaves SMs idle, i.e. small and medium batches).
constexpr size_t kQueueSlabBudget = size_t{48} << 30;
constexpr uint64_t kQueueMaxRows = 8192;

// von Neumann above S = 15 exists on the queue schedule only (vn_large.cuh)
bool vn_large(uint32_t spins, int entropy_kind) {
  return entropy_kind == TG_VON_NEUMANN && spins >= static_cast<uint32_t>(kVnQueueMinSpins) &&
         spins <= static_cast<uint32_t>(kVnQueueMaxSpins);
}
size_t queue_row_bytes(uint32_t spins, int entropy_kind) {  // slab (+ rho planes)
  return (size_t{32} << spins) + (vn_large(spins, entropy_kind) ? 8 * hbmq::QLayout::rho_doubles(spins) : 0);
}

bool queue_possible(uint32_t spins, uint64_t rows, int entropy_kind, bool half = false) {
  if ((entropy_kind != TG_RENYI2 && !vn_large(spins, entropy_kind)) || rows == 0 || rows > kQueueMaxRows ||
      !hbm_use_tma())
    return false;
  const char* env = std::getenv("TG_HBM_QUEUE");
  if (env && env[0] == '0' && !half && !vn_large(spins, entropy_kind)) return false;
  return rows * queue_row_bytes(spins, entropy_kind) <= kQueueSlabBudget;
}

// Schedule choice by a tile-time model. Cluster schedule: ceil(rows / clusters) waves of
// ceil(ntt / cs) tiles per CTA; queue: ceil(rows * ntt / sms) tiles per CTA. Each is scaled
// by its measured per-tile overhead at this chain length (gate pass, decision, pipeline
// refills; queue: also the per-item handoffs, which weigh more the fewer tiles a replica
// has): profiles/r02_queue_vs_cluster.txt.
// TG_HBM_QUEUE=1 forces the queue, =0 the cluster schedule; TG_HBM_CTAS_PER_REPLICA or the
// phase-trace probe force the cluster schedule.
bool queue_pick(uint32_t spins, uint64_t rows, int entropy_kind, int device, bool trace, bool half = false) {
  if (trace || !queue_possible(spins, rows, entropy_kind, half)) return false;
  if (half || vn_large(spins, entropy_kind)) return true;  // options that run on the queue only
  const char* env = std::getenv("TG_HBM_QUEUE");
  if (env && env[0] == '1') return true;
  if (std::getenv("TG_HBM_CTAS_PER_REPLICA")) return false;
  int sms = 0, cs = 1;
  uint64_t clusters = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (hbm_geometry(spins, rows, entropy_kind, device, cs, clusters) != cudaSuccess || clusters == 0 || sms <= 0)
    return false;
  const uint64_t nt = (uint64_t{1} << (spins / 2)) / hbm::TB, ntt = nt * nt;
  // measured (r02_queue_vs_cluster.txt): S = 14: 0.36 / 0.23, 16: 0.175 / 0.15, 20: 0.05 / 0.067
  static const double kQueueOver[] = {0.5, 0.36, 0.25, 0.175, 0.12};     // S = 13..17, then 0.05
  static const double kClusterOver[] = {0.3, 0.23, 0.19, 0.15, 0.11};    // S = 13..17, then 0.067
  const double qo = spins <= 17 ? kQueueOver[spins - 13] : 0.05;
  const double co = spins <= 17 ? kClusterOver[spins - 13] : 0.067;
  const double t_cluster = static_cast<double>((rows + clusters - 1) / clusters) *
                           static_cast<double>((ntt + cs - 1) / cs) * (1.0 + co);
  const double t_queue = static_cast<double>((rows * ntt + sms - 1) / sms) * (1.0 + qo);
  return t_queue < t_cluster;
}

}  // namespace

uint64_t anneal_hbm_queue_rows(uint32_t spins, uint64_t rows, int entropy_kind) {
  return queue_possible(spins, rows, entropy_kind, true) ? rows : 0;
}

uint64_t anneal_hbm_queue_max_rows(uint32_t spins, int entropy_kind) {
  return std::min<uint64_t>(kQueueMaxRows, kQueueSlabBudget / queue_row_bytes(spins, entropy_kind));
}

int anneal_hbm_schedule(const AnnealParams& p, int device) {
  return queue_pick(p.spins, p.rows, p.entropy_kind, device, false, p.rho_half != 0) ? 1 : 0;
}

// [max(cluster slabs, queue rows) slabs][queue region (partials, row state, counters)]
size_t anneal_hbm_workspace_bytes(uint32_t spins, uint64_t rows, int device, int entropy_kind) {
  const uint64_t clusters = anneal_hbm_slab_clusters(rows, device);
  const uint64_t qrows = anneal_hbm_queue_rows(spins, rows, entropy_kind);
  const size_t da = size_t{1} << (spins / 2);
  // von Neumann with d_a > 64: rho (2 planes of d_a^2) after each slab (vn_packed.cuh)
  const bool big_vn = vn_large(spins, entropy_kind);  // queue only: rho lives in the queue region
  const size_t rho = entropy_kind == 0 && da > static_cast<size_t>(hbm::TB) && !big_vn ? 2 * da * da : 0;
  const size_t slab = (4 * (size_t{1} << spins) + rho) * sizeof(double);
  return static_cast<size_t>(big_vn ? qrows : std::max(clusters, qrows)) * slab +
         (qrows ? hbmq::QLayout::bytes(spins, qrows, vn_large(spins, entropy_kind)) : 0);
}

uint64_t anneal_hbm_wave_rows(const AnnealParams& p) {  // co-resident clusters = replicas per wave
  int dev = 0, cs = 1;
  uint64_t clusters = 0;
  cudaGetDevice(&dev);
  if (queue_pick(p.spins, p.rows, p.entropy_kind, dev, false, p.rho_half != 0)) return p.rows;  // one wave
  if (hbm_geometry(p.spins, p.rows, p.entropy_kind, dev, cs, clusters) != cudaSuccess) return 0;
  return clusters;
}

namespace {

cudaError_t launch_queue(const AnnealParams& p, cudaStream_t stream, int dev, int* grid_out, bool stats) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  cudaError_t e = hbm_tensor_map(p, p.rows, &tmap);  // slot = row
  if (e != cudaSuccess) return e;
  const hbmq::QLayout L(reinterpret_cast<char*>(p.workspace + p.queue_rows * 4 * (uint64_t{1} << p.spins)), p.spins,
                        p.queue_rows);
  e = cudaMemsetAsync(L.ctr, 0, L.counter_bytes, stream);
  if (e != cudaSuccess) return e;
  const bool vn = p.entropy_kind == TG_VON_NEUMANN;
  auto kern = vn ? (stats ? hbmq::anneal_queue_kernel<true, 1> : hbmq::anneal_queue_kernel<false, 1>)
                 : (stats ? hbmq::anneal_queue_kernel<true, 0> : hbmq::anneal_queue_kernel<false, 0>);
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, hbmq::kQSmemBytes);
  if (e != cudaSuccess) return e;
  const int grid = std::min(sms > 0 ? sms : 1, hbmq::QLayout::kMaxCtas);  // one CTA per SM (deadlock-free at any residency)
  if (grid_out) *grid_out = grid;
  if (std::getenv("TG_VERBOSE"))
    std::fprintf(stderr, "[tg] hbm work queue: spins %u rows %llu on %d CTAs\n", p.spins,
                 static_cast<unsigned long long>(p.rows), grid);
  kern<<<grid, hbmq::kQThreads, hbmq::kQSmemBytes, stream>>>(p, tmap);
  e = cudaGetLastError();
  if (e != cudaSuccess || vn) return e;
  return launch_finish_renyi(p, stream);  // Renyi-2 traces were stored as raw ||rho||_F^2
}

}  // namespace

cudaError_t launch_anneal_hbm(const AnnealParams& p, cudaStream_t stream, int* grid_out,
                              bool trace) {
  if (p.spins < 13 || p.spins > 24) return cudaErrorInvalidValue;
  if (!p.workspace) return cudaErrorInvalidValue;
  if (p.entropy_kind == 0 && p.spins > static_cast<uint32_t>(kVnQueueMaxSpins)) return cudaErrorInvalidValue;
  int dev = 0, cs = 1;
  uint64_t clusters = 0;
  cudaGetDevice(&dev);
  // the phase-trace probe runs the cluster schedule; tg_probe_queue_stats asks for the work
  // queue's per-CTA statistics kernel instead
  const bool queue_stats = trace && p.queue_stats != 0;
  if (p.rows > 0 && p.queue_rows >= p.rows &&
      (queue_stats ? queue_possible(p.spins, p.rows, p.entropy_kind)
                   : queue_pick(p.spins, p.rows, p.entropy_kind, dev, trace, p.rho_half != 0)))
    return launch_queue(p, stream, dev, grid_out, queue_stats);
  if (p.rho_half || vn_large(p.spins, p.entropy_kind)) return cudaErrorInvalidValue;  // queue-only options
  cudaError_t e = hbm_geometry(p.spins, p.rows, p.entropy_kind, dev, cs, clusters);
  if (e != cudaSuccess) return e;
  // never more clusters than the workspace has slabs (the persistent loop strides over rows)
  if (p.slab_clusters > 0 && clusters > p.slab_clusters) clusters = p.slab_clusters;
  const int grid = static_cast<int>(clusters) * cs;
  if (grid_out) *grid_out = grid;
  if (grid == 0) return cudaSuccess;
  // TMA staging needs a tensor map of the workspace (16-B aligned base, driver entry point);
  // when it cannot be encoded the cp.async pipeline runs (same kernel family, same bits)
  bool tma = p.entropy_kind == 1 && hbm_use_tma();
  CUtensorMap tmap;
  std::memset(&tmap, 0, sizeof(tmap));
  if (tma && hbm_tensor_map(p, clusters, &tmap) != cudaSuccess) tma = false;
  HbmKernel kern = hbm_kernel(p.entropy_kind, cs, trace, tma);
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, hbm::kSmemBytes);
  if (e != cudaSuccess) return e;
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = hbm_config(grid, cs, stream, attr);
  AnnealParams q = p;
  const char* lf = std::getenv("TG_HBM_LIGHT_FENCE");
  q.light_fence = !(lf && lf[0] == '0');
  e = cudaLaunchKernelEx(&cfg, kern, q, tmap);
  if (e != cudaSuccess) return e;
  e = cudaGetLastError();
  if (e != cudaSuccess || p.entropy_kind == 0) return e;
  return launch_finish_renyi(p, stream);  // Renyi-2 traces were stored as raw ||rho||_F^2
}

}  // namespace tg
