// tg_internal.h — launch interface between the C-ABI host layer (capi.cpp) and the
// CUDA translation units. Not part of the public boundary (include/taskgemm_b200.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/taskgemm_b200.h"

namespace tg {

struct GateRec;  // tg_device.cuh

// Everything one persistent anneal launch needs. Rows r in [0, rows) are replicas
// p = p_first + r * p_stride (p mod devices / shard binding, bench.cpp:171).
struct AnnealParams {
  uint32_t spins;
  int32_t objective;      // 0 maximize, 1 minimize
  int32_t initial_state;  // 0 product, 1 random
  int32_t inject_fault;
  int32_t entropy_kind;   // 0 von Neumann, 1 Renyi-2 (tg_entropy_kind)
  uint64_t steps, seed, renorm;
  double t0, t_min;
  uint64_t rows, p_first, p_stride;
  double* initial_entropy;
  double* entropies;
  uint8_t* accepted;
  uint8_t* sites;
  int64_t* wall_ns;
  double* final_entropy;
  int32_t* status;
  int64_t* status_step;
  double* workspace;  // HBM tier: per-cluster psi/psi' slabs
  uint64_t slab_clusters;  // HBM tier: slabs the workspace holds (launch_anneal_hbm clamps to it)
  uint64_t queue_rows;     // HBM tier: rows the workspace's work-queue region is sized for (0 = none)
  int64_t* trace;     // phase-trace probe only: clock64 stamps [steps][8] of CTA 0's first row
  const GateRec* gates;        // [rows][steps] proposal stream (gate_stream.cu)
  const double* init_states;   // [rows][2^S] interleaved, unnormalised (random start) or null
  int32_t light_fence;         // HBM tier: no GPU-scope fence between gate pass and GEMM (A/B knob)
  double* status_norm;         // [rows] or null: ||psi|| of a failed norm check
  int64_t* initial_wall_ns;    // [rows] or null: initial state + entropy, %globaltimer ns
  unsigned long long* tie_stats;  // [2] or null: fallback decisions, near ties (atomic counters)
  tg_near_tie* tie_log;        // [tie_capacity] or null
  uint64_t tie_capacity;
  double tie_eps;              // near tie: |u - p| < tie_eps (1e-9; TG_NEAR_TIE_EPS widens it in tests)
  int32_t gate_fault;          // tg_anneal_config inject_fault == 2: the gate of
  uint64_t fault_procedure;    // (fault_procedure, fault_step) is scaled by 1.001
  uint64_t fault_step;
  uint64_t fault_row1;         // 1 + its row in this launch (0 = not in it; zero-init safe), per batch
  int32_t rho_half;            // Renyi-2, HBM tier, work-queue schedule only: upper-triangle tiles
  int32_t queue_stats;         // profiling probe (tg_probe_queue_stats): the work queue's STATS kernel
  int32_t gate_bulk;           // HBM cluster schedule, S >= gate_bulk_min: TMA-staged gate pass (TG_GATE_BULK=0 disables)
  int32_t gate_bulk_min;       // (TG_GATE_BULK_MIN, default 16)
  int32_t gate_chunk;          // groups per staged chunk (TG_GATE_CHUNK; 0 = kGateChunk)
};

// Pre-generated proposal stream of one launch (gate_stream.cu).
struct GateStream {
  GateRec* recs;
  double* init_states;
};
size_t gate_stream_bytes_per_row(uint32_t spins, uint64_t steps, int random_init);
uint64_t rng_chunk_steps();
void rng_jump_words(uint64_t seed, uint64_t p, int init_spins, uint64_t chunks, uint64_t extra, uint64_t n,
                    uint64_t* out);
cudaError_t probe_rng_chunking(uint32_t spins, uint64_t rows, uint64_t steps, int random_init,
                               uint64_t reject_below, uint64_t* mismatches);
cudaError_t launch_gate_stream(const AnnealParams& p, void* ws, size_t ws_bytes, GateStream* gs,
                               cudaStream_t stream);

// Status codes written per row by the kernels.
enum : int32_t { kRowOk = 0, kRowNotNormalized = 2 };

constexpr int kSmemMaxSpins = 12;
constexpr uint64_t kMaxSteps = uint64_t{1} << 22;  // gate_stream.cu jump tables (kJumpBits)
constexpr int kVnMaxSpins = 15;
constexpr int kVnQueueMinSpins = 16, kVnQueueMaxSpins = 21;  // von Neumann on the work queue (vn_large.cuh: d_a 256..1024)  // device von Neumann: d_a <= 64 (vn.cuh: SMEM tier, HBM tier S=13), d_a = 128 (vn_packed.cuh: S=14,15)

// anneal_smem.cu (S <= 12)
// replicas processed per wave by one launch (resident CTAs / clusters), 0 if unknown
uint64_t anneal_smem_wave_rows(const AnnealParams& p);
uint64_t anneal_hbm_wave_rows(const AnnealParams& p);
cudaError_t launch_anneal_smem(const AnnealParams& p, cudaStream_t stream, int* grid_out,
                               bool trace = false);
// anneal_hbm.cu (S >= 13)
cudaError_t launch_anneal_hbm(const AnnealParams& p, cudaStream_t stream, int* grid_out,
                              bool trace = false);
cudaError_t launch_finish_renyi(const AnnealParams& p, cudaStream_t stream);
size_t anneal_hbm_workspace_bytes(uint32_t spins, uint64_t rows, int device, int entropy_kind);
// which HBM-tier schedule a launch of p uses: 0 cluster, 1 work queue (hbm_queue.cuh)
int anneal_hbm_schedule(const AnnealParams& p, int device);
uint64_t anneal_hbm_slab_clusters(uint64_t rows, int device);  // slabs for launches of <= rows replicas
uint64_t anneal_hbm_queue_rows(uint32_t spins, uint64_t rows, int entropy_kind);  // queue region capacity
uint64_t anneal_hbm_queue_max_rows(uint32_t spins, int entropy_kind);  // largest launch the queue schedule takes

// probes.cu
cudaError_t probe_rng(uint64_t seed, uint64_t p, uint64_t n, uint64_t* d_out, cudaStream_t s);
cudaError_t probe_gates(uint32_t spins, uint64_t seed, uint64_t p, uint64_t steps, int initial,
                        uint8_t* d_sites, double* d_u, double* d_uacc, cudaStream_t s);
cudaError_t probe_apply_gate(uint32_t spins, const double* d_psi, int site, const double* d_u,
                             double* d_out, cudaStream_t s);
cudaError_t probe_entropy(uint32_t spins, uint64_t count, const double* d_psi, double* d_e,
                          double* d_norm, bool fault, cudaStream_t s, bool von_neumann = false);
cudaError_t fp64_dmma_peak(double* tflops, double* clock_ghz);

// zgemm.cu
cudaError_t launch_zgemm_strided(int batch, int m, int n, int k, double ar, double ai,
                                 const double* A, int64_t sA, const double* B, int64_t sB,
                                 double br, double bi, const double* C, int64_t sC, double* out,
                                 int64_t sO, int inject_fault, cudaStream_t stream);

}  // namespace tg
