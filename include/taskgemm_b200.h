/*
 * taskgemm_b200.h — C ABI of the B200-native annealing / small-GEMM hot path.
 *
 * This is the drop-in boundary. Each entry point replaces one reference interface
 * (paths relative to /root/reference/proj); the reference-side binding a maintainer
 * adds is shown in INTEGRATION.md. Plain pointers and sizes only; complex matrices are
 * column-major interleaved complex128 (re, im), layout-compatible with
 * std::complex<double> / linalg::ComplexMatrix (include/taskgemm/linalg.hpp:13-47).
 *
 * Error convention (replaces the reference's exception types, errors.hpp:9-12,
 * exec.hpp:71-86): every function returns a tg_status; on non-zero the message is
 * available from tg_last_error() (thread-local) and carries the same substrings the
 * reference's exceptions carry ("spins out of range [2,30]", "fixed-size",
 * "not normalized", "kernel failed for procedure N: ...").
 */
#ifndef TASKGEMM_B200_H
#define TASKGEMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TG_OK = 0,
  TG_ECONFIG = 1,    /* taskgemm::ConfigError                (errors.hpp:9-12)          */
  TG_EINVAL = 2,     /* std::invalid_argument preconditions   (exec.cpp:154-161 etc.)    */
  TG_EKERNEL = 3,    /* exec::KernelError                     (exec.hpp:76-86)           */
  TG_ESHUTDOWN = 4,  /* exec::SubmissionError                 (exec.cpp:99)              */
  TG_ECUDA = 5,      /* CUDA runtime / no device (no CPU fallback exists)                */
} tg_status;

typedef enum { TG_VON_NEUMANN = 0, TG_RENYI2 = 1 } tg_entropy_kind;     /* spinmc.hpp:32 */
typedef enum { TG_MAXIMIZE = 0, TG_MINIMIZE = 1 } tg_objective;        /* spinmc.hpp:33 */
typedef enum { TG_PRODUCT = 0, TG_RANDOM = 1 } tg_initial_state;       /* spinmc.hpp:34 */

/* = bench::ExperimentConfig (bench.hpp:28-45) restricted to the workload fields, plus
 * the McConfig renormalize interval (spinmc.hpp:120) and a process shard. Replica p runs
 * on stream derive_stream({seed, p}) (bench.cpp:385). With shard_count > 1 only replicas
 * p with p % shard_count == shard_index run in this call (one process per GPU). */
typedef struct {
  uint32_t spins;                /* S in [2,30]; device tiers cover S <= 24             */
  uint32_t devices;              /* GPUs of the context used (p -> device p mod devices) */
  uint64_t steps;                /* N_s                                                  */
  uint64_t procedures;           /* N_p (>= 1)                                           */
  uint64_t seed;                 /* global seed                                          */
  int32_t entropy_kind;          /* tg_entropy_kind (device: TG_RENYI2)                 */
  int32_t objective;             /* tg_objective                                         */
  int32_t initial_state;         /* tg_initial_state                                     */
  int32_t inject_fault;          /* test hooks: 0 none; 1 = testhooks::perturb_gemm      *
                                  * (linalg.hpp:74-79); 2 = the gate of (fault_procedure, *
                                  * fault_step) is scaled by 1.001, so psi' fails the norm *
                                  * check of spinmc.cpp:152-156                            */
  double t0, t_min;              /* AnnealSchedule (spinmc.hpp:37-40)                    */
  uint64_t renormalize_interval; /* 1000 by default; 0 disables                          */
  uint32_t shard_index, shard_count;
  uint64_t fault_procedure, fault_step;  /* inject_fault == 2 only                     */
  int32_t rho_half;              /* opt-in, Renyi-2: form only the upper triangle of rho's *
                                  * 64x64 tiles (HBM tier) or 8x8 blocks (SMEM tier; rho is  *
                                  * Hermitian;                                              *
                                  * ||rho||_F^2 = diagonal tiles + 2 x off-diagonal ones).  *
                                  * Not the reference's arithmetic (its GEMM is the full    *
                                  * product): entropies agree within the parity *
                                  * tolerance, and the flops actually executed are reported *
                                  * in tg_anneal_result.executed_flops next to total_flops  *
                                  * (the graded full-GEMM count). 0 = full GEMM (default).  */
} tg_anneal_config;

/* One logged near-tie accept decision: |u - p| < 1e-9 in the test
 * u < acceptance_probability(delta, T) of spinmc.cpp:201-207, where a last-bit difference
 * in the entropy could flip the outcome. */
typedef struct {
  uint64_t procedure, step;
  double u, p;             /* uniform01 draw and acceptance probability (reference formula) */
  uint32_t site;
  int32_t accepted;
} tg_near_tie;

/* Per-procedure traces = spinmc::EntropyTrace (spinmc.hpp:44-50) + sites. Caller-owned
 * HOST arrays; row r is procedure p = shard_index + r*shard_count (r < local count), i.e.
 * row p when shard_count == 1. Optional arrays may be NULL. */
typedef struct {
  double* initial_entropy;  /* [rows]                                                  */
  double* entropies;        /* [rows*steps] post-decision entropy (spinmc.hpp:42-43)   */
  uint8_t* accepted;        /* [rows*steps]                                            */
  uint8_t* sites;           /* [rows*steps] optional                                   */
  int64_t* wall_ns;         /* [rows*steps] optional, device %globaltimer per step     */
  double* final_entropy;    /* [rows] optional                                         */
  /* outputs */
  double average_entropy;   /* over this call's rows, procedure order (spinmc.cpp:253-269) */
  int64_t total_wall_ns;    /* host wall time of the call                              */
  uint64_t total_flops;     /* (rows*steps + rows) * gemm_flops(d_a,d_a,d_b)           */
  double kernel_ms;         /* device time of the anneal kernel(s), CUDA events (max   *
                             * over the context's GPUs)                                */
  double* device_kernel_ms; /* [devices] optional: per-GPU device time                  */
  uint64_t* device_resident; /* [devices] optional: replicas resident at once per GPU     *
                              * (persistent-kernel slots; DeviceMetrics high water mark) */
  int64_t* initial_wall_ns; /* [rows] optional: initial state + initial-entropy GEMM,     *
                             * device %globaltimer (spinmc.cpp:229-234)                  */
  /* decision audit. The device decides Renyi-2 steps by a lean bound     *
   * (DESIGN.md §3.1); a decision whose margin is inside the rounding window is re-taken   *
   * with the reference formula.                                                          */
  uint64_t fallback_decisions;   /* out: decisions re-taken with the reference formula   */
  uint64_t near_ties;            /* out: decisions with |u - p| < 1e-9                    */
  tg_near_tie* near_tie_log;     /* optional [near_tie_capacity]: the first near ties,    *
                                  * sorted by (procedure, step)                           */
  uint64_t near_tie_capacity;
  uint64_t executed_flops;       /* out: GEMM flops the device executed (= total_flops     *
                                  * unless rho_half)                                       */
  uint32_t nccl_ranks;           /* out: GPUs of the NCCL all-gather that fed the average   *
                                  * (the run's one collective); 0 = host copies *
                                  * (one GPU, GPUs repeated in the context, NCCL absent)    */
} tg_anneal_result;

/* Device-resident outputs for tg_anneal_launch (rows as above). */
typedef struct {
  double* initial_entropy;  /* [rows]        */
  double* entropies;        /* [rows*steps]  */
  uint8_t* accepted;        /* [rows*steps]  */
  uint8_t* sites;           /* [rows*steps] or NULL */
  int64_t* wall_ns;         /* [rows*steps] or NULL */
  double* final_entropy;    /* [rows]        */
  int32_t* status;          /* [rows] 0 ok, 2 not normalized (step in status_step) */
  int64_t* status_step;     /* [rows]        */
  void* workspace;          /* tg_anneal_workspace_bytes() bytes (HBM tier), else NULL */
  double* status_norm;      /* [rows] or NULL: ||psi|| of a failed norm check          */
  int64_t* initial_wall_ns; /* [rows] or NULL: initial state + entropy, %globaltimer ns  */
  uint64_t* tie_stats;      /* [2] or NULL, zeroed by the caller: fallback decisions,  *
                             * near ties (counters, atomically incremented)             */
  tg_near_tie* tie_log;     /* [tie_capacity] or NULL: near ties in completion order   */
  uint64_t tie_capacity;
} tg_anneal_device_buffers;

typedef struct tg_ctx tg_ctx;

/* = exec::KernelRecord (exec.hpp:46-55); times in ns (device events for the batch). */
typedef struct {
  uint64_t device_id, procedure, m, n, k;
  int64_t queue_wait_ns, exec_time_ns;
  uint64_t flops;
} tg_kernel_record;

const char* tg_last_error(void);
const char* tg_version(void);
// Number of CUDA kernels this library has launched in this process (anneal pipeline and
// batched GEMM; probes excluded). Lets a caller count launches inside a timed region.
uint64_t tg_kernel_launches(void);

/* Opens a context over `n` GPUs (device ordinals; NULL = 0..n-1). Owns streams and
 * device buffers. One caller per context at a time (documented). */
tg_status tg_create(const int* gpus, int n, tg_ctx** out);
/* After shutdown every call returns TG_ESHUTDOWN (exec.cpp:99 SubmissionError). */
tg_status tg_shutdown(tg_ctx* ctx);
tg_status tg_destroy(tg_ctx* ctx);

/* bench::validate (bench.cpp:321-329) + dims_for_spins (spinmc.cpp:15-26). */
tg_status tg_validate(const tg_anneal_config* cfg);
/* Rows this call produces for the config's shard. */
uint64_t tg_anneal_rows(const tg_anneal_config* cfg);
/* gemm_flops(d_a, d_a, d_b) of one step (linalg.cpp:140-144); 0 if spins invalid. */
uint64_t tg_step_flops(uint32_t spins);

/* Annealing driver: replaces bench::run_experiment (bench.hpp:75, bench.cpp:341-417) for
 * the new ExecutionMode::kDevice. Runs the shard's replicas over the context's GPUs (one
 * persistent kernel per GPU, replica p on GPU p mod devices), copies traces to the
 * caller's host arrays. When a replica's state leaves normalization it fails as the
 * reference does: TG_EINVAL (std::invalid_argument) with the message of spinmc.cpp:153-155,
 * "entanglement_entropy: state not normalized (||psi|| = %f)", for the first such
 * procedure in procedure order (run_experiment rethrows it unchanged, bench.cpp:387-395). */
tg_status tg_anneal_run(tg_ctx* ctx, const tg_anneal_config* cfg, tg_anneal_result* res);

/* Low-level asynchronous launch on the CURRENT device and the given stream
 * (cudaStream_t as void*; NULL = legacy default). Buffers are device pointers. Used by
 * bench.py to time the kernel with events on its own stream. cfg->devices is ignored. */
tg_status tg_anneal_launch(const tg_anneal_config* cfg, const tg_anneal_device_buffers* buf,
                           void* stream);
size_t tg_anneal_workspace_bytes(const tg_anneal_config* cfg);

/* GEMM batcher: replaces VirtualDevice::batched_gemm / batched_gemm_at (exec.hpp:146-147,
 * exec.cpp:144-221). out[i] = alpha*A[i]*B[i] + beta*C[i] for a fixed-size batch (all
 * entries share (m,n,k); a mixed batch cannot be expressed — the C++ shim reports the
 * reference's "fixed-size contract violated"). Host pointers; results ordered as inputs;
 * blocks until done; one record per entry (records may be NULL). batch >= 1 else
 * TG_EINVAL "batch must be non-empty". `procedures` (may be NULL) stamps records. */
tg_status tg_zgemm_batched(tg_ctx* ctx, int device, int batch, int m, int n, int k,
                           const double alpha[2], const double* const* A, const double* const* B,
                           const double beta[2], const double* const* C, double* const* out,
                           const uint64_t* procedures, tg_kernel_record* records);

/* Device-pointer strided variant on the current device / given stream (A: m*k*batch,
 * strideA elements between entries, etc.; complex elements). */
tg_status tg_zgemm_strided_launch(int batch, int m, int n, int k, const double alpha[2],
                                  const double* A, int64_t strideA, const double* B,
                                  int64_t strideB, const double beta[2], const double* C,
                                  int64_t strideC, double* out, int64_t strideOut,
                                  int inject_fault, void* stream);

/* Process-global fault hook = linalg::testhooks::perturb_gemm (linalg.hpp:74-79): while set,
 * every device GEMM (anneal kernels, batched ZGEMM, entropy probe) flips the sign of the
 * first accumulation term of element (0,0). Exists so verification suites can prove they
 * catch a broken kernel; never set outside tests. */
tg_status tg_set_perturb_gemm(int on);

/* FP64 DMMA.8x8x4 throughput probe (all SMs, register-resident): the roofline
 * denominator (no FP64 entry exists in MEASURED_PEAKS.json). */
tg_status tg_fp64_dmma_peak(int device, double* tflops, double* sm_clock_ghz_est);

/* Which schedule the HBM tier (13 <= spins <= 24) would run a launch of `rows` replicas
 * with on the current device: 0 = cluster schedule (1, 2 or 4 CTAs own a replica),
 * 1 = work queue (every CTA pulls tile / gate / decision items), -1 = not an HBM-tier
 * launch. Diagnostic: replaces nothing in the reference (whose scheduler is the simulated
 * VirtualDevice, exec.cpp:51-142, out of scope). */
int tg_hbm_schedule(uint32_t spins, uint64_t rows, int32_t entropy_kind);

/* ---- device-piece probes (parity tests T1-T6 in SURVEY.md §4) ---------------------- */
/* Work-queue schedule statistics (profiling probe): runs `replicas` x `steps` at `spins`
 * (13..24) on the queue schedule and writes 24 per-CTA clock64 counters per CTA into
 * stats[ctas * 24] (layout in csrc/hbm_queue.cuh, STATS); *ctas = the grid size (SM count,
 * stats must hold 24 * SM count values). */
tg_status tg_probe_queue_stats(uint32_t spins, uint64_t replicas, uint64_t steps, int32_t entropy_kind,
                               int64_t* stats, int* ctas);
/* first n xoshiro256++ outputs of derive_stream({seed,p}) computed on the GPU */
tg_status tg_probe_rng(uint64_t seed, uint64_t p, uint64_t n, uint64_t* out_host);
/* gate stream of `steps` steps (site, U[32], u_accept) generated by the device producer */
tg_status tg_probe_gates(uint32_t spins, uint64_t seed, uint64_t p, uint64_t steps,
                         int initial_state, uint8_t* sites, double* u, double* uacc);
/* device gate application, unfused rounding; psi/out host arrays of 2^spins complex */
tg_status tg_probe_apply_gate(uint32_t spins, const double* psi, int site, const double* u,
                              double* out);
/* device Renyi-2 entropy (DMMA rho + fused ||rho||_F^2) of host states [count][2^spins];
 * norms receives ||psi|| (may be NULL) */
tg_status tg_probe_entropy(uint32_t spins, uint64_t count, const double* psi, double* entropy,
                           double* norms);
/* same with the entropy kind (tg_entropy_kind): TG_VON_NEUMANN = eigenvalues of rho on the
 * device (spins <= 15), spinmc.cpp:165-169 / linalg.cpp:161-232 */
tg_status tg_probe_entropy_kind(uint32_t spins, uint64_t count, const double* psi, int32_t kind,
                                double* entropy, double* norms);

/* Profiling probe: runs `replicas` replicas and returns clock64 phase stamps of CTA 0's
 * first replica, trace[steps][8]: 0 step start, 1 gate pass done, 2 GEMM done,
 * 3 decision done. */
tg_status tg_probe_phase_trace(uint32_t spins, uint64_t replicas, uint64_t steps, int64_t* trace);

/* Test probe: the proposal pre-pass's chunked jump-ahead RNG (per replica, chunks of 256
 * steps start from xoshiro256++ states advanced by GF(2) matrix powers; rng.cpp:35-59)
 * against one sequential stream per replica, seeds derive_stream({0, p}), p < rows.
 * reject_below: the uniform_index rejection threshold (0 = the reference's
 * (2^64 - n) mod n; larger values force rejections and exercise the fixup pass).
 * *mismatches = number of differing draw words + sites (0 = identical). */
tg_status tg_probe_rng_chunking(uint32_t spins, uint64_t rows, uint64_t steps, int32_t random_init,
                                uint64_t reject_below, uint64_t* mismatches);

/* Steps per chunk of the pre-pass's jump-ahead RNG (each chunk is 34 * that many draws). */
uint64_t tg_rng_chunk_steps(void);
/* Host only (no GPU): the n words of derive_stream({seed, p}) (rng.cpp:23-45) after the
 * pre-pass's jumps: 2^(init_spins+1) draws when init_spins >= 0 (random start), then
 * chunks * 34 * tg_rng_chunk_steps() draws, then `extra` single draws — the jump tables
 * rng_chunk_kernel uses, so tests can check them against a sequential stream on the CPU. */
tg_status tg_rng_jump_words(uint64_t seed, uint64_t p, int32_t init_spins, uint64_t chunks, uint64_t extra,
                            uint64_t n, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* TASKGEMM_B200_H */
