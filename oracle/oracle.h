/*
 * oracle.h — CPU restatement of the reference annealing hot path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product path (paper_2203_09353_b200/,
 * include/) may link or call this; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, as the checker.
 *
 * Restates, function by function, /root/reference/proj/src/{rng,linalg,spinmc}.cpp
 * with the reference's unfused arithmetic (built with -ffp-contract=off), so that on
 * the same glibc it is bitwise identical to the reference. Pinned against the
 * reference itself (oracle/_ref, built from the reference sources by oracle/Makefile)
 * and against tests/golden/ fixtures generated from it (tools/make_golden.py).
 */
#ifndef TG_ORACLE_H
#define TG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint64_t s[4];
} tgo_stream;

/* rng.cpp:23-33 (derive_stream({seed, p})) */
void tgo_stream_init(tgo_stream* st, uint64_t global_seed, uint64_t procedure_index);
/* rng.cpp:35-45 */
uint64_t tgo_next_u64(tgo_stream* st);
/* rng.cpp:47-49 */
double tgo_uniform01(tgo_stream* st);
/* rng.cpp:51-59; n >= 1 */
uint64_t tgo_uniform_index(tgo_stream* st, uint64_t n);
/* rng.cpp:61-67 */
void tgo_normal_pair(tgo_stream* st, double* a, double* b);

/* spinmc.cpp:65-89; u is 4x4 column-major interleaved complex (32 doubles) */
void tgo_haar(tgo_stream* st, double* u);

/* spinmc.cpp:91-136; psi/out interleaved complex of length 2^spins. returns 0 or -1 (bad args) */
int tgo_apply_gate(int spins, const double* psi, int site, const double* u, double* out);

/* spinmc.cpp:50-54 */
double tgo_state_norm(int spins, const double* psi);

/* linalg.cpp:79-113: out = alpha*A*B + beta*C, column-major interleaved complex. */
void tgo_gemm(int m, int n, int k, const double* alpha, const double* a, const double* b,
              const double* beta, const double* c, double* out);

/* linalg.cpp:131-138 */
double tgo_frobenius(int rows, int cols, const double* a);

/* spinmc.cpp:150-176 (Renyi-2 branch; kind 1) and the von Neumann branch (kind 0,
 * linalg.cpp:161-232). Returns 0 on success, -1 if ||psi|| deviates from 1 by > 1e-9
 * (the "not normalized" invalid_argument of spinmc.cpp:153-156). */
int tgo_entropy(int spins, const double* psi, int kind, double* entropy_out);

/* spinmc.cpp:178-184 */
double tgo_temperature(double t0, double t_min, uint64_t step, uint64_t total);
/* spinmc.cpp:186-191 */
double tgo_acceptance(double delta, double t);

/* linalg.cpp:161-232; h is n x n column-major interleaved; eig (ascending) of length n.
 * returns 0, or -1 if not Hermitian within 1e-10 relative. */
int tgo_hermitian_eigenvalues(int n, const double* h, double* eig);

typedef struct {
  int32_t spins;
  int32_t entropy_kind;  /* 0 von-neumann, 1 renyi-2 (spinmc.hpp:32) */
  int32_t objective;     /* 0 maximize, 1 minimize (spinmc.hpp:33) */
  int32_t initial_state; /* 0 product, 1 random (spinmc.hpp:34) */
  uint64_t steps;
  uint64_t seed;
  double t0, t_min;
  uint64_t renormalize_interval; /* spinmc.hpp:120, default 1000 */
} tgo_config;

/* spinmc.cpp:215-251 for replica p on stream derive_stream({seed, p}).
 * entropies/accepted/sites have length cfg->steps (sites/accepted/u_out/p_out may be NULL).
 * u_out/p_out record the acceptance draw and probability per step (near-tie diagnostics).
 * Returns 0, -1 config error, -2 "not normalized" (KernelError analogue). */
int tgo_mc_procedure(const tgo_config* cfg, uint64_t p, double* initial_entropy,
                     double* entropies, uint8_t* accepted, uint8_t* sites, double* u_out,
                     double* p_out);

/* Runs replicas [p0, p0+count) over `threads` host threads (pooled driver).
 * Row r of the outputs is replica p0+r. Returns 0 or the first error code. */
int tgo_run_pool(const tgo_config* cfg, uint64_t p0, uint64_t count, int threads,
                 double* initial_entropy, double* entropies, uint8_t* accepted, uint8_t* sites);

/* spinmc.cpp:253-269 + bench.cpp:401-407: mean of finals in procedure order
 * (steps == 0: mean of initial entropies). */
double tgo_average_entropy(uint64_t procedures, uint64_t steps, const double* initial_entropy,
                           const double* entropies);

#ifdef __cplusplus
}
#endif

#endif
