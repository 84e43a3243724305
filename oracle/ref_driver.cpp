// ref_driver.cpp — C entry points over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY. oracle/Makefile compiles this file together with
// /root/reference/proj/src/{linalg,rng,exec,spinmc,bench}.cpp (where they lie, never
// copied) into oracle/_ref/libtgref.so. Tests use it to pin oracle/oracle.c and to
// generate tests/golden/; bench.py --impl reference and the cpu_baseline leg time it.
// Every function calls the reference's own API; nothing here re-implements the path.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "taskgemm/bench.hpp"
#include "taskgemm/errors.hpp"
#include "taskgemm/exec.hpp"
#include "taskgemm/linalg.hpp"
#include "taskgemm/rng.hpp"
#include "taskgemm/spinmc.hpp"

using namespace taskgemm;
using linalg::Complex;
using linalg::ComplexMatrix;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

spinmc::SpinChainState make_state(int spins, const double* psi) {
  spinmc::SpinChainState s;
  s.spins = static_cast<std::size_t>(spins);
  s.amplitudes.resize(std::size_t{1} << spins);
  std::memcpy(s.amplitudes.data(), psi, sizeof(Complex) * s.amplitudes.size());
  return s;
}

ComplexMatrix make_matrix(int rows, int cols, const double* data) {
  std::vector<Complex> v(static_cast<std::size_t>(rows) * cols);
  std::memcpy(v.data(), data, sizeof(Complex) * v.size());
  return ComplexMatrix(rows, cols, std::move(v));
}
}  // namespace

extern "C" {

struct tgr_config {  // field-for-field with oracle.h tgo_config
  int32_t spins, entropy_kind, objective, initial_state;
  uint64_t steps, seed;
  double t0, t_min;
  uint64_t renormalize_interval;
};

const char* tgr_last_error() { return g_err.c_str(); }

void tgr_first_u64(uint64_t seed, uint64_t p, uint64_t n, uint64_t* out) {
  auto st = rng::derive_stream({seed, static_cast<std::size_t>(p)});
  for (uint64_t i = 0; i < n; ++i) out[i] = st.next_u64();
}

void tgr_normal_pairs(uint64_t seed, uint64_t p, uint64_t n, double* out) {
  auto st = rng::derive_stream({seed, static_cast<std::size_t>(p)});
  for (uint64_t i = 0; i < n; ++i) {
    auto [a, b] = st.standard_normal_pair();
    out[2 * i] = a;
    out[2 * i + 1] = b;
  }
}

// Successive Haar unitaries from one stream, column-major interleaved, 32 doubles each.
void tgr_haar(uint64_t seed, uint64_t p, uint64_t count, double* out) {
  auto st = rng::derive_stream({seed, static_cast<std::size_t>(p)});
  for (uint64_t c = 0; c < count; ++c) {
    ComplexMatrix u = spinmc::haar_two_site_unitary(st);
    std::memcpy(out + 32 * c, u.data(), sizeof(Complex) * 16);
  }
}

int tgr_apply_gate(int spins, const double* psi, int site, const double* u, double* out) {
  try {
    auto s = make_state(spins, psi);
    auto r = spinmc::apply_two_site_gate(s, static_cast<std::size_t>(site), make_matrix(4, 4, u));
    std::memcpy(out, r.amplitudes.data(), sizeof(Complex) * r.amplitudes.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

int tgr_entropy(int spins, const double* psi, int kind, double* out) {
  try {
    exec::DirectExecutor ex;
    *out = spinmc::entanglement_entropy(
        make_state(spins, psi), kind == 0 ? spinmc::EntropyKind::kVonNeumann : spinmc::EntropyKind::kRenyi2,
        ex);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

int tgr_gemm(int m, int n, int k, const double* alpha, const double* a, const double* b,
             const double* beta, const double* c, double* out) {
  try {
    ComplexMatrix r = linalg::gemm(Complex{alpha[0], alpha[1]}, make_matrix(m, k, a), make_matrix(k, n, b),
                                   Complex{beta[0], beta[1]}, make_matrix(m, n, c));
    std::memcpy(out, r.data(), sizeof(Complex) * r.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

int tgr_hermitian_eigenvalues(int n, const double* h, double* eig) {
  try {
    auto v = linalg::hermitian_eigenvalues(make_matrix(n, n, h));
    std::memcpy(eig, v.data(), sizeof(double) * v.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, -1);
  }
}

double tgr_temperature(double t0, double t_min, uint64_t step, uint64_t total) {
  return spinmc::temperature({t0, t_min}, step, total);
}

double tgr_acceptance(double delta, double t) { return spinmc::acceptance_probability(delta, t); }

static spinmc::McConfig to_mc(const tgr_config* c) {
  spinmc::McConfig mc;
  mc.spins = static_cast<std::size_t>(c->spins);
  mc.steps = c->steps;
  mc.entropy_kind = c->entropy_kind == 0 ? spinmc::EntropyKind::kVonNeumann : spinmc::EntropyKind::kRenyi2;
  mc.objective = c->objective == 0 ? spinmc::Objective::kMaximize : spinmc::Objective::kMinimize;
  mc.schedule = {c->t0, c->t_min};
  mc.initial_state = c->initial_state == 0 ? spinmc::InitialState::kProduct : spinmc::InitialState::kRandom;
  mc.renormalize_interval = c->renormalize_interval;
  return mc;
}

// Sites are not part of EntropyTrace; they are regenerated from an identical stream
// by replaying the draw order of mc_procedure/metropolis_step (spinmc.cpp:229-232,198-207).
static void replay_sites(const tgr_config* c, uint64_t p, uint8_t* sites) {
  auto st = rng::derive_stream({c->seed, static_cast<std::size_t>(p)});
  if (c->initial_state != 0) spinmc::random_state(static_cast<std::size_t>(c->spins), st);
  for (uint64_t s = 0; s < c->steps; ++s) {
    sites[s] = static_cast<uint8_t>(st.uniform_index(static_cast<std::size_t>(c->spins - 1)));
    spinmc::haar_two_site_unitary(st);
    st.uniform01();
  }
}

// Pooled CPU driver: `threads` host threads pull replicas from a
// counter; replica p runs spinmc::mc_procedure on derive_stream({seed,p}) with a
// DirectExecutor. Returns wall ns in *wall_ns; sites optional.
int tgr_run_pool(const tgr_config* c, uint64_t p0, uint64_t count, int threads, double* init,
                 double* ent, uint8_t* acc, uint8_t* sites, int64_t* wall_ns) {
  const spinmc::McConfig mc = to_mc(c);
  std::atomic<uint64_t> next{0};
  std::atomic<int> rc{0};
  std::string first_err;
  std::mutex mu;
  auto t0 = std::chrono::steady_clock::now();
  auto worker = [&] {
    for (;;) {
      const uint64_t r = next.fetch_add(1);
      if (r >= count) return;
      try {
        exec::DirectExecutor ex;
        auto st = rng::derive_stream({c->seed, static_cast<std::size_t>(p0 + r)});
        spinmc::EntropyTrace t = spinmc::mc_procedure(mc, p0 + r, st, ex);
        if (init) init[r] = t.initial_entropy;
        for (uint64_t s = 0; s < c->steps; ++s) {
          if (ent) ent[r * c->steps + s] = t.entropies[s];
          if (acc) acc[r * c->steps + s] = t.accepted_flags[s] ? 1 : 0;
        }
      } catch (const ConfigError& e) {
        std::lock_guard lk(mu);
        if (rc.load() == 0) { first_err = e.what(); rc = -1; }
      } catch (const std::exception& e) {
        std::lock_guard lk(mu);
        if (rc.load() == 0) { first_err = e.what(); rc = -2; }
      }
    }
  };
  std::vector<std::thread> pool;
  for (int i = 0; i < std::max(1, threads); ++i) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  if (wall_ns)
    *wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  if (rc.load() != 0) {
    g_err = first_err;
    return rc.load();
  }
  if (sites)
    for (uint64_t r = 0; r < count; ++r) replay_sites(c, p0 + r, sites + r * c->steps);
  return 0;
}

// Timed CPU sample for bench.py's reference arm / cpu_baseline: the pooled
// driver above, recording per replica the wall time of the whole mc_procedure (total_ns)
// and the sum of its per-step wall times (steps_ns: EntropyTrace::wall_times, which the
// reference fills from DirectExecutor::now(), a steady clock; spinmc.cpp:238-245). The
// difference is the initial state + initial-entropy GEMM (spinmc.cpp:229-234), so a short
// sample extrapolates linearly in steps (bench::extrapolate_runtime, bench.cpp:429-438).
int tgr_time_sample(const tgr_config* c, uint64_t p0, uint64_t count, int threads, int64_t* total_ns,
                    int64_t* steps_ns, int64_t* wall_ns) {
  const spinmc::McConfig mc = to_mc(c);
  std::atomic<uint64_t> next{0};
  std::atomic<int> rc{0};
  std::string first_err;
  std::mutex mu;
  auto t0 = std::chrono::steady_clock::now();
  auto worker = [&] {
    for (;;) {
      const uint64_t r = next.fetch_add(1);
      if (r >= count) return;
      try {
        exec::DirectExecutor ex;
        auto st = rng::derive_stream({c->seed, static_cast<std::size_t>(p0 + r)});
        const auto a = std::chrono::steady_clock::now();
        spinmc::EntropyTrace t = spinmc::mc_procedure(mc, p0 + r, st, ex);
        const auto b = std::chrono::steady_clock::now();
        int64_t s = 0;
        for (const auto& w : t.wall_times) s += w.count();
        total_ns[r] = std::chrono::duration_cast<std::chrono::nanoseconds>(b - a).count();
        steps_ns[r] = s;
      } catch (const std::exception& e) {
        std::lock_guard lk(mu);
        if (rc.load() == 0) { first_err = e.what(); rc = -2; }
      }
    }
  };
  std::vector<std::thread> pool;
  for (int i = 0; i < std::max(1, threads); ++i) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  if (wall_ns)
    *wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  if (rc.load() != 0) {
    g_err = first_err;
    return rc.load();
  }
  return 0;
}

// The reference's own driver (bench::run_experiment, bench.cpp:341-417) in a given mode.
// virtual_wall_ns receives report.total_wall (a VIRTUAL makespan).
int tgr_run_experiment(const tgr_config* c, uint64_t procedures, uint64_t devices, const char* mode,
                       double* init, double* ent, uint8_t* acc, double* average, int64_t* virtual_wall_ns) {
  try {
    bench::ExperimentConfig cfg;
    cfg.spins = static_cast<std::size_t>(c->spins);
    cfg.steps = c->steps;
    cfg.procedures = procedures;
    cfg.devices = devices;
    auto m = bench::mode_from_string(mode);
    if (!m) throw ConfigError(std::string("unknown mode ") + mode);
    cfg.mode = *m;
    cfg.entropy_kind = c->entropy_kind == 0 ? spinmc::EntropyKind::kVonNeumann : spinmc::EntropyKind::kRenyi2;
    cfg.objective = c->objective == 0 ? spinmc::Objective::kMaximize : spinmc::Objective::kMinimize;
    cfg.schedule = {c->t0, c->t_min};
    cfg.initial_state = c->initial_state == 0 ? spinmc::InitialState::kProduct : spinmc::InitialState::kRandom;
    cfg.seed = c->seed;
    bench::RunReport rep = bench::run_experiment(cfg);
    for (uint64_t p = 0; p < procedures; ++p) {
      const auto& t = rep.traces[p];
      if (init) init[p] = t.initial_entropy;
      for (uint64_t s = 0; s < c->steps; ++s) {
        if (ent) ent[p * c->steps + s] = t.entropies[s];
        if (acc) acc[p * c->steps + s] = t.accepted_flags[s] ? 1 : 0;
      }
    }
    if (average) *average = rep.average_entropy;
    if (virtual_wall_ns) *virtual_wall_ns = rep.total_wall.count();
    return 0;
  } catch (const ConfigError& e) {
    return fail(e, -1);
  } catch (const std::exception& e) {
    return fail(e, -2);
  }
}

}  // extern "C"
