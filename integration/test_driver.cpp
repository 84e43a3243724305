// test_driver.cpp — C entry points so tests/test_integration_reference_api.py can drive the
// reference-side binding (taskgemm_device.hpp) through the reference's OWN C++ API.
#include <algorithm>
#include <cstring>
#include <string>

#include "taskgemm/errors.hpp"
#include "taskgemm/report_io.hpp"
#include "taskgemm/spinmc.hpp"
#include "taskgemm_device.hpp"

using namespace taskgemm;

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = std::string("ConfigError: ") + e.what();
    return 1;
  } catch (const exec::KernelError& e) {
    g_err = std::string("KernelError: ") + e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = std::string("exception: ") + e.what();
    return 5;
  }
}
}  // namespace

extern "C" {
const char* tgi_last_error() { return g_err.c_str(); }

// The reference's own spinmc::mc_procedure (spinmc.cpp:215-251), GEMMs on the GPU via
// CudaGemmExecutor: host loop identical to the reference, only the GEMM differs.
int tgi_mc_procedure_cuda(int spins, uint64_t steps, uint64_t seed, uint64_t p, int kind,
                          double* init, double* ent, uint8_t* acc) {
  return guard([&] {
    device::CudaDevice dev(0);
    device::CudaGemmExecutor ex(dev, p);
    spinmc::McConfig mc;
    mc.spins = spins;
    mc.steps = steps;
    mc.entropy_kind = kind == 0 ? spinmc::EntropyKind::kVonNeumann : spinmc::EntropyKind::kRenyi2;
    auto stream = rng::derive_stream({seed, p});
    spinmc::EntropyTrace t = spinmc::mc_procedure(mc, p, stream, ex);
    *init = t.initial_entropy;
    for (uint64_t s = 0; s < steps; ++s) {
      ent[s] = t.entropies[s];
      acc[s] = t.accepted_flags[s];
    }
    if (dev.records().size() != steps + 1) throw std::runtime_error("one KernelRecord per GEMM expected");
  });
}

// bench::run_experiment in ExecutionMode "device".
int tgi_run_experiment_device(int spins, uint64_t steps, uint64_t procedures, uint64_t devices,
                              uint64_t seed, int objective, int initial, double* init, double* ent,
                              uint8_t* acc, double* average) {
  return guard([&] {
    bench::ExperimentConfig cfg;
    cfg.spins = spins;
    cfg.steps = steps;
    cfg.procedures = procedures;
    cfg.devices = devices;
    cfg.seed = seed;
    cfg.objective = objective == 0 ? spinmc::Objective::kMaximize : spinmc::Objective::kMinimize;
    cfg.initial_state = initial == 0 ? spinmc::InitialState::kProduct : spinmc::InitialState::kRandom;
    bench::RunReport rep = device::run_experiment_device(cfg);
    for (uint64_t p = 0; p < procedures; ++p) {
      init[p] = rep.traces[p].initial_entropy;
      for (uint64_t s = 0; s < steps; ++s) {
        ent[p * steps + s] = rep.traces[p].entropies[s];
        acc[p * steps + s] = rep.traces[p].accepted_flags[s];
      }
    }
    *average = rep.average_entropy;
    // the reference's own helper accepts the report (same-workload check, bench.cpp:440-455)
    if (bench::speedup(rep, rep) != 1.0) throw std::runtime_error("speedup(rep, rep) != 1");
    if (steps > 0 && spinmc::average_entropy(rep.traces) != rep.average_entropy)
      throw std::runtime_error("average_entropy differs from spinmc::average_entropy");
  });
}

// run_experiment_device with testhooks::gate_fault set on (fault_procedure, fault_step):
// the reference contract is std::invalid_argument "entanglement_entropy: state not
// normalized (||psi|| = ...)" (spinmc.cpp:152-156, rethrown by bench.cpp:387-395) -> rc 2.
int tgi_run_experiment_device_fault(int spins, uint64_t steps, uint64_t procedures, int kind,
                                    uint64_t fault_procedure, uint64_t fault_step) {
  device::testhooks::gate_fault = device::testhooks::GateFault{fault_procedure, fault_step};
  const int rc = guard([&] {
    bench::ExperimentConfig cfg;
    cfg.spins = spins;
    cfg.steps = steps;
    cfg.procedures = procedures;
    cfg.entropy_kind = kind == 0 ? spinmc::EntropyKind::kVonNeumann : spinmc::EntropyKind::kRenyi2;
    device::run_experiment_device(cfg);
  });
  device::testhooks::gate_fault.reset();
  return rc;
}

// RunReport completeness: run in device mode, then serialise with the reference's own
// report_io::report_json and kernel_csv / trace_csv. Returns the JSON in `json` (cap
// bytes), and stats = {records per device..., wall_times > 0 count, kernel_csv lines,
// trace_csv lines, fallback decisions, near ties}.
int tgi_run_experiment_report(int spins, uint64_t steps, uint64_t procedures, uint64_t devices, int kind,
                              int objective, double t_min, char* json, uint64_t cap, uint64_t* stats) {
  return guard([&] {
    bench::ExperimentConfig cfg;
    cfg.spins = spins;
    cfg.steps = steps;
    cfg.procedures = procedures;
    cfg.devices = devices;
    cfg.entropy_kind = kind == 0 ? spinmc::EntropyKind::kVonNeumann : spinmc::EntropyKind::kRenyi2;
    cfg.objective = objective == 0 ? spinmc::Objective::kMaximize : spinmc::Objective::kMinimize;
    cfg.schedule.t_min = t_min;
    device::DeviceAudit audit;
    bench::RunReport rep = device::run_experiment_device(cfg, &audit);
    const std::string j = report_io::report_json(rep);
    if (j.size() + 1 > cap) throw std::runtime_error("json buffer too small");
    std::memcpy(json, j.c_str(), j.size() + 1);
    uint64_t positive = 0;
    for (const auto& t : rep.traces)
      for (const auto& w : t.wall_times) positive += w.count() > 0;
    auto lines = [](const std::string& x) { return static_cast<uint64_t>(std::count(x.begin(), x.end(), '\n')); };
    for (std::size_t d = 0; d < devices; ++d) stats[d] = rep.devices.at(d).records.size();
    stats[devices] = positive;
    stats[devices + 1] = lines(report_io::kernel_csv(rep));
    stats[devices + 2] = lines(report_io::trace_csv(rep.traces));
    stats[devices + 3] = audit.fallback_decisions;
    stats[devices + 4] = audit.near_ties;
  });
}

// Batched GEMM through the reference's GemmBatch/GemmTask types. mode 0: valid batch of
// `batch` random (m,n,k) GEMMs compared against linalg::gemm (max relative error returned);
// 1: mixed shapes (expects "fixed-size"); 2: empty batch; 3: dims mismatch.
int tgi_batched_gemm(int mode, int batch, int m, int n, int k, double* max_rel_err) {
  return guard([&] {
    device::CudaDevice dev(0);
    exec::GemmBatch b;
    auto stream = rng::derive_stream({77, 0});
    auto rnd = [&](std::size_t r, std::size_t c) {
      linalg::ComplexMatrix x(r, c);
      for (std::size_t j = 0; j < c; ++j)
        for (std::size_t i = 0; i < r; ++i) {
          auto [re, im] = stream.standard_normal_pair();
          x(i, j) = {re, im};
        }
      return x;
    };
    if (mode == 2) {
      dev.batched_gemm(std::move(b));
      return;
    }
    for (int i = 0; i < batch; ++i) {
      exec::GemmTask t;
      const int kk = (mode == 3 && i == 0) ? k + 1 : k;
      const int mm = (mode == 1 && i == batch - 1) ? m + 1 : m;
      t.a = rnd(mm, kk);
      t.b = rnd(k, n);
      t.c = rnd(mm, n);
      t.alpha = {0.5, -1.25};
      t.beta = {2.0, 0.75};
      t.origin_procedure = 1000 + i;
      b.tasks.push_back(std::move(t));
    }
    std::vector<exec::GemmTask> copy = b.tasks;
    exec::BatchResult res = dev.batched_gemm_at(std::move(b), exec::VirtualTime{5});
    double err = 0.0;
    for (int i = 0; i < batch; ++i) {
      const auto& t = copy[i];
      linalg::ComplexMatrix want = linalg::gemm(t.alpha, t.a, t.b, t.beta, t.c);
      double mx = 0.0, e = 0.0;
      for (std::size_t q = 0; q < want.size(); ++q) {
        mx = std::max(mx, std::abs(want.data()[q]));
        e = std::max(e, std::abs(want.data()[q] - res.results[i].data()[q]));
      }
      err = std::max(err, e / mx);
      if (res.records[i].procedure != static_cast<std::size_t>(1000 + i) ||
          res.records[i].flops != linalg::gemm_flops(m, n, k))
        throw std::runtime_error("KernelRecord mismatch");
    }
    *max_rel_err = err;
  });
}
}
