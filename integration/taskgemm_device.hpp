// taskgemm_device.hpp — reference-side binding of the B200 path.
//
// Compiles against the reference's OWN headers (/root/reference/proj/include/taskgemm/*.hpp)
// and calls the C ABI (include/taskgemm_b200.h). This is the code a maintainer adds to the
// reference: a GEMM batcher with VirtualDevice::batched_gemm's contract (exec.hpp:146-147),
// a GemmExecutor (exec.hpp:196-201) so the reference's own spinmc::mc_procedure runs its
// GEMMs on the GPU, and bench::run_experiment for ExecutionMode "device" (bench.hpp:75).
#pragma once
#include <chrono>
#include <cstdint>
#include <optional>
#include <vector>

#include "taskgemm/bench.hpp"
#include "taskgemm/exec.hpp"
#include "taskgemm_b200.h"

namespace taskgemm::device {

// Maps a non-OK tg_status to the reference's exception types.
void throw_on(tg_status s);

class CudaDevice {
 public:
  explicit CudaDevice(int gpu = 0);
  ~CudaDevice();
  CudaDevice(const CudaDevice&) = delete;
  CudaDevice& operator=(const CudaDevice&) = delete;

  std::vector<linalg::ComplexMatrix> batched_gemm(exec::GemmBatch batch);
  exec::BatchResult batched_gemm_at(exec::GemmBatch batch, exec::VirtualTime when);
  void shutdown();
  std::vector<exec::KernelRecord> records() const { return records_; }

 private:
  tg_ctx* ctx_ = nullptr;
  std::vector<exec::KernelRecord> records_;
};

// Per-GEMM executor: every executor.run() is a device batch of one (the paper's
// "one rank per GEMM" scheme when many threads each own one).
class CudaGemmExecutor : public exec::GemmExecutor {
 public:
  CudaGemmExecutor(CudaDevice& device, std::size_t procedure);
  linalg::ComplexMatrix run(exec::GemmTask task) override;
  exec::VirtualTime now() override;

 private:
  CudaDevice& device_;
  std::size_t procedure_;
  std::chrono::steady_clock::time_point origin_;
};

// Decision audit of a device run (tg_anneal_result): decisions whose lean
// margin fell inside the rounding window and were re-taken with the reference formula, and
// the accept tests with |u - p| < 1e-9, logged in (procedure, step) order.
struct DeviceAudit {
  std::uint64_t fallback_decisions = 0;
  std::uint64_t near_ties = 0;
  std::vector<tg_near_tie> near_tie_log;
};

namespace testhooks {
// Like linalg::testhooks::perturb_gemm (linalg.hpp:74-79): while set, run_experiment_device
// scales the Haar gate of (procedure, step) by 1.001, so that proposal fails the norm check
// of entanglement_entropy (spinmc.cpp:152-156) and the run throws std::invalid_argument.
struct GateFault {
  std::size_t procedure = 0, step = 0;
};
extern std::optional<GateFault> gate_fault;
}  // namespace testhooks

// bench::run_experiment for ExecutionMode "device": one persistent kernel per GPU. Fills
// the RunReport as the reference does (bench.cpp:396-415): traces with per-step wall
// times (device %globaltimer, spinmc.cpp:238-245), and per device its procedures, one
// KernelRecord per GEMM (the initial-entropy GEMM and one per step; exec_time = that
// step's device time) and DeviceMetrics (the persistent kernel is the device's one job:
// busy = makespan = its device time, high water = its resident replicas).
bench::RunReport run_experiment_device(const bench::ExperimentConfig& config, DeviceAudit* audit = nullptr);

}  // namespace taskgemm::device
