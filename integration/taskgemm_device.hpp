// taskgemm_device.hpp — reference-side binding of the B200 path.
//
// Compiles against the reference's OWN headers (/root/reference/proj/include/taskgemm/*.hpp)
// and calls the C ABI (include/taskgemm_b200.h). This is the code a maintainer adds to the
// reference: a GEMM batcher with VirtualDevice::batched_gemm's contract (exec.hpp:146-147),
// a GemmExecutor (exec.hpp:196-201) so the reference's own spinmc::mc_procedure runs its
// GEMMs on the GPU, and bench::run_experiment for ExecutionMode "device" (bench.hpp:75).
#pragma once
#include <chrono>
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

// bench::run_experiment for ExecutionMode "device": one persistent kernel per GPU.
bench::RunReport run_experiment_device(const bench::ExperimentConfig& config);

}  // namespace taskgemm::device
