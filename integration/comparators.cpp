// comparators.cpp — the paper's GPU execution schemes on real hardware, built from the
// reference's OWN host code (for BASELINE.json config 5: "vs the paper's ranks-per-GPU
// scheme"). Not the product path: these are the baselines the persistent kernel replaces.
//
//  tasked  ("ranks per GPU", bench.cpp:186-197 semantics): R host threads
//           share one GPU, each with its own CUDA stream and cuBLAS handle (an MPI rank);
//           each runs the reference's spinmc::mc_procedure for its replicas with a GemmExecutor
//           that ships every GEMM to the device (H2D A, B; cublasZgemm; D2H rho).
//  batched (batchedGEMM, bench.cpp:248-298 semantics): all replicas advance in lock-step;
//           per step the host builds every proposal (reference gate/Haar code), one
//           cublasZgemmStridedBatched forms all rho = Psi Psi^H, the host decides (host
//           proposal / decision loops are OpenMP-parallel over replicas).
// Both report wall time and traces (which must match the oracle within tolerance).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "taskgemm/errors.hpp"
#include "taskgemm/exec.hpp"
#include "taskgemm/rng.hpp"
#include "taskgemm/spinmc.hpp"

using namespace taskgemm;
using linalg::Complex;
using linalg::ComplexMatrix;

namespace {
thread_local std::string g_err;

void ck(cudaError_t e, const char* w) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(w) + ": " + cudaGetErrorString(e));
}
void ckb(cublasStatus_t s, const char* w) {
  if (s != CUBLAS_STATUS_SUCCESS) throw std::runtime_error(std::string(w) + ": cublas status " + std::to_string(s));
}

// One "rank": its own stream + cuBLAS handle + device buffers; every GEMM goes to the GPU.
class CublasExecutor : public exec::GemmExecutor {
 public:
  // A rank is long-lived (an MPI process): stream, handle and device buffers are set up
  // once, before any timed work.
  explicit CublasExecutor(size_t reserve_bytes) {
    ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
    ckb(cublasCreate(&handle_), "cublasCreate");
    ckb(cublasSetStream(handle_, stream_), "cublasSetStream");
    ck(cudaMalloc(&dbuf_, reserve_bytes), "cudaMalloc");
    cap_ = reserve_bytes;
    origin_ = std::chrono::steady_clock::now();
  }
  ~CublasExecutor() override {
    cudaFree(dbuf_);
    cublasDestroy(handle_);
    cudaStreamDestroy(stream_);
  }
  ComplexMatrix run(exec::GemmTask t) override {
    const int m = static_cast<int>(t.a.rows()), n = static_cast<int>(t.b.cols()), k = static_cast<int>(t.a.cols());
    const size_t need = 16ull * (m * k + k * n + m * n);
    if (need > cap_) {
      cudaFree(dbuf_);
      ck(cudaMalloc(&dbuf_, need), "cudaMalloc");
      cap_ = need;
    }
    auto* A = static_cast<cuDoubleComplex*>(dbuf_);
    cuDoubleComplex* B = A + m * k;
    cuDoubleComplex* C = B + k * n;
    ck(cudaMemcpyAsync(A, t.a.data(), 16ull * m * k, cudaMemcpyHostToDevice, stream_), "H2D A");
    ck(cudaMemcpyAsync(B, t.b.data(), 16ull * k * n, cudaMemcpyHostToDevice, stream_), "H2D B");
    const cuDoubleComplex al = make_cuDoubleComplex(t.alpha.real(), t.alpha.imag());
    const cuDoubleComplex be = make_cuDoubleComplex(0.0, 0.0);  // C = 0 in the workload
    ckb(cublasZgemm(handle_, CUBLAS_OP_N, CUBLAS_OP_N, m, n, k, &al, A, m, B, k, &be, C, m), "zgemm");
    ComplexMatrix out(m, n);
    ck(cudaMemcpyAsync(out.data(), C, 16ull * m * n, cudaMemcpyDeviceToHost, stream_), "D2H");
    ck(cudaStreamSynchronize(stream_), "sync");
    ++gemms_;
    return out;
  }
  exec::VirtualTime now() override {
    return std::chrono::duration_cast<exec::VirtualTime>(std::chrono::steady_clock::now() - origin_);
  }
  uint64_t gemms() const { return gemms_; }

 private:
  cudaStream_t stream_{};
  cublasHandle_t handle_{};
  void* dbuf_ = nullptr;
  size_t cap_ = 0;
  uint64_t gemms_ = 0;
  std::chrono::steady_clock::time_point origin_;
};

spinmc::McConfig mc_of(int spins, uint64_t steps) {
  spinmc::McConfig mc;
  mc.spins = spins;
  mc.steps = steps;
  mc.entropy_kind = spinmc::EntropyKind::kRenyi2;
  return mc;
}

double renyi2_of(const ComplexMatrix& rho) {  // spinmc.cpp:171-175
  const double f = linalg::frobenius_norm(rho);
  const double e = -std::log(f * f);
  return std::max(e, 0.0);
}
}  // namespace

extern "C" {
const char* tgc_last_error() { return g_err.c_str(); }

// Ranks-per-GPU scheme: `ranks` host threads, replica p handled by rank p % ranks.
int tgc_tasked(int spins, uint64_t steps, uint64_t replicas, uint64_t seed, int ranks, double* init,
               double* ent, uint8_t* acc, int64_t* wall_ns) {
  try {
    const spinmc::McConfig mc = mc_of(spins, steps);
    const auto dims = spinmc::dims_for_spins(spins);
    const size_t bytes = 16 * (2 * dims.d_a * dims.d_b + dims.d_a * dims.d_a);
    std::vector<std::unique_ptr<CublasExecutor>> rank_ex;
    for (int r = 0; r < ranks; ++r) rank_ex.push_back(std::make_unique<CublasExecutor>(bytes));
    ck(cudaDeviceSynchronize(), "setup");
    std::vector<std::thread> th;
    std::mutex mu;
    std::string first;
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < ranks; ++r) {
      th.emplace_back([&, r] {
        try {
          CublasExecutor& ex = *rank_ex[r];
          for (uint64_t p = r; p < replicas; p += ranks) {
            auto st = rng::derive_stream({seed, static_cast<std::size_t>(p)});
            spinmc::EntropyTrace t = spinmc::mc_procedure(mc, p, st, ex);
            init[p] = t.initial_entropy;
            for (uint64_t s = 0; s < steps; ++s) {
              ent[p * steps + s] = t.entropies[s];
              acc[p * steps + s] = t.accepted_flags[s];
            }
          }
        } catch (const std::exception& e) {
          std::lock_guard lk(mu);
          if (first.empty()) first = e.what();
        }
      });
    }
    for (auto& t : th) t.join();
    *wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    if (!first.empty()) throw std::runtime_error(first);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// batchedGEMM scheme: lock-step over all replicas, one strided-batched ZGEMM per step.
int tgc_batched(int spins, uint64_t steps, uint64_t replicas, uint64_t seed, double* init, double* ent,
                uint8_t* acc, int64_t* wall_ns) {
  try {
    const auto dims = spinmc::dims_for_spins(spins);
    const int da = static_cast<int>(dims.d_a), db = static_cast<int>(dims.d_b);
    const size_t n_amp = size_t{1} << spins;
    spinmc::AnnealSchedule sched;  // t0 = 1, t_min = 1e-3 (spinmc.hpp:37-40)
    std::vector<rng::RandomStream> streams;
    std::vector<spinmc::SpinChainState> state(replicas), scratch(replicas);
    std::vector<double> cur(replicas);
    for (uint64_t p = 0; p < replicas; ++p) {
      streams.push_back(rng::derive_stream({seed, static_cast<std::size_t>(p)}));
      state[p] = spinmc::product_state(spins);
      scratch[p] = state[p];
    }
    cudaStream_t stream;
    cublasHandle_t h;
    ck(cudaStreamCreate(&stream), "stream");
    ckb(cublasCreate(&h), "cublasCreate");
    ckb(cublasSetStream(h, stream), "setStream");
    cuDoubleComplex *dpsi = nullptr, *drho = nullptr;
    ck(cudaMalloc(&dpsi, 16 * n_amp * replicas), "malloc psi");
    ck(cudaMalloc(&drho, 16ull * da * da * replicas), "malloc rho");
    std::vector<Complex> hrho(static_cast<size_t>(da) * da * replicas);
    const cuDoubleComplex one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
    // all rho = Psi Psi^H of the batch in one call (the GEMM of entanglement_entropy)
    auto batch_rho = [&](std::vector<spinmc::SpinChainState>& src) {
      for (uint64_t p = 0; p < replicas; ++p)
        ck(cudaMemcpyAsync(dpsi + p * n_amp, src[p].amplitudes.data(), 16 * n_amp, cudaMemcpyHostToDevice,
                           stream), "H2D");
      ckb(cublasZgemmStridedBatched(h, CUBLAS_OP_N, CUBLAS_OP_C, da, da, db, &one, dpsi, da,
                                    static_cast<long long>(n_amp), dpsi, da, static_cast<long long>(n_amp),
                                    &zero, drho, da, static_cast<long long>(da) * da,
                                    static_cast<int>(replicas)),
          "zgemmStridedBatched");
      ck(cudaMemcpyAsync(hrho.data(), drho, 16ull * da * da * replicas, cudaMemcpyDeviceToHost, stream), "D2H");
      ck(cudaStreamSynchronize(stream), "sync");
    };
    auto rho_of = [&](uint64_t p) {
      std::vector<Complex> v(hrho.begin() + p * da * da, hrho.begin() + (p + 1) * da * da);
      return ComplexMatrix(da, da, std::move(v));
    };
    const auto t0 = std::chrono::steady_clock::now();
    batch_rho(state);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < static_cast<int64_t>(replicas); ++p) cur[p] = init[p] = renyi2_of(rho_of(p));
    std::vector<int> sites(replicas);
    std::atomic<bool> bad{false};
    const int64_t nrep = static_cast<int64_t>(replicas);
    for (uint64_t s = 0; s < steps; ++s) {
#pragma omp parallel for schedule(static)
      for (int64_t p = 0; p < nrep; ++p) {  // metropolis_step, spinmc.cpp:198-200
        sites[p] = static_cast<int>(streams[p].uniform_index(spins - 1));
        const ComplexMatrix u = spinmc::haar_two_site_unitary(streams[p]);
        spinmc::apply_two_site_gate_into(state[p], sites[p], u, scratch[p]);
        const double nrm = spinmc::state_norm(scratch[p]);
        if (std::abs(nrm - 1.0) > 1e-9) bad = true;
      }
      if (bad) throw std::invalid_argument("entanglement_entropy: state not normalized");
      batch_rho(scratch);
#pragma omp parallel for schedule(static)
      for (int64_t p = 0; p < nrep; ++p) {  // spinmc.cpp:201-212
        const double proposed = renyi2_of(rho_of(p));
        const double delta = proposed - cur[p];
        const double pr = spinmc::acceptance_probability(delta, spinmc::temperature(sched, s, steps));
        const bool a = streams[p].uniform01() < pr;
        if (a) {
          std::swap(state[p].amplitudes, scratch[p].amplitudes);
          cur[p] = proposed;
        }
        ent[p * steps + s] = cur[p];
        acc[p * steps + s] = a;
        if ((s + 1) % 1000 == 0) spinmc::renormalize(state[p]);
      }
    }
    *wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
    cudaFree(dpsi);
    cudaFree(drho);
    cublasDestroy(h);
    cudaStreamDestroy(stream);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}
