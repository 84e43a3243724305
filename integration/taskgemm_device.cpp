// taskgemm_device.cpp — see taskgemm_device.hpp. Written against the reference headers.
#include "taskgemm_device.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

#include "taskgemm/errors.hpp"
#include "taskgemm/spinmc.hpp"

namespace taskgemm::device {

void throw_on(tg_status s) {
  if (s == TG_OK) return;
  const std::string msg = tg_last_error();
  switch (s) {
    case TG_ECONFIG: throw ConfigError(msg);
    case TG_EINVAL: throw std::invalid_argument(msg);
    case TG_EKERNEL: {
      // "kernel failed for procedure N: what" -> exec::KernelError(N, what)
      const auto a = msg.find("procedure "), b = msg.find(": ");
      std::size_t p = 0;
      std::string what = msg;
      if (a != std::string::npos && b != std::string::npos && b > a) {
        p = std::stoull(msg.substr(a + 10, b - a - 10));
        what = msg.substr(b + 2);
      }
      throw exec::KernelError(p, what);
    }
    case TG_ESHUTDOWN: throw exec::SubmissionError(msg);
    default: throw std::runtime_error(msg);
  }
}

CudaDevice::CudaDevice(int gpu) { throw_on(tg_create(&gpu, 1, &ctx_)); }
CudaDevice::~CudaDevice() { tg_destroy(ctx_); }
void CudaDevice::shutdown() { throw_on(tg_shutdown(ctx_)); }

std::vector<linalg::ComplexMatrix> CudaDevice::batched_gemm(exec::GemmBatch batch) {
  return batched_gemm_at(std::move(batch), exec::VirtualTime{0}).results;
}

exec::BatchResult CudaDevice::batched_gemm_at(exec::GemmBatch batch, exec::VirtualTime when) {
  // exec.cpp:154-161: non-empty, fixed-size
  if (batch.tasks.empty()) throw std::invalid_argument("batched_gemm: batch must be non-empty");
  const auto& t0 = batch.tasks.front();
  for (const exec::GemmTask& t : batch.tasks)
    if (t.a.rows() != t0.a.rows() || t.b.cols() != t0.b.cols() || t.a.cols() != t0.a.cols())
      throw std::invalid_argument("batched_gemm: fixed-size contract violated, batch mixes GEMM shapes");
  for (const exec::GemmTask& t : batch.tasks) {  // linalg.cpp:59-73 messages
    if (t.a.cols() != t.b.rows())
      throw std::invalid_argument("gemm: A.cols (" + std::to_string(t.a.cols()) + ") != B.rows (" +
                                  std::to_string(t.b.rows()) + ")");
    if (t.c.rows() != t.a.rows() || t.c.cols() != t.b.cols())
      throw std::invalid_argument("gemm: C shape does not match A*B");
  }
  const int nb = static_cast<int>(batch.tasks.size());
  const int m = static_cast<int>(t0.a.rows()), n = static_cast<int>(t0.b.cols()), k = static_cast<int>(t0.a.cols());
  std::vector<const double*> A(nb), B(nb), C(nb);
  std::vector<double*> O(nb);
  std::vector<uint64_t> procs(nb);
  std::vector<tg_kernel_record> recs(nb);
  exec::BatchResult out;
  out.results.reserve(nb);
  for (int i = 0; i < nb; ++i) {
    const exec::GemmTask& t = batch.tasks[i];
    out.results.emplace_back(t.c.rows(), t.c.cols());
    A[i] = reinterpret_cast<const double*>(t.a.data());
    B[i] = reinterpret_cast<const double*>(t.b.data());
    C[i] = reinterpret_cast<const double*>(t.c.data());
    O[i] = reinterpret_cast<double*>(out.results.back().data());
    procs[i] = t.origin_procedure;
  }
  // One alpha/beta per batch in the ABI; per-task scalars are honoured by splitting.
  bool uniform = true;
  for (const exec::GemmTask& t : batch.tasks) uniform &= (t.alpha == t0.alpha && t.beta == t0.beta);
  const auto t_start = std::chrono::steady_clock::now();
  if (uniform) {
    const double al[2] = {t0.alpha.real(), t0.alpha.imag()}, be[2] = {t0.beta.real(), t0.beta.imag()};
    throw_on(tg_zgemm_batched(ctx_, 0, nb, m, n, k, al, A.data(), B.data(), be, C.data(), O.data(),
                              procs.data(), recs.data()));
  } else {
    for (int i = 0; i < nb; ++i) {
      const auto& t = batch.tasks[i];
      const double al[2] = {t.alpha.real(), t.alpha.imag()}, be[2] = {t.beta.real(), t.beta.imag()};
      throw_on(tg_zgemm_batched(ctx_, 0, 1, m, n, k, al, &A[i], &B[i], be, &C[i], &O[i], &procs[i], &recs[i]));
    }
  }
  const auto elapsed = std::chrono::steady_clock::now() - t_start;
  out.started_at = when;
  out.completed_at = when + std::chrono::duration_cast<exec::VirtualTime>(elapsed);
  for (const tg_kernel_record& r : recs) {
    exec::KernelRecord kr;
    kr.device_id = r.device_id;
    kr.procedure = r.procedure;
    kr.m = r.m;
    kr.n = r.n;
    kr.k = r.k;
    kr.queue_wait = exec::VirtualTime{r.queue_wait_ns};
    kr.exec_time = exec::VirtualTime{r.exec_time_ns};
    kr.flops = r.flops;
    out.records.push_back(kr);
  }
  records_.insert(records_.end(), out.records.begin(), out.records.end());
  return out;
}

CudaGemmExecutor::CudaGemmExecutor(CudaDevice& device, std::size_t procedure)
    : device_(device), procedure_(procedure), origin_(std::chrono::steady_clock::now()) {}

linalg::ComplexMatrix CudaGemmExecutor::run(exec::GemmTask task) {
  task.origin_procedure = procedure_;
  exec::GemmBatch b;
  b.tasks.push_back(std::move(task));
  return std::move(device_.batched_gemm(std::move(b)).front());
}

exec::VirtualTime CudaGemmExecutor::now() {
  return std::chrono::duration_cast<exec::VirtualTime>(std::chrono::steady_clock::now() - origin_);
}

namespace testhooks {
std::optional<GateFault> gate_fault;
}

bench::RunReport run_experiment_device(const bench::ExperimentConfig& config, DeviceAudit* audit) {
  bench::validate(config);
  tg_anneal_config c{};
  c.spins = static_cast<uint32_t>(config.spins);
  c.devices = static_cast<uint32_t>(config.devices);
  c.steps = config.steps;
  c.procedures = config.procedures;
  c.seed = config.seed;
  c.entropy_kind = config.entropy_kind == spinmc::EntropyKind::kRenyi2 ? TG_RENYI2 : TG_VON_NEUMANN;
  c.objective = config.objective == spinmc::Objective::kMaximize ? TG_MAXIMIZE : TG_MINIMIZE;
  c.initial_state = config.initial_state == spinmc::InitialState::kProduct ? TG_PRODUCT : TG_RANDOM;
  c.t0 = config.schedule.t0;
  c.t_min = config.schedule.t_min;
  c.renormalize_interval = spinmc::McConfig{}.renormalize_interval;
  c.shard_index = 0;
  c.shard_count = 1;
  if (testhooks::gate_fault) {
    c.inject_fault = 2;
    c.fault_procedure = testhooks::gate_fault->procedure;
    c.fault_step = testhooks::gate_fault->step;
  }
  const std::size_t np = config.procedures, s = config.steps, nd = config.devices;
  std::vector<double> init(np), ent(np * s), fin(np), dev_ms(nd);
  std::vector<uint8_t> acc(np * s);
  std::vector<int64_t> wall(np * s), init_wall(np);
  std::vector<uint64_t> resident(nd);
  std::vector<tg_near_tie> ties(audit ? 1024 : 0);
  tg_anneal_result r{};
  r.initial_entropy = init.data();
  r.entropies = ent.data();
  r.accepted = acc.data();
  r.final_entropy = fin.data();
  r.wall_ns = wall.data();
  r.initial_wall_ns = init_wall.data();
  r.device_kernel_ms = dev_ms.data();
  r.device_resident = resident.data();
  r.near_tie_log = ties.empty() ? nullptr : ties.data();
  r.near_tie_capacity = ties.size();
  std::vector<int> gpus(nd);
  for (std::size_t i = 0; i < gpus.size(); ++i) gpus[i] = static_cast<int>(i);
  tg_ctx* ctx = nullptr;
  throw_on(tg_create(gpus.data(), static_cast<int>(gpus.size()), &ctx));
  const tg_status st = tg_anneal_run(ctx, &c, &r);
  tg_destroy(ctx);
  throw_on(st);
  bench::RunReport rep;
  rep.config = config;
  rep.traces.resize(np);
  for (std::size_t p = 0; p < np; ++p) {
    spinmc::EntropyTrace& t = rep.traces[p];
    t.procedure_index = p;
    t.initial_entropy = init[p];
    t.entropies.assign(ent.begin() + p * s, ent.begin() + (p + 1) * s);
    t.accepted_flags.resize(s);
    t.wall_times.resize(s);
    for (std::size_t i = 0; i < s; ++i) {
      t.accepted_flags[i] = acc[p * s + i] != 0;
      t.wall_times[i] = exec::VirtualTime{wall[p * s + i]};
    }
  }
  // per device (bench.cpp:408-415): procedures p = d (mod devices), records, metrics
  const spinmc::BipartitionDims dims = spinmc::dims_for_spins(config.spins);
  const uint64_t gf = linalg::gemm_flops(dims.d_a, dims.d_a, dims.d_b);
  for (std::size_t d = 0; d < nd; ++d) {
    bench::DeviceReport dr;
    dr.device_id = d;
    for (std::size_t p = d; p < np; p += nd) dr.procedures.push_back(p);
    dr.records.reserve(dr.procedures.size() * (s + 1));
    auto add = [&](std::size_t p, int64_t ns) {
      exec::KernelRecord kr;
      kr.device_id = d;
      kr.procedure = p;
      kr.m = dims.d_a;
      kr.n = dims.d_a;
      kr.k = dims.d_b;
      kr.exec_time = exec::VirtualTime{std::max<int64_t>(ns, 1)};
      kr.flops = gf;
      dr.records.push_back(kr);
    };
    for (std::size_t p : dr.procedures) {
      add(p, init_wall[p]);  // initial-entropy GEMM (spinmc.cpp:234)
      for (std::size_t i = 0; i < s; ++i) add(p, wall[p * s + i]);
    }
    exec::DeviceMetrics& m = dr.metrics;
    m.kernel_count = dr.records.size();
    m.per_gemm_throughput.reserve(dr.records.size());
    for (const exec::KernelRecord& kr : dr.records) {
      m.total_flops += kr.flops;
      m.per_gemm_throughput.push_back(static_cast<double>(kr.flops) /
                                      std::chrono::duration<double>(kr.exec_time).count());
    }
    m.makespan = exec::VirtualTime{static_cast<int64_t>(dev_ms[d] * 1e6)};
    m.busy_time = m.makespan;
    m.idle_time = exec::VirtualTime{0};
    m.high_water_concurrency = resident[d];
    m.total_throughput = m.makespan.count() > 0
                             ? static_cast<double>(m.total_flops) / std::chrono::duration<double>(m.makespan).count()
                             : 0.0;
    rep.devices.push_back(std::move(dr));
  }
  rep.total_wall = exec::VirtualTime{r.total_wall_ns};
  rep.average_entropy = r.average_entropy;
  if (audit) {
    audit->fallback_decisions = r.fallback_decisions;
    audit->near_ties = r.near_ties;
    audit->near_tie_log.assign(ties.begin(), ties.begin() + std::min<uint64_t>(r.near_ties, ties.size()));
  }
  return rep;
}

}  // namespace taskgemm::device
