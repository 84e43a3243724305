// capi.cpp — host side of the C ABI (include/taskgemm_b200.h).
//
// Replaces, for ExecutionMode::kDevice, the reference's annealing driver
// (bench::run_experiment, bench.cpp:341-417) and GEMM batcher (VirtualDevice::batched_gemm,
// exec.cpp:144-221): configuration validation with the reference's messages, the
// p -> device binding (bench.cpp:171), one host thread per GPU, one persistent kernel per
// GPU, trace copy-back and the procedure-order average (spinmc.cpp:253-269). There is no
// CPU fallback: without a CUDA device every entry point fails with TG_ECUDA.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/taskgemm_b200.h"
#include "tg_internal.h"

namespace {

thread_local std::string g_err;
std::atomic<int> g_perturb{0};  // tg_set_perturb_gemm

tg_status fail(tg_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

tg_status cuda_fail(cudaError_t e, const char* where) {
  return fail(TG_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define TG_CUDA(call)                                         \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);       \
  } while (0)

struct DeviceState {
  int ordinal = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;  // trace copy-back of finished waves, overlapping the last wave
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_part = nullptr;
  // grow-only device buffers reused across calls
  void* trace = nullptr;
  size_t trace_bytes = 0;
  void* workspace = nullptr;
  size_t workspace_bytes = 0;
  // batched GEMM (tg_zgemm_batched): device operands and two pinned host staging slots
  void* gemm_dev = nullptr;
  size_t gemm_dev_bytes = 0;
  void* gemm_pin = nullptr;
  size_t gemm_pin_bytes = 0;
  double* gather = nullptr;  // NCCL all-gather of the final entropies: [send: maxrows][recv: D x maxrows]
  size_t gather_bytes = 0;
};

}  // namespace

struct tg_ctx {
  std::vector<DeviceState> devs;
  std::vector<ncclComm_t> comms;  // in-process NCCL communicator over devs (distinct GPUs), lazily
  bool comms_tried = false;
  std::mutex mu;
  bool shutdown = false;
};

namespace {

// NCCL, loaded at run time: the process may already hold torch's libnccl.so.2 (same soname),
// which dlopen then returns; linking one at build time could pin a second version first.
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
};
const NcclApi* nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!a.h) return a;
    a.CommInitAll = reinterpret_cast<decltype(a.CommInitAll)>(dlsym(a.h, "ncclCommInitAll"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(a.h, "ncclAllGather"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(a.h, "ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(a.h, "ncclGroupEnd"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(a.h, "ncclCommDestroy"));
    if (!a.CommInitAll || !a.AllGather || !a.GroupStart || !a.GroupEnd || !a.CommDestroy) a.h = nullptr;
    return a;
  }();
  return api.h ? &api : nullptr;
}

uint64_t rows_for(const tg_anneal_config* c) {
  const uint64_t sc = c->shard_count ? c->shard_count : 1;
  if (c->shard_index >= c->procedures) return 0;
  return (c->procedures - c->shard_index + sc - 1) / sc;
}

// bench::validate (bench.cpp:321-329) + dims_for_spins (spinmc.cpp:15-26) + device tiers.
tg_status validate(const tg_anneal_config* c) {
  if (!c) return fail(TG_EINVAL, "config must not be NULL");
  if (c->spins < 2 || c->spins > 30)
    return fail(TG_ECONFIG, "spins out of range [2,30]: " + std::to_string(c->spins));
  if (c->procedures < 1) return fail(TG_ECONFIG, "procedures must be >= 1");
  if (c->devices < 1) return fail(TG_ECONFIG, "devices must be >= 1");
  if (!(c->t0 > 0.0) || !(c->t_min > 0.0) || c->t_min > c->t0)
    return fail(TG_ECONFIG, "anneal schedule requires 0 < t_min <= t0");
  const uint32_t sc = c->shard_count ? c->shard_count : 1;
  if (c->shard_index >= sc) return fail(TG_ECONFIG, "shard_index must be < shard_count");
  if (c->spins > 24)
    return fail(TG_EINVAL, "device tiers cover spins <= 24 (state of 2^" + std::to_string(c->spins) +
                               " amplitudes per replica)");
  if (c->entropy_kind != TG_RENYI2 && c->entropy_kind != TG_VON_NEUMANN)
    return fail(TG_ECONFIG, "entropy_kind must be von-neumann or renyi-2");
  if (c->entropy_kind == TG_VON_NEUMANN && c->spins > static_cast<uint32_t>(tg::kVnQueueMaxSpins))
    return fail(TG_EINVAL, "device von-neumann entropy covers spins <= " + std::to_string(tg::kVnQueueMaxSpins) +
                               " (d_a <= 1024); use renyi-2");
  if (c->inject_fault < 0 || c->inject_fault > 2) return fail(TG_ECONFIG, "inject_fault must be 0, 1 or 2");
  if (c->rho_half != 0 && c->rho_half != 1) return fail(TG_ECONFIG, "rho_half must be 0 or 1");
  if (c->rho_half && c->entropy_kind != TG_RENYI2)
    return fail(TG_ECONFIG, "rho_half (Hermitian half of rho) needs renyi-2 (the eigen-solvers take the full rho)");
  if (c->objective != TG_MAXIMIZE && c->objective != TG_MINIMIZE)
    return fail(TG_ECONFIG, "objective must be max or min");
  if (c->initial_state != TG_PRODUCT && c->initial_state != TG_RANDOM)
    return fail(TG_ECONFIG, "initial_state must be product or random");
  // the proposal pre-pass jumps each replica's stream ahead by GF(2) matrix powers
  // (gate_stream.cu, kJumpBits): runs up to 2^22 steps per replica
  if (c->steps > tg::kMaxSteps)
    return fail(TG_ECONFIG, "steps (" + std::to_string(c->steps) + ") exceed the device path's limit of " +
                                std::to_string(tg::kMaxSteps) + " steps per procedure");
  return TG_OK;
}

tg::AnnealParams make_params(const tg_anneal_config* c, uint64_t rows, uint64_t p_first,
                             uint64_t p_stride) {
  tg::AnnealParams p{};
  p.spins = c->spins;
  p.objective = c->objective;
  p.initial_state = c->initial_state;
  p.inject_fault = (c->inject_fault == 1 || g_perturb.load()) ? 1 : 0;  // GEMM perturbation only
  p.gate_fault = c->inject_fault == 2;
  p.fault_procedure = c->fault_procedure;
  p.fault_step = c->fault_step;
  p.rho_half = c->rho_half;
  p.fault_row1 = 0;
  p.tie_eps = 1e-9;  // SURVEY.md §8c near tie; tests widen it to exercise the audit log
  if (const char* e = std::getenv("TG_NEAR_TIE_EPS")) {
    const double v = std::atof(e);
    if (v > 0.0 && v < 0.5) p.tie_eps = v;
  }
  p.gate_bulk = 1;
  if (const char* e = std::getenv("TG_GATE_BULK")) p.gate_bulk = std::atoi(e);
  p.gate_bulk_min = 16;
  if (const char* e = std::getenv("TG_GATE_BULK_MIN")) p.gate_bulk_min = std::atoi(e);
  p.gate_chunk = 0;
  if (const char* e = std::getenv("TG_GATE_CHUNK")) {
    const int v = std::atoi(e);
    if (v >= 64 && v <= 1024 && (v & (v - 1)) == 0) p.gate_chunk = v;
  }
  p.entropy_kind = c->entropy_kind;
  p.steps = c->steps;
  p.seed = c->seed;
  p.renorm = c->renormalize_interval;
  p.t0 = c->t0;
  p.t_min = c->t_min;
  p.rows = rows;
  p.p_first = p_first;
  p.p_stride = p_stride;
  return p;
}

// Replicas per batch are capped so the pre-generated proposal stream (288 B per
// replica-step + raw draws) stays within this many bytes of workspace.
constexpr size_t kStreamBudget = size_t{16} << 30;

// HBM-tier slabs for any launch of up to `rows` replicas: a sub-range (the batch tail, the
// e2e split) can pick a different cluster geometry than the full batch, so the region is
// sized for the most clusters any row count <= rows can use (anneal_hbm_workspace_bytes).
size_t slab_bytes(uint32_t spins, uint64_t rows, int device, int entropy_kind) {
  return spins > static_cast<uint32_t>(tg::kSmemMaxSpins) ? tg::anneal_hbm_workspace_bytes(spins, rows, device, entropy_kind)
                                                         : 0;
}
uint64_t slab_clusters(uint32_t spins, uint64_t rows, int device) {
  return spins > static_cast<uint32_t>(tg::kSmemMaxSpins) ? tg::anneal_hbm_slab_clusters(rows, device) : 0;
}

// Workspace for one launch: [proposal stream of one batch][HBM-tier slabs] (+ alignment).
size_t workspace_for(const tg::AnnealParams& p, int device) {
  const size_t per_row = tg::gate_stream_bytes_per_row(p.spins, p.steps, p.initial_state == 1);
  uint64_t batch = std::max<uint64_t>(1, std::min<uint64_t>(p.rows, kStreamBudget / per_row));
  if (p.rho_half || (p.entropy_kind == TG_VON_NEUMANN && p.spins >= static_cast<uint32_t>(tg::kVnQueueMinSpins)))
    batch = std::max<uint64_t>(1, std::min<uint64_t>(batch, tg::anneal_hbm_queue_max_rows(p.spins, p.entropy_kind)));
  return batch * per_row + slab_bytes(p.spins, batch, device, p.entropy_kind) + 1024;
}

// Kernels this library has launched (process lifetime): tg_kernel_launches().
std::atomic<uint64_t> g_launches{0};

// The whole device pipeline of one launch, on one stream: per batch of replicas, the
// proposal-stream pre-pass (gate_stream.cu) then the persistent anneal kernel.
cudaError_t launch(const tg::AnnealParams& p, void* ws, size_t ws_bytes, cudaStream_t s,
                   bool trace = false) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (p.rows == 0) return cudaSuccess;
  const size_t per_row = tg::gate_stream_bytes_per_row(p.spins, p.steps, p.initial_state == 1);
  uint64_t batch = std::min<uint64_t>(p.rows, kStreamBudget / per_row);
  const bool queue_only = p.rho_half || (p.entropy_kind == TG_VON_NEUMANN && p.spins >= static_cast<uint32_t>(tg::kVnQueueMinSpins));
  if (queue_only) batch = std::min<uint64_t>(batch, tg::anneal_hbm_queue_max_rows(p.spins, p.entropy_kind));
  while (batch > 0 && batch * per_row + slab_bytes(p.spins, batch, dev, p.entropy_kind) + 1024 > ws_bytes) --batch;
  if (batch == 0) return cudaErrorMemoryAllocation;
  const size_t stream_bytes = batch * per_row;
  char* base = static_cast<char*>(ws);
  char* slabs = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(base + stream_bytes) + 255) & ~uintptr_t{255});
  for (uint64_t b0 = 0; b0 < p.rows; b0 += batch) {
    tg::AnnealParams q = p;
    q.rows = std::min<uint64_t>(batch, p.rows - b0);
    q.p_first = p.p_first + b0 * p.p_stride;
    q.fault_row1 = 0;
    if (p.gate_fault && p.fault_procedure >= q.p_first && (p.fault_procedure - q.p_first) % p.p_stride == 0 &&
        (p.fault_procedure - q.p_first) / p.p_stride < q.rows)
      q.fault_row1 = 1 + (p.fault_procedure - q.p_first) / p.p_stride;
    const uint64_t o = b0 * p.steps;
    q.initial_entropy = p.initial_entropy + b0;
    q.final_entropy = p.final_entropy ? p.final_entropy + b0 : nullptr;
    q.status = p.status + b0;
    q.status_step = p.status_step + b0;
    q.status_norm = p.status_norm ? p.status_norm + b0 : nullptr;
    q.initial_wall_ns = p.initial_wall_ns ? p.initial_wall_ns + b0 : nullptr;
    q.entropies = p.entropies + o;
    q.accepted = p.accepted + o;
    q.sites = p.sites ? p.sites + o : nullptr;
    q.wall_ns = p.wall_ns ? p.wall_ns + o : nullptr;
    tg::GateStream gs{};
    cudaError_t e = tg::launch_gate_stream(q, base, stream_bytes, &gs, s);
    if (e != cudaSuccess) return e;
    g_launches += p.initial_state == 1 ? 3 : 2;  // rng_chunk (fused records), rng_fixup (, init_convert)
    q.gates = gs.recs;
    q.init_states = gs.init_states;
    q.workspace = reinterpret_cast<double*>(slabs);
    q.slab_clusters = slab_clusters(p.spins, batch, dev);
    q.queue_rows = p.spins > static_cast<uint32_t>(tg::kSmemMaxSpins) ? tg::anneal_hbm_queue_rows(p.spins, batch, p.entropy_kind) : 0;
    e = p.spins <= static_cast<uint32_t>(tg::kSmemMaxSpins) ? tg::launch_anneal_smem(q, s, nullptr, trace)
                                                           : tg::launch_anneal_hbm(q, s, nullptr, trace);
    if (e != cudaSuccess) return e;
    // anneal kernel (+ finish_renyi_kernel for Renyi-2: traces are stored as raw ||rho||_F^2)
    g_launches += p.entropy_kind == TG_RENYI2 ? 2 : 1;
  }
  return cudaSuccess;
}

template <class T>
T* carve(char*& cursor, size_t count) {
  cursor = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(cursor) + 255) & ~uintptr_t{255});
  T* p = reinterpret_cast<T*>(cursor);
  cursor += count * sizeof(T);
  return p;
}

size_t trace_bytes(uint64_t rows, uint64_t steps, bool sites, bool wall, uint64_t ties = 0) {
  const size_t rs = rows * steps;
  return rows * (8 + 8 + 4 + 8 + 8 + 8) + rs * (8 + 1) + (sites ? rs : 0) + (wall ? rs * 8 : 0) + 16 +
         ties * sizeof(tg_near_tie) + 10 * 256;
}

// reference message of spinmc.cpp:153-155 (std::to_string(double) is "%f")
std::string not_normalized_message(double nrm) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%f", nrm);
  return std::string("entanglement_entropy: state not normalized (||psi|| = ") + buf + ")";
}

}  // namespace

extern "C" {

const char* tg_last_error(void) { return g_err.c_str(); }
uint64_t tg_kernel_launches(void) { return g_launches.load(); }

const char* tg_version(void) { return "taskgemm-b200 0.1 (sm_100a, DMMA.8x8x4 persistent anneal)"; }

uint64_t tg_anneal_rows(const tg_anneal_config* cfg) { return cfg ? rows_for(cfg) : 0; }

uint64_t tg_step_flops(uint32_t spins) {
  if (spins < 2 || spins > 30) return 0;
  const uint64_t da = uint64_t{1} << (spins / 2), db = uint64_t{1} << (spins - spins / 2);
  return 8ull * da * da * db;  // gemm_flops(d_a, d_a, d_b), linalg.cpp:140-144
}

tg_status tg_validate(const tg_anneal_config* cfg) { return validate(cfg); }

tg_status tg_create(const int* gpus, int n, tg_ctx** out) {
  if (!out) return fail(TG_EINVAL, "out must not be NULL");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return fail(TG_ECUDA, std::string("no CUDA device available (") + cudaGetErrorString(e) +
                              "); the device path has no CPU fallback");
  if (n < 1) return fail(TG_ECONFIG, "devices must be >= 1");
  auto ctx = std::make_unique<tg_ctx>();
  for (int i = 0; i < n; ++i) {
    DeviceState d;
    d.ordinal = gpus ? gpus[i] : i;
    if (d.ordinal < 0 || d.ordinal >= count)
      return fail(TG_ECONFIG, "GPU ordinal " + std::to_string(d.ordinal) + " out of range (" +
                                  std::to_string(count) + " visible)");
    TG_CUDA(cudaSetDevice(d.ordinal));
    TG_CUDA(cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking));
    TG_CUDA(cudaStreamCreateWithFlags(&d.copy, cudaStreamNonBlocking));
    TG_CUDA(cudaEventCreate(&d.ev0));
    TG_CUDA(cudaEventCreate(&d.ev1));
    TG_CUDA(cudaEventCreateWithFlags(&d.ev_part, cudaEventDisableTiming));
    ctx->devs.push_back(d);
  }
  *out = ctx.release();
  return TG_OK;
}

tg_status tg_shutdown(tg_ctx* ctx) {
  if (!ctx) return fail(TG_EINVAL, "ctx must not be NULL");
  std::lock_guard<std::mutex> lk(ctx->mu);
  ctx->shutdown = true;
  return TG_OK;
}

tg_status tg_destroy(tg_ctx* ctx) {
  if (!ctx) return TG_OK;
  if (const NcclApi* n = nccl_api())
    for (ncclComm_t cm : ctx->comms) n->CommDestroy(cm);
  for (auto& d : ctx->devs) {
    cudaSetDevice(d.ordinal);
    cudaStreamSynchronize(d.stream);
    if (d.trace) cudaFree(d.trace);
    if (d.workspace) cudaFree(d.workspace);
    if (d.gemm_dev) cudaFree(d.gemm_dev);
    if (d.gemm_pin) cudaFreeHost(d.gemm_pin);
    if (d.gather) cudaFree(d.gather);
    cudaStreamSynchronize(d.copy);
    cudaEventDestroy(d.ev0);
    cudaEventDestroy(d.ev1);
    cudaEventDestroy(d.ev_part);
    cudaStreamDestroy(d.stream);
    cudaStreamDestroy(d.copy);
  }
  delete ctx;
  return TG_OK;
}

size_t tg_anneal_workspace_bytes(const tg_anneal_config* cfg) {
  if (!cfg || cfg->spins < 2 || cfg->spins > 24) return 0;
  int dev = 0;
  cudaGetDevice(&dev);
  return workspace_for(make_params(cfg, rows_for(cfg), 0, 1), dev);
}

tg_status tg_anneal_launch(const tg_anneal_config* cfg, const tg_anneal_device_buffers* b,
                           void* stream) {
  if (tg_status s = validate(cfg)) return s;
  if (!b || !b->initial_entropy || !b->entropies || !b->accepted || !b->final_entropy ||
      !b->status || !b->status_step)
    return fail(TG_EINVAL, "device buffers initial_entropy/entropies/accepted/final_entropy/status "
                           "must not be NULL");
  const uint64_t rows = rows_for(cfg);
  tg::AnnealParams p = make_params(cfg, rows, cfg->shard_index, cfg->shard_count ? cfg->shard_count : 1);
  p.initial_entropy = b->initial_entropy;
  p.entropies = b->entropies;
  p.accepted = b->accepted;
  p.sites = b->sites;
  p.wall_ns = b->wall_ns;
  p.final_entropy = b->final_entropy;
  p.status = b->status;
  p.status_step = b->status_step;
  p.status_norm = b->status_norm;
  p.initial_wall_ns = b->initial_wall_ns;
  p.tie_stats = reinterpret_cast<unsigned long long*>(b->tie_stats);
  p.tie_log = b->tie_log;
  p.tie_capacity = b->tie_log ? b->tie_capacity : 0;
  if (!b->workspace && rows > 0)
    return fail(TG_EINVAL, "workspace required (tg_anneal_workspace_bytes)");
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e = launch(p, b->workspace, workspace_for(p, dev), static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "anneal launch");
  return TG_OK;
}

tg_status tg_anneal_run(tg_ctx* ctx, const tg_anneal_config* cfg, tg_anneal_result* res) {
  if (!ctx) return fail(TG_EINVAL, "ctx must not be NULL");
  if (tg_status s = validate(cfg)) return s;
  if (!res || !res->initial_entropy || !res->entropies || !res->accepted)
    return fail(TG_EINVAL, "result arrays initial_entropy/entropies/accepted must not be NULL");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (ctx->shutdown) return fail(TG_ESHUTDOWN, "VirtualDevice: submit after shutdown");
  if (cfg->devices > ctx->devs.size())
    return fail(TG_ECONFIG, "devices (" + std::to_string(cfg->devices) + ") exceeds the context's " +
                                std::to_string(ctx->devs.size()) + " GPUs");
  const auto t_begin = std::chrono::steady_clock::now();
  const uint64_t rows = rows_for(cfg);
  const uint64_t D = cfg->devices;
  const uint64_t sc = cfg->shard_count ? cfg->shard_count : 1;
  const uint64_t steps = cfg->steps;
  const bool want_sites = res->sites != nullptr, want_wall = res->wall_ns != nullptr;
  const bool want_init_wall = res->initial_wall_ns != nullptr;

  std::vector<tg_status> st(D, TG_OK);
  std::vector<std::string> msg(D);
  std::vector<float> ms(D, 0.f);
  std::vector<std::vector<int32_t>> status(D);
  std::vector<std::vector<int64_t>> status_step(D);
  std::vector<std::vector<double>> status_norm(D);
  std::vector<std::vector<int64_t>> iwall(D);
  std::vector<uint64_t> resident(D, 0);
  std::vector<std::vector<double>> finals(D);
  std::vector<double*> fin_dev(D, nullptr);  // the device copy of each GPU's final entropies
  std::vector<unsigned long long> tie_stats(2 * D, 0);
  std::vector<std::vector<tg_near_tie>> ties(D);

  auto worker = [&](uint64_t g) {
    DeviceState& d = ctx->devs[g];
    auto err = [&](tg_status s, const std::string& m) {
      st[g] = s;
      msg[g] = m;
    };
    auto cu = [&](cudaError_t e, const char* w) {
      if (e != cudaSuccess) err(TG_ECUDA, std::string(w) + ": " + cudaGetErrorString(e));
      return e == cudaSuccess;
    };
    if (!cu(cudaSetDevice(d.ordinal), "cudaSetDevice")) return;
    const uint64_t lrows = rows > g ? (rows - g + D - 1) / D : 0;
    if (lrows == 0) return;
    // device buffers (grow-only)
    const uint64_t tie_cap = res->near_tie_log ? res->near_tie_capacity : 0;
    const size_t need = trace_bytes(lrows, steps, want_sites, want_wall, tie_cap);
    if (need > d.trace_bytes) {
      if (d.trace) cudaFree(d.trace);
      d.trace = nullptr;
      d.trace_bytes = 0;
      if (!cu(cudaMalloc(&d.trace, need), "cudaMalloc(traces)")) return;
      d.trace_bytes = need;
    }
    char* cur = static_cast<char*>(d.trace);
    tg::AnnealParams p = make_params(cfg, lrows, cfg->shard_index + g * sc, D * sc);
    p.initial_entropy = carve<double>(cur, lrows);
    p.final_entropy = carve<double>(cur, lrows);
    p.status = carve<int32_t>(cur, lrows);
    p.status_step = carve<int64_t>(cur, lrows);
    p.entropies = carve<double>(cur, lrows * steps);
    p.accepted = carve<uint8_t>(cur, lrows * steps);
    p.sites = want_sites ? carve<uint8_t>(cur, lrows * steps) : nullptr;
    p.wall_ns = want_wall ? carve<int64_t>(cur, lrows * steps) : nullptr;
    p.status_norm = carve<double>(cur, lrows);
    p.initial_wall_ns = want_init_wall ? carve<int64_t>(cur, lrows) : nullptr;
    p.tie_stats = carve<unsigned long long>(cur, 2);
    p.tie_log = tie_cap ? carve<tg_near_tie>(cur, tie_cap) : nullptr;
    p.tie_capacity = tie_cap;
    if (!cu(cudaMemsetAsync(p.tie_stats, 0, 16, d.stream), "cudaMemsetAsync")) return;
    const size_t ws = workspace_for(p, d.ordinal);
    if (ws > d.workspace_bytes) {
      if (d.workspace) cudaFree(d.workspace);
      d.workspace = nullptr;
      d.workspace_bytes = 0;
      if (!cu(cudaMalloc(&d.workspace, ws), "cudaMalloc(workspace)")) return;
      d.workspace_bytes = ws;
    }
    // Replicas run in waves of `wave` (resident CTAs / clusters). With D == 1 the traces go
    // straight into the caller's arrays, so the rows of all full waves but the last are
    // launched first and copied back on a second stream while the remaining rows run.
    // A device-to-pageable copy blocks the host until it completes, which would serialise
    // the two launches: split only when the caller's trace arrays are page-locked.
    auto pinned = [](const void* h) {
      cudaPointerAttributes a{};
      if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      return a.type == cudaMemoryTypeHost;
    };
    uint64_t split = 0;
    if (D == 1 && steps > 0 && pinned(res->entropies) && pinned(res->accepted) &&
        (!want_sites || pinned(res->sites)) && (!want_wall || pinned(res->wall_ns))) {
      const uint64_t wave = p.spins <= static_cast<uint32_t>(tg::kSmemMaxSpins) ? tg::anneal_smem_wave_rows(p)
                                                                                : tg::anneal_hbm_wave_rows(p);
      if (wave > 0 && lrows > wave) split = lrows % wave ? lrows - lrows % wave : lrows - wave;
    }
    auto rows_of = [&](uint64_t r0, uint64_t r1) {  // AnnealParams of host rows [r0, r1)
      tg::AnnealParams q = p;
      q.rows = r1 - r0;
      q.p_first = p.p_first + r0 * p.p_stride;
      q.initial_entropy = p.initial_entropy + r0;
      q.final_entropy = p.final_entropy + r0;
      q.status = p.status + r0;
      q.status_step = p.status_step + r0;
      q.status_norm = p.status_norm + r0;
      q.initial_wall_ns = p.initial_wall_ns ? p.initial_wall_ns + r0 : nullptr;
      q.entropies = p.entropies + r0 * steps;
      q.accepted = p.accepted + r0 * steps;
      q.sites = p.sites ? p.sites + r0 * steps : nullptr;
      q.wall_ns = p.wall_ns ? p.wall_ns + r0 * steps : nullptr;
      return q;
    };
    std::vector<double> init(lrows), fin(lrows), ent(D > 1 ? lrows * steps : 0);
    std::vector<uint8_t> acc(D > 1 ? lrows * steps : 0), sit(want_sites && D > 1 ? lrows * steps : 0);
    std::vector<int64_t> wall(want_wall && D > 1 ? lrows * steps : 0);
    status[g].resize(lrows);
    status_step[g].resize(lrows);
    status_norm[g].resize(lrows);
    iwall[g].resize(want_init_wall ? lrows : 0);
    resident[g] = std::min<uint64_t>(lrows, p.spins <= static_cast<uint32_t>(tg::kSmemMaxSpins)
                                                ? tg::anneal_smem_wave_rows(p)
                                                : tg::anneal_hbm_wave_rows(p));
    // trace rows [r0, r1) -> host (caller arrays when D == 1) on stream `st`
    auto copy_back = [&](uint64_t r0, uint64_t r1, cudaStream_t st) {
      const uint64_t n = r1 - r0, o = r0 * steps, ns = n * steps;
      bool ok = cu(cudaMemcpyAsync(init.data() + r0, p.initial_entropy + r0, 8 * n, cudaMemcpyDeviceToHost, st), "D2H") &&
                cu(cudaMemcpyAsync(fin.data() + r0, p.final_entropy + r0, 8 * n, cudaMemcpyDeviceToHost, st), "D2H") &&
                cu(cudaMemcpyAsync(status[g].data() + r0, p.status + r0, 4 * n, cudaMemcpyDeviceToHost, st), "D2H") &&
                cu(cudaMemcpyAsync(status_step[g].data() + r0, p.status_step + r0, 8 * n, cudaMemcpyDeviceToHost, st), "D2H") &&
                cu(cudaMemcpyAsync(status_norm[g].data() + r0, p.status_norm + r0, 8 * n, cudaMemcpyDeviceToHost, st), "D2H") &&
                (!want_init_wall ||
                 cu(cudaMemcpyAsync(iwall[g].data() + r0, p.initial_wall_ns + r0, 8 * n, cudaMemcpyDeviceToHost, st), "D2H"));
      if (ok && steps > 0) {
        // D == 1 and host rows contiguous: copy straight into the caller's arrays
        double* ent_dst = D == 1 ? res->entropies + o : ent.data() + o;
        uint8_t* acc_dst = D == 1 ? res->accepted + o : acc.data() + o;
        ok = cu(cudaMemcpyAsync(ent_dst, p.entropies + o, 8 * ns, cudaMemcpyDeviceToHost, st), "D2H") &&
             cu(cudaMemcpyAsync(acc_dst, p.accepted + o, ns, cudaMemcpyDeviceToHost, st), "D2H");
        if (ok && want_sites)
          ok = cu(cudaMemcpyAsync(D == 1 ? res->sites + o : sit.data() + o, p.sites + o, ns, cudaMemcpyDeviceToHost, st), "D2H");
        if (ok && want_wall)
          ok = cu(cudaMemcpyAsync(D == 1 ? res->wall_ns + o : wall.data() + o, p.wall_ns + o, 8 * ns,
                                  cudaMemcpyDeviceToHost, st), "D2H");
      }
      return ok;
    };
    if (!cu(cudaEventRecord(d.ev0, d.stream), "cudaEventRecord")) return;
    bool ok = true;
    if (split > 0) {
      if (!cu(launch(rows_of(0, split), d.workspace, d.workspace_bytes, d.stream), "anneal launch")) return;
      if (!cu(cudaEventRecord(d.ev_part, d.stream), "cudaEventRecord")) return;
      if (!cu(cudaStreamWaitEvent(d.copy, d.ev_part, 0), "cudaStreamWaitEvent")) return;
      ok = copy_back(0, split, d.copy);
      if (!ok) return;
      if (!cu(launch(rows_of(split, lrows), d.workspace, d.workspace_bytes, d.stream), "anneal launch")) return;
    } else {
      if (!cu(launch(p, d.workspace, d.workspace_bytes, d.stream), "anneal launch")) return;
    }
    if (!cu(cudaEventRecord(d.ev1, d.stream), "cudaEventRecord")) return;
    ok = copy_back(split, lrows, d.stream);
    if (ok && split > 0) ok = cu(cudaStreamSynchronize(d.copy), "trace copy");
    if (!ok) return;
    if (!cu(cudaMemcpyAsync(&tie_stats[2 * g], p.tie_stats, 16, cudaMemcpyDeviceToHost, d.stream), "D2H")) return;
    if (!cu(cudaStreamSynchronize(d.stream), "anneal kernel")) return;
    cudaEventElapsedTime(&ms[g], d.ev0, d.ev1);
    const uint64_t nlog = std::min<uint64_t>(tie_stats[2 * g + 1], tie_cap);
    ties[g].resize(nlog);
    if (nlog && !cu(cudaMemcpy(ties[g].data(), p.tie_log, nlog * sizeof(tg_near_tie), cudaMemcpyDeviceToHost), "D2H"))
      return;
    for (uint64_t q = 0; q < lrows; ++q) {
      const uint64_t hr = g + D * q;
      res->initial_entropy[hr] = init[q];
      if (want_init_wall) res->initial_wall_ns[hr] = iwall[g][q];
      if (res->final_entropy) res->final_entropy[hr] = fin[q];
      if (D > 1 && steps > 0) {
        std::memcpy(res->entropies + hr * steps, ent.data() + q * steps, 8 * steps);
        std::memcpy(res->accepted + hr * steps, acc.data() + q * steps, steps);
        if (want_sites) std::memcpy(res->sites + hr * steps, sit.data() + q * steps, steps);
        if (want_wall) std::memcpy(res->wall_ns + hr * steps, wall.data() + q * steps, 8 * steps);
      }
    }
    finals[g] = std::move(fin);
    fin_dev[g] = p.final_entropy;
  };

  if (D == 1) {
    worker(0);
  } else {
    std::vector<std::thread> th;
    for (uint64_t g = 0; g < D; ++g) th.emplace_back(worker, g);
    for (auto& t : th) t.join();
  }
  for (uint64_t g = 0; g < D; ++g)
    if (st[g] != TG_OK) return fail(st[g], msg[g]);
  // the first procedure (in procedure order) whose state left normalization: the reference
  // throws std::invalid_argument from entanglement_entropy (spinmc.cpp:152-156) and
  // run_experiment rethrows the first procedure error unchanged (bench.cpp:387-395)
  for (uint64_t hr = 0; hr < rows; ++hr) {
    const uint64_t g = hr % D, q = hr / D;
    if (status[g][q] != tg::kRowOk) return fail(TG_EINVAL, not_normalized_message(status_norm[g][q]));
  }
  // decision audit: counts over all GPUs, the logged near ties in (procedure, step) order
  res->fallback_decisions = 0;
  res->near_ties = 0;
  std::vector<tg_near_tie> all_ties;
  for (uint64_t g = 0; g < D; ++g) {
    res->fallback_decisions += tie_stats[2 * g];
    res->near_ties += tie_stats[2 * g + 1];
    all_ties.insert(all_ties.end(), ties[g].begin(), ties[g].end());
  }
  std::sort(all_ties.begin(), all_ties.end(), [](const tg_near_tie& a, const tg_near_tie& b) {
    return a.procedure != b.procedure ? a.procedure < b.procedure : a.step < b.step;
  });
  if (res->near_tie_log)
    for (uint64_t i = 0; i < std::min<uint64_t>(all_ties.size(), res->near_tie_capacity); ++i)
      res->near_tie_log[i] = all_ties[i];
  if (res->device_kernel_ms)
    for (uint64_t g = 0; g < D; ++g) res->device_kernel_ms[g] = ms[g];
  if (res->device_resident)
    for (uint64_t g = 0; g < D; ++g) res->device_resident[g] = resident[g];
  // The final entropies of all GPUs, for the average: one NCCL all-gather over the context's
  // GPUs (the run's only collective), launched as a group from this thread
  // once every GPU's anneal has finished; the host copies are the fallback (GPUs repeated in
  // the context, NCCL unavailable, TG_NCCL=0). TG_NCCL_FORCE=1 also gathers with one GPU.
  res->nccl_ranks = 0;
  if (steps > 0 && (D > 1 || std::getenv("TG_NCCL_FORCE")) && !(std::getenv("TG_NCCL") && std::getenv("TG_NCCL")[0] == '0')) {
    const NcclApi* n = nccl_api();
    if (n && !ctx->comms_tried) {
      ctx->comms_tried = true;
      std::vector<int> ord(ctx->devs.size());
      for (size_t g = 0; g < ord.size(); ++g) ord[g] = ctx->devs[g].ordinal;
      std::vector<int> sorted = ord;
      std::sort(sorted.begin(), sorted.end());
      if (std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end()) {  // NCCL: one rank per GPU
        std::vector<ncclComm_t> cm(ord.size());
        if (n->CommInitAll(cm.data(), static_cast<int>(ord.size()), ord.data()) == ncclSuccess) ctx->comms = cm;
      }
    }
    if (n && ctx->comms.size() == D) {  // every rank of the communicator takes part
      uint64_t maxrows = 0;
      for (uint64_t g = 0; g < D; ++g) maxrows = std::max<uint64_t>(maxrows, finals[g].size());
      bool ok = maxrows > 0;
      for (uint64_t g = 0; g < D && ok; ++g) {  // send buffer: this GPU's finals, zero padded
        DeviceState& d = ctx->devs[g];
        const size_t need = 8 * maxrows * (D + 1);
        ok = cudaSetDevice(d.ordinal) == cudaSuccess;
        if (ok && d.gather_bytes < need) {
          if (d.gather) cudaFree(d.gather);
          d.gather = nullptr;
          d.gather_bytes = 0;
          ok = cudaMalloc(&d.gather, need) == cudaSuccess;
          if (ok) d.gather_bytes = need;
        }
        ok = ok && cudaMemsetAsync(d.gather, 0, 8 * maxrows, d.stream) == cudaSuccess &&
             cudaMemcpyAsync(d.gather, fin_dev[g], 8 * finals[g].size(), cudaMemcpyDeviceToDevice, d.stream) ==
                 cudaSuccess;
      }
      if (ok) {
        ok = n->GroupStart() == ncclSuccess;
        for (uint64_t g = 0; g < D && ok; ++g) {
          DeviceState& d = ctx->devs[g];
          ok = cudaSetDevice(d.ordinal) == cudaSuccess &&
               n->AllGather(d.gather, d.gather + maxrows, maxrows, ncclFloat64, ctx->comms[g], d.stream) == ncclSuccess;
        }
        ok = (n->GroupEnd() == ncclSuccess) && ok;
      }
      std::vector<double> all(D * maxrows);
      for (uint64_t g = 0; g < D && ok; ++g) {
        DeviceState& d = ctx->devs[g];
        ok = cudaSetDevice(d.ordinal) == cudaSuccess && cudaStreamSynchronize(d.stream) == cudaSuccess;
      }
      ok = ok && cudaSetDevice(ctx->devs[0].ordinal) == cudaSuccess &&
           cudaMemcpy(all.data(), ctx->devs[0].gather + maxrows, 8 * D * maxrows, cudaMemcpyDeviceToHost) == cudaSuccess;
      if (ok) {
        for (uint64_t g = 0; g < D; ++g)
          for (uint64_t q = 0; q < finals[g].size(); ++q) finals[g][q] = all[g * maxrows + q];
        res->nccl_ranks = static_cast<uint32_t>(D);
      } else {
        cudaGetLastError();  // host copies stay the source of the average
      }
    }
  }
  double sum = 0.0;  // procedure order, spinmc.cpp:259-268 / bench.cpp:401-407
  for (uint64_t hr = 0; hr < rows; ++hr)
    sum += steps > 0 ? finals[hr % D][hr / D] : res->initial_entropy[hr];
  res->average_entropy = rows ? sum / static_cast<double>(rows) : 0.0;
  res->total_flops = (rows * steps + rows) * tg_step_flops(cfg->spins);
  res->executed_flops = res->total_flops;
  if (cfg->rho_half) {  // upper-triangle blocks only: nb (nb + 1) / 2 of nb^2
    // (HBM tier: 64x64 tiles; SMEM tier: 8x8 blocks of the padded d_a >= 8 rows)
    const uint64_t da = uint64_t{1} << (cfg->spins / 2);
    const uint64_t nb = cfg->spins > static_cast<uint32_t>(tg::kSmemMaxSpins) ? da / 64 : std::max<uint64_t>(da, 8) / 8;
    res->executed_flops = res->total_flops / (nb * nb) * (nb * (nb + 1) / 2);
  }
  res->kernel_ms = *std::max_element(ms.begin(), ms.end());
  res->total_wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(
                           std::chrono::steady_clock::now() - t_begin)
                           .count();
  return TG_OK;
}

tg_status tg_zgemm_strided_launch(int batch, int m, int n, int k, const double alpha[2],
                                  const double* A, int64_t sA, const double* B, int64_t sB,
                                  const double beta[2], const double* C, int64_t sC, double* out,
                                  int64_t sO, int inject_fault, void* stream) {
  if (batch < 1) return fail(TG_EINVAL, "batched_gemm: batch must be non-empty");
  if (m < 1 || n < 1 || k < 1) return fail(TG_EINVAL, "gemm: dims must be >= 1");
  if (!alpha || !beta || !A || !B || !out) return fail(TG_EINVAL, "gemm: NULL operand");
  cudaError_t e = tg::launch_zgemm_strided(batch, m, n, k, alpha[0], alpha[1], A, sA, B, sB, beta[0],
                                           beta[1], C, sC, out, sO, inject_fault || g_perturb.load(),
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "zgemm launch");
  ++g_launches;
  return TG_OK;
}

tg_status tg_zgemm_batched(tg_ctx* ctx, int device, int batch, int m, int n, int k,
                           const double alpha[2], const double* const* A, const double* const* B,
                           const double beta[2], const double* const* C, double* const* out,
                           const uint64_t* procedures, tg_kernel_record* records) {
  if (!ctx) return fail(TG_EINVAL, "ctx must not be NULL");
  if (batch < 1) return fail(TG_EINVAL, "batched_gemm: batch must be non-empty");
  if (m < 1 || n < 1 || k < 1) return fail(TG_EINVAL, "gemm: dims must be >= 1");
  if (!alpha || !beta || !A || !B || !out) return fail(TG_EINVAL, "gemm: NULL operand");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (ctx->shutdown) return fail(TG_ESHUTDOWN, "VirtualDevice: submit after shutdown");
  if (device < 0 || static_cast<size_t>(device) >= ctx->devs.size())
    return fail(TG_EINVAL, "device index out of range");
  DeviceState& d = ctx->devs[device];
  TG_CUDA(cudaSetDevice(d.ordinal));
  // Column-major interleaved complex128 operands, copied in and out by the library
  // (GemmTask ownership, exec.hpp:30-31). The batch runs in chunks through two pinned host
  // slots: while chunk c is on the device (H2D, kernel, D2H on the stream), the host packs
  // chunk c+1 into the other slot and unpacks chunk c-1; the device buffer and the pinned
  // slots are grow-only and reused across calls.
  const size_t ea = 2ull * m * k, eb = 2ull * k * n, ec = 2ull * m * n;  // doubles per entry
  const bool has_c = C != nullptr;
  const size_t in_per = ea + eb + (has_c ? ec : 0), per = in_per + ec;
  constexpr size_t kChunkBytes = size_t{64} << 20;
  const int chunk = static_cast<int>(std::max<size_t>(1, std::min<size_t>(batch, kChunkBytes / (8 * per))));
  const int nchunks = (batch + chunk - 1) / chunk;
  const size_t slot = 8 * per * static_cast<size_t>(chunk);
  const size_t dev_bytes = nchunks > 1 ? 2 * slot : slot;
  if (d.gemm_dev_bytes < dev_bytes) {
    if (d.gemm_dev) cudaFree(d.gemm_dev);
    d.gemm_dev = nullptr;
    d.gemm_dev_bytes = 0;
    TG_CUDA(cudaMalloc(&d.gemm_dev, dev_bytes));
    d.gemm_dev_bytes = dev_bytes;
  }
  if (d.gemm_pin_bytes < dev_bytes) {
    if (d.gemm_pin) cudaFreeHost(d.gemm_pin);
    d.gemm_pin = nullptr;
    d.gemm_pin_bytes = 0;
    TG_CUDA(cudaMallocHost(&d.gemm_pin, dev_bytes));
    d.gemm_pin_bytes = dev_bytes;
  }
  // host copies of `count` entries, split over threads when large
  auto par_copy = [](int count, size_t bytes_each, auto&& one) {
    const size_t total = bytes_each * static_cast<size_t>(count);
    const int nt = total >= (size_t{8} << 20) ? std::min(8, std::max(1, static_cast<int>(std::thread::hardware_concurrency()))) : 1;
    if (nt <= 1 || count < 2) {
      for (int i = 0; i < count; ++i) one(i);
      return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        for (int i = t; i < count; i += nt) one(i);
      });
    for (auto& x : th) x.join();
  };
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<cudaEvent_t> evs(2 * nchunks + 2, nullptr);
  struct EvGuard {
    std::vector<cudaEvent_t>& v;
    ~EvGuard() {
      for (auto e : v)
        if (e) cudaEventDestroy(e);
    }
  } ev_guard{evs};
  for (auto& ev : evs) TG_CUDA(cudaEventCreate(&ev));
  cudaEvent_t* kev = evs.data();                 // kernel start/end per chunk
  cudaEvent_t* done = evs.data() + 2 * nchunks;  // slot reuse: D2H of the slot's last chunk
  auto unpack = [&](int c) {
    const int b0 = c * chunk, cnt = std::min(chunk, batch - b0);
    const double* hs = reinterpret_cast<const double*>(static_cast<char*>(d.gemm_pin) + (c & 1) * slot);
    const double* ho = hs + static_cast<size_t>(cnt) * in_per;
    par_copy(cnt, 8 * ec, [&](int i) { std::memcpy(out[b0 + i], ho + i * ec, 8 * ec); });
  };
  for (int c = 0; c < nchunks; ++c) {
    const int b0 = c * chunk, cnt = std::min(chunk, batch - b0);
    char* hslot = static_cast<char*>(d.gemm_pin) + (c & 1) * slot;
    char* dslot = static_cast<char*>(d.gemm_dev) + (c & 1) * slot;
    if (c >= 2) {  // the slot's previous chunk (c - 2): results out before the slot is reused
      TG_CUDA(cudaEventSynchronize(done[c & 1]));
      unpack(c - 2);
    }
    double* hA = reinterpret_cast<double*>(hslot);
    double* hB = hA + static_cast<size_t>(cnt) * ea;
    double* hC = hB + static_cast<size_t>(cnt) * eb;
    par_copy(cnt, 8 * (ea + eb + (has_c ? ec : 0)), [&](int i) {
      std::memcpy(hA + i * ea, A[b0 + i], 8 * ea);
      std::memcpy(hB + i * eb, B[b0 + i], 8 * eb);
      if (has_c) std::memcpy(hC + i * ec, C[b0 + i], 8 * ec);
    });
    const size_t in_bytes = 8 * in_per * static_cast<size_t>(cnt);
    TG_CUDA(cudaMemcpyAsync(dslot, hslot, in_bytes, cudaMemcpyHostToDevice, d.stream));
    double* dA = reinterpret_cast<double*>(dslot);
    double* dB = dA + static_cast<size_t>(cnt) * ea;
    double* dC = has_c ? dB + static_cast<size_t>(cnt) * eb : nullptr;
    double* dO = dA + static_cast<size_t>(cnt) * in_per;
    TG_CUDA(cudaEventRecord(kev[2 * c], d.stream));
    cudaError_t e = tg::launch_zgemm_strided(cnt, m, n, k, alpha[0], alpha[1], dA, ea / 2, dB, eb / 2, beta[0],
                                             beta[1], dC, ec / 2, dO, ec / 2, g_perturb.load(), d.stream);
    if (e != cudaSuccess) return cuda_fail(e, "zgemm launch");
    ++g_launches;
    TG_CUDA(cudaEventRecord(kev[2 * c + 1], d.stream));
    TG_CUDA(cudaMemcpyAsync(hslot + in_bytes, dO, 8 * ec * static_cast<size_t>(cnt), cudaMemcpyDeviceToHost, d.stream));
    TG_CUDA(cudaEventRecord(done[c & 1], d.stream));
  }
  TG_CUDA(cudaStreamSynchronize(d.stream));
  for (int c = std::max(0, nchunks - 2); c < nchunks; ++c) unpack(c);
  float kms = 0.f;
  for (int c = 0; c < nchunks; ++c) {
    float x = 0.f;
    cudaEventElapsedTime(&x, kev[2 * c], kev[2 * c + 1]);
    kms += x;
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (records) {
    const int64_t exec_ns = std::max<int64_t>(1, static_cast<int64_t>(kms * 1e6 / batch));
    const int64_t wait_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count() -
                            static_cast<int64_t>(kms * 1e6);
    for (int i = 0; i < batch; ++i) {
      records[i].device_id = static_cast<uint64_t>(device);
      records[i].procedure = procedures ? procedures[i] : static_cast<uint64_t>(i);
      records[i].m = m;
      records[i].n = n;
      records[i].k = k;
      records[i].queue_wait_ns = std::max<int64_t>(0, wait_ns);
      records[i].exec_time_ns = exec_ns;
      records[i].flops = 8ull * m * n * k;
    }
  }
  return TG_OK;
}

tg_status tg_set_perturb_gemm(int on) {
  g_perturb.store(on ? 1 : 0);
  return TG_OK;
}

tg_status tg_fp64_dmma_peak(int device, double* tflops, double* clock_ghz) {
  if (!tflops) return fail(TG_EINVAL, "tflops must not be NULL");
  TG_CUDA(cudaSetDevice(device));
  TG_CUDA(tg::fp64_dmma_peak(tflops, clock_ghz));
  return TG_OK;
}

int tg_hbm_schedule(uint32_t spins, uint64_t rows, int32_t entropy_kind) {
  if (spins <= static_cast<uint32_t>(tg::kSmemMaxSpins) || spins > 24) return -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  tg::AnnealParams p{};
  p.spins = spins;
  p.rows = rows;
  p.entropy_kind = entropy_kind;
  return tg::anneal_hbm_schedule(p, dev);
}

// ------------------------------------------------------------------------- probes
tg_status tg_probe_rng(uint64_t seed, uint64_t p, uint64_t n, uint64_t* out) {
  uint64_t* d = nullptr;
  TG_CUDA(cudaMalloc(&d, 8 * std::max<uint64_t>(n, 1)));
  cudaError_t e = tg::probe_rng(seed, p, n, d, nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(out, d, 8 * n, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "probe_rng");
  return TG_OK;
}

tg_status tg_probe_gates(uint32_t spins, uint64_t seed, uint64_t p, uint64_t steps,
                         int initial_state, uint8_t* sites, double* u, double* uacc) {
  if (spins < 2 || spins > 30) return fail(TG_ECONFIG, "spins out of range [2,30]: " + std::to_string(spins));
  char* d = nullptr;
  const size_t n = std::max<uint64_t>(steps, 1);
  TG_CUDA(cudaMalloc(&d, n * (1 + 32 * 8 + 8) + 512));
  double* du = reinterpret_cast<double*>(d);
  double* da = du + 32 * n;
  uint8_t* ds = reinterpret_cast<uint8_t*>(da + n);
  cudaError_t e = tg::probe_gates(spins, seed, p, steps, initial_state, ds, du, da, nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(sites, ds, steps, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(u, du, 8 * 32 * steps, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(uacc, da, 8 * steps, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "probe_gates");
  return TG_OK;
}

tg_status tg_probe_apply_gate(uint32_t spins, const double* psi, int site, const double* u,
                              double* out) {
  if (spins < 2 || spins > 24) return fail(TG_EINVAL, "probe_apply_gate: spins must be in [2,24]");
  if (site < 0 || static_cast<uint32_t>(site) + 2 > spins)
    return fail(TG_EINVAL, "apply_two_site_gate: site " + std::to_string(site) + " out of range [0," +
                               std::to_string(spins - 2) + "]");
  const size_t n = size_t{1} << spins;
  double* d = nullptr;
  TG_CUDA(cudaMalloc(&d, 8 * (4 * n + 32)));
  double *dp = d, *dout = d + 2 * n, *du = d + 4 * n;
  cudaError_t e = cudaMemcpy(dp, psi, 16 * n, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(du, u, 256, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = tg::probe_apply_gate(spins, dp, site, du, dout, nullptr);
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, 16 * n, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "probe_apply_gate");
  return TG_OK;
}

tg_status tg_probe_entropy_kind(uint32_t spins, uint64_t count, const double* psi, int32_t kind,
                                double* entropy, double* norms) {
  if (spins < 2 || spins > 24) return fail(TG_EINVAL, "probe_entropy: spins must be in [2,24]");
  if (kind != TG_RENYI2 && kind != TG_VON_NEUMANN) return fail(TG_ECONFIG, "probe_entropy: unknown entropy kind");
  if (kind == TG_VON_NEUMANN && spins > static_cast<uint32_t>(tg::kVnMaxSpins))
    return fail(TG_EINVAL, "probe_entropy: device von-neumann covers spins <= " + std::to_string(tg::kVnMaxSpins));
  if (count < 1) return TG_OK;
  const size_t n = size_t{1} << spins;
  double* d = nullptr;
  TG_CUDA(cudaMalloc(&d, 8 * (2 * n * count + 2 * count)));
  double *dp = d, *de = d + 2 * n * count, *dn = de + count;
  cudaError_t e = cudaMemcpy(dp, psi, 16 * n * count, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = tg::probe_entropy(spins, count, dp, de, dn, g_perturb.load() != 0, nullptr, kind == TG_VON_NEUMANN);
  if (e == cudaSuccess) e = cudaMemcpy(entropy, de, 8 * count, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && norms) e = cudaMemcpy(norms, dn, 8 * count, cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "probe_entropy");
  return TG_OK;
}

tg_status tg_probe_entropy(uint32_t spins, uint64_t count, const double* psi, double* entropy,
                           double* norms) {
  return tg_probe_entropy_kind(spins, count, psi, TG_RENYI2, entropy, norms);
}

uint64_t tg_rng_chunk_steps(void) { return tg::rng_chunk_steps(); }

tg_status tg_rng_jump_words(uint64_t seed, uint64_t p, int32_t init_spins, uint64_t chunks, uint64_t extra,
                            uint64_t n, uint64_t* out) {
  if (!out && n) return fail(TG_EINVAL, "out must not be NULL");
  if (init_spins > 24 || chunks >= (uint64_t{1} << 16)) return fail(TG_EINVAL, "rng_jump_words: init_spins <= 24, chunks < 2^16");
  tg::rng_jump_words(seed, p, init_spins, chunks, extra, n, out);
  return TG_OK;
}

tg_status tg_probe_rng_chunking(uint32_t spins, uint64_t rows, uint64_t steps, int32_t random_init,
                                uint64_t reject_below, uint64_t* mismatches) {
  if (!mismatches) return fail(TG_EINVAL, "mismatches must not be NULL");
  if (spins < 3 || spins > 24 || rows == 0) return fail(TG_EINVAL, "probe_rng_chunking: spins in [3,24], rows > 0");
  TG_CUDA(tg::probe_rng_chunking(spins, rows, steps, random_init, reject_below, mismatches));
  return TG_OK;
}

tg_status tg_probe_phase_trace(uint32_t spins, uint64_t replicas, uint64_t steps, int64_t* trace) {
  if (spins < 2 || spins > 24) return fail(TG_EINVAL, "phase trace covers spins in [2,24]");
  tg_anneal_config c{};
  c.spins = spins;
  c.devices = 1;
  c.steps = steps;
  c.procedures = replicas;
  c.entropy_kind = TG_RENYI2;
  c.t0 = 1.0;
  c.t_min = 1e-3;
  c.renormalize_interval = 1000;
  c.shard_count = 1;
  tg::AnnealParams p = make_params(&c, replicas, 0, 1);
  char* d = nullptr;
  const size_t bytes = trace_bytes(replicas, steps, false, false) + 64 * std::max<uint64_t>(steps, 1);
  TG_CUDA(cudaMalloc(&d, bytes));
  char* cur = d;
  p.initial_entropy = carve<double>(cur, replicas);
  p.final_entropy = carve<double>(cur, replicas);
  p.status = carve<int32_t>(cur, replicas);
  p.status_step = carve<int64_t>(cur, replicas);
  p.entropies = carve<double>(cur, replicas * steps);
  p.accepted = carve<uint8_t>(cur, replicas * steps);
  int64_t* tr = carve<int64_t>(cur, 8 * steps);
  p.trace = tr;
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t wsb = workspace_for(p, dev);
  void* ws = nullptr;
  cudaError_t e = cudaMalloc(&ws, wsb);
  if (e == cudaSuccess) e = cudaMemset(tr, 0, 64 * steps);
  if (e == cudaSuccess) e = launch(p, ws, wsb, nullptr, /*trace=*/true);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(trace, tr, 64 * steps, cudaMemcpyDeviceToHost);
  cudaFree(ws);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "probe_phase_trace");
  return TG_OK;
}

tg_status tg_probe_queue_stats(uint32_t spins, uint64_t replicas, uint64_t steps, int32_t entropy_kind, int64_t* stats,
                               int* ctas) {
  if (spins <= static_cast<uint32_t>(tg::kSmemMaxSpins) || spins > 24) return fail(TG_EINVAL, "queue stats cover spins in [13,24]");
  if (!stats || !ctas) return fail(TG_EINVAL, "stats / ctas must not be NULL");
  tg_anneal_config c{};
  c.spins = spins;
  c.devices = 1;
  c.steps = steps;
  c.procedures = replicas;
  c.entropy_kind = entropy_kind;
  c.t0 = 1.0;
  c.t_min = 1e-3;
  c.renormalize_interval = 1000;
  c.shard_count = 1;
  tg::AnnealParams p = make_params(&c, replicas, 0, 1);
  p.queue_stats = 1;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  char* d = nullptr;
  const size_t stat_bytes = 8 * 24 * static_cast<size_t>(sms);  // hbm_queue.cuh kQStats per CTA
  const size_t bytes = trace_bytes(replicas, steps, false, false) + stat_bytes + 256;
  TG_CUDA(cudaMalloc(&d, bytes));
  char* cur = d;
  p.initial_entropy = carve<double>(cur, replicas);
  p.final_entropy = carve<double>(cur, replicas);
  p.status = carve<int32_t>(cur, replicas);
  p.status_step = carve<int64_t>(cur, replicas);
  p.entropies = carve<double>(cur, replicas * steps);
  p.accepted = carve<uint8_t>(cur, replicas * steps);
  p.trace = carve<int64_t>(cur, 24 * static_cast<size_t>(sms));
  const size_t wsb = workspace_for(p, dev);
  void* ws = nullptr;
  cudaError_t e = cudaMalloc(&ws, wsb);
  if (e == cudaSuccess) e = cudaMemset(p.trace, 0, stat_bytes);
  if (e == cudaSuccess) e = launch(p, ws, wsb, nullptr, /*trace=*/true);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(stats, p.trace, stat_bytes, cudaMemcpyDeviceToHost);
  cudaFree(ws);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "probe_queue_stats");
  *ctas = sms;
  return TG_OK;
}

}  // extern "C"
