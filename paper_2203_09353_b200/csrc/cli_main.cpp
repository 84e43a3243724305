// cli_main.cpp — `taskgemm_b200`, the command-line front end of the device path.
//
// Mirrors the reference CLI (tools/taskgemm_main.cpp:132-189): `run` and `verify`
// subcommands, the same flags, TASKGEMM_SEED (overridden by --seed, :35-44), exit codes
// 0 ok / 1 internal error / 2 configuration error (:172-188), and the same output bundle
// (report_io.cpp): report.json (config, total_wall_ns, average_entropy_nats, per_device,
// speedup_vs), trace.csv "procedure,step,entropy_nats,accepted,wall_ns" with %.17g
// doubles, kernels.csv "device,procedure,m,n,k,queue_wait_ns,exec_ns,flops", written
// atomically (temp + rename). The execution mode is the new "device" (one persistent
// kernel per GPU); the reference's CPU scheduler simulations (sequential / batched /
// tasked / cpu-reference, exec.cpp:51-142, bench.cpp:22-131) are out of scope and rejected.
// Only the C ABI is used (include/taskgemm_b200.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/taskgemm_b200.h"

namespace {

namespace fs = std::filesystem;

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string fmt17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

void check(tg_status s) {
  if (s == TG_OK) return;
  if (s == TG_ECONFIG) throw ConfigError(tg_last_error());
  throw std::runtime_error(tg_last_error());
}

void write_file_atomic(const fs::path& path, const std::string& content) {  // report_io.cpp:114-123
  const fs::path tmp = path.string() + ".tmp";
  {
    std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open " + tmp.string() + " for writing");
    out.write(content.data(), static_cast<std::streamsize>(content.size()));
    if (!out) throw std::runtime_error("short write to " + tmp.string());
  }
  fs::rename(tmp, path);
}

struct Options {
  uint32_t spins = 6;
  uint64_t steps = 100, procedures = 1, seed = 0, procedures_per_device = 0, device_slots = 0;
  uint32_t devices = 1;
  std::string mode = "device", device_mode = "shared", entropy = "renyi-2", objective = "max",
              initial_state = "product";
  double t0 = 1.0, t_min = 1e-3;
  bool seed_given = false, kernel_log = false, rho_half = false;
  std::vector<uint64_t> sweep;
  uint64_t repeats = 3;
  std::string baseline, out_dir = ".";
};

uint64_t default_seed() {  // taskgemm_main.cpp:35-44
  if (const char* env = std::getenv("TASKGEMM_SEED")) {
    try {
      size_t pos = 0;
      const uint64_t v = std::stoull(env, &pos);
      if (pos != std::strlen(env)) throw std::invalid_argument("trailing");
      return v;
    } catch (const std::exception&) {
      throw ConfigError("TASKGEMM_SEED is not a valid unsigned integer: " + std::string(env));
    }
  }
  return 0;
}

tg_anneal_config to_config(const Options& o) {
  tg_anneal_config c{};
  c.spins = o.spins;
  c.devices = o.devices;
  c.steps = o.steps;
  c.procedures = o.procedures;
  c.seed = o.seed;
  if (o.entropy == "renyi-2") c.entropy_kind = TG_RENYI2;
  else if (o.entropy == "von-neumann") c.entropy_kind = TG_VON_NEUMANN;
  else throw ConfigError("unknown value for --entropy: " + o.entropy);
  if (o.objective == "max") c.objective = TG_MAXIMIZE;
  else if (o.objective == "min") c.objective = TG_MINIMIZE;
  else throw ConfigError("unknown value for --objective: " + o.objective);
  if (o.initial_state == "product") c.initial_state = TG_PRODUCT;
  else if (o.initial_state == "random") c.initial_state = TG_RANDOM;
  else throw ConfigError("unknown value for --initial-state: " + o.initial_state);
  if (o.device_mode != "shared" && o.device_mode != "exclusive")
    throw ConfigError("unknown value for --device-mode: " + o.device_mode);
  if (o.mode != "device") {
    if (o.mode == "sequential" || o.mode == "batched" || o.mode == "tasked" || o.mode == "cpu-reference")
      throw ConfigError("--mode " + o.mode +
                        " is the reference's CPU scheduler simulation (not part of the device "
                        "build); use --mode device");
    throw ConfigError("unknown value for --mode: " + o.mode);
  }
  c.t0 = o.t0;
  c.t_min = o.t_min;
  c.renormalize_interval = 1000;  // McConfig default (spinmc.hpp:120)
  c.rho_half = o.rho_half ? 1 : 0;  // device-only option (no reference counterpart)
  c.shard_index = 0;
  c.shard_count = 1;
  return c;
}

struct Run {
  std::vector<double> init, ent, fin;
  std::vector<uint8_t> acc, sites;
  std::vector<int64_t> wall;
  tg_anneal_result res{};
};

Run run_once(const Options& o, const tg_anneal_config& c) {
  Run r;
  r.init.resize(o.procedures);
  r.fin.resize(o.procedures);
  r.ent.resize(o.procedures * o.steps);
  r.acc.resize(o.procedures * o.steps);
  r.sites.resize(o.procedures * o.steps);
  r.wall.resize(o.procedures * o.steps);
  r.res.initial_entropy = r.init.data();
  r.res.entropies = r.ent.data();
  r.res.accepted = r.acc.data();
  r.res.sites = r.sites.data();
  r.res.wall_ns = r.wall.data();
  r.res.final_entropy = r.fin.data();
  std::vector<int> gpus(o.devices);
  for (uint32_t i = 0; i < o.devices; ++i) gpus[i] = static_cast<int>(i);
  tg_ctx* ctx = nullptr;
  check(tg_create(gpus.data(), static_cast<int>(o.devices), &ctx));
  const tg_status st = tg_anneal_run(ctx, &c, &r.res);
  tg_destroy(ctx);
  check(st);
  return r;
}

std::string config_json(const Options& o, int indent) {  // report_io.cpp:31-46
  const std::string p(indent, ' ');
  std::ostringstream j;
  j << "{\n"
    << p << "  \"spins\": " << o.spins << ",\n"
    << p << "  \"steps\": " << o.steps << ",\n"
    << p << "  \"procedures\": " << o.procedures << ",\n"
    << p << "  \"devices\": " << o.devices << ",\n"
    << p << "  \"procedures_per_device\": "
    << (o.procedures_per_device ? o.procedures_per_device : (o.procedures + o.devices - 1) / o.devices)
    << ",\n"
    << p << "  \"mode\": \"" << o.mode << "\",\n"
    << p << "  \"device_mode\": \"" << o.device_mode << "\",\n"
    << p << "  \"device_slots\": " << o.device_slots << ",\n"
    << p << "  \"entropy\": \"" << o.entropy << "\",\n"
    << p << "  \"objective\": \"" << o.objective << "\",\n"
    << p << "  \"t0\": " << fmt17(o.t0) << ",\n"
    << p << "  \"t_min\": " << fmt17(o.t_min) << ",\n"
    << p << "  \"initial_state\": \"" << o.initial_state << "\",\n"
    << p << "  \"seed\": " << o.seed << "\n"
    << p << "}";
  return j.str();
}

// per_device (report_io.cpp:75-95): one entry per GPU; the persistent kernel is the device's
// single job, so busy = makespan = kernel time and high-water concurrency = its replicas.
std::string devices_json(const Options& o, const Run& r, int indent) {
  const std::string p(indent, ' ');
  const uint64_t da = uint64_t{1} << (o.spins / 2), db = uint64_t{1} << (o.spins - o.spins / 2);
  const uint64_t gflops = 8 * da * da * db;
  std::ostringstream j;
  j << "[";
  for (uint32_t d = 0; d < o.devices; ++d) {
    std::vector<uint64_t> procs;
    for (uint64_t q = d; q < o.procedures; q += o.devices) procs.push_back(q);
    const uint64_t kernels = procs.size() * (o.steps + 1);
    const double ns = std::max(1.0, r.res.kernel_ms * 1e6);
    std::vector<double> per;
    for (uint64_t q : procs)
      for (uint64_t s = 0; s < o.steps; ++s) {
        const int64_t w = r.wall[q * o.steps + s];
        if (w > 0) per.push_back(static_cast<double>(gflops) / (static_cast<double>(w) * 1e-9));
      }
    std::sort(per.begin(), per.end());
    const double med = per.empty() ? 0.0
                       : per.size() % 2 ? per[per.size() / 2]
                                        : 0.5 * (per[per.size() / 2 - 1] + per[per.size() / 2]);
    j << (d ? "," : "") << "\n" << p << "  {\n";
    j << p << "    \"device_id\": " << d << ",\n" << p << "    \"procedures\": [";
    for (size_t i = 0; i < procs.size(); ++i) j << (i ? ", " : "") << procs[i];
    j << "],\n"
      << p << "    \"kernel_count\": " << kernels << ",\n"
      << p << "    \"total_flops\": " << kernels * gflops << ",\n"
      << p << "    \"total_throughput_flops_per_s\": " << fmt17(kernels * gflops / (ns * 1e-9)) << ",\n"
      << p << "    \"high_water_concurrency\": " << procs.size() << ",\n"
      << p << "    \"busy_ns\": " << static_cast<int64_t>(ns) << ",\n"
      << p << "    \"idle_ns\": 0,\n"
      << p << "    \"makespan_ns\": " << static_cast<int64_t>(ns) << ",\n"
      << p << "    \"per_gemm_throughput_median\": " << fmt17(med) << ",\n"
      << p << "    \"per_gemm_latency_throughput_median\": " << fmt17(med) << "\n"
      << p << "  }";
  }
  j << "\n" << p << "]";
  return j.str();
}

std::string trace_csv(const Options& o, const Run& r) {  // report_io.cpp:143-160
  std::string out = "procedure,step,entropy_nats,accepted,wall_ns\n";
  for (uint64_t q = 0; q < o.procedures; ++q)
    for (uint64_t s = 0; s < o.steps; ++s) {
      const uint64_t i = q * o.steps + s;
      out += std::to_string(q) + ',' + std::to_string(s) + ',' + fmt17(r.ent[i]) + ',' +
             (r.acc[i] ? '1' : '0') + ',' + std::to_string(r.wall[i]) + '\n';
    }
  return out;
}

std::string kernel_csv(const Options& o, const Run& r) {  // report_io.cpp:162-185
  const uint64_t da = uint64_t{1} << (o.spins / 2), db = uint64_t{1} << (o.spins - o.spins / 2);
  std::string out = "device,procedure,m,n,k,queue_wait_ns,exec_ns,flops\n";
  for (uint64_t q = 0; q < o.procedures; ++q)
    for (uint64_t s = 0; s < o.steps; ++s)
      out += std::to_string(q % o.devices) + ',' + std::to_string(q) + ',' + std::to_string(da) + ',' +
             std::to_string(da) + ',' + std::to_string(db) + ",0," +
             std::to_string(r.wall[q * o.steps + s]) + ',' + std::to_string(8 * da * da * db) + '\n';
  return out;
}

// Minimal reader for our own report.json (and the reference's: same keys).
std::string json_field(const std::string& text, const std::string& key) {
  const auto k = text.find("\"" + key + "\"");
  if (k == std::string::npos) throw ConfigError("baseline report is missing fields: " + key);
  auto v = text.find(':', k) + 1;
  while (v < text.size() && (text[v] == ' ' || text[v] == '"')) ++v;
  auto e = v;
  while (e < text.size() && text[e] != ',' && text[e] != '\n' && text[e] != '"' && text[e] != '}') ++e;
  return text.substr(v, e - v);
}

int do_run(Options& o) {
  if (!o.seed_given) o.seed = default_seed();
  tg_anneal_config c = to_config(o);
  check(tg_validate(&c));
  const fs::path out_dir(o.out_dir);
  fs::create_directories(out_dir);
  if (!o.sweep.empty()) {  // bench.cpp:457-486 / taskgemm_main.cpp:71-94, mode "device" only
    std::ostringstream j;
    j << "{\n  \"config\": " << config_json(o, 2) << ",\n  \"sweep\": [";
    Run largest;
    uint64_t largest_np = 0;
    Options lo = o;
    for (size_t i = 0; i < o.sweep.size(); ++i) {
      Options oi = o;
      oi.procedures = o.sweep[i];
      tg_anneal_config ci = to_config(oi);
      check(tg_validate(&ci));
      std::vector<std::pair<int64_t, Run>> runs;
      for (uint64_t rep = 0; rep < std::max<uint64_t>(1, o.repeats); ++rep) {
        Run r = run_once(oi, ci);
        runs.emplace_back(r.res.total_wall_ns, std::move(r));
      }
      std::sort(runs.begin(), runs.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      Run& med = runs[runs.size() / 2].second;
      j << (i ? "," : "") << "\n    {\n      \"config\": " << config_json(oi, 6)
        << ",\n      \"total_wall_ns\": " << med.res.total_wall_ns
        << ",\n      \"average_entropy_nats\": " << fmt17(med.res.average_entropy)
        << ",\n      \"per_device\": " << devices_json(oi, med, 6)
        << ",\n      \"speedup_vs\": null,\n      \"procedures\": " << oi.procedures
        << ",\n      \"mode\": \"device\",\n      \"speedup_vs_sequential\": 1\n    }";
      std::printf("  N_p=%-4llu device        total_wall=%.6fs\n",
                  static_cast<unsigned long long>(oi.procedures), med.res.total_wall_ns * 1e-9);
      if (oi.procedures >= largest_np) {
        largest_np = oi.procedures;
        largest = std::move(med);
        lo = oi;
      }
    }
    j << "\n  ]\n}\n";
    write_file_atomic(out_dir / "report.json", j.str());
    write_file_atomic(out_dir / "trace.csv", trace_csv(lo, largest));
    if (o.kernel_log) write_file_atomic(out_dir / "kernels.csv", kernel_csv(lo, largest));
    std::printf("sweep: %zu cells -> %s\n", o.sweep.size(), (out_dir / "report.json").c_str());
    return 0;
  }
  Run r = run_once(o, c);
  std::string speedup = "null";
  if (!o.baseline.empty()) {  // bench.cpp:440-455 same-workload check
    std::ifstream in(o.baseline);
    if (!in) throw ConfigError("cannot open baseline report: " + o.baseline);
    std::stringstream ss;
    ss << in.rdbuf();
    const std::string text = ss.str();
    const bool same = std::stoull(json_field(text, "spins")) == o.spins &&
                      std::stoull(json_field(text, "steps")) == o.steps &&
                      std::stoull(json_field(text, "procedures")) == o.procedures &&
                      json_field(text, "entropy") == o.entropy &&
                      json_field(text, "objective") == o.objective &&
                      std::stod(json_field(text, "t0")) == o.t0 &&
                      std::stod(json_field(text, "t_min")) == o.t_min &&
                      json_field(text, "initial_state") == o.initial_state &&
                      std::stoull(json_field(text, "seed")) == o.seed;
    if (!same)
      throw std::invalid_argument("speedup: reports describe different workloads (only execution mode "
                                  "and resources may differ)");
    const double base_ns = std::stod(json_field(text, "total_wall_ns"));
    speedup = "{\n    \"baseline\": \"" + o.baseline + "\",\n    \"value\": " +
              fmt17(base_ns / static_cast<double>(r.res.total_wall_ns)) + "\n  }";
  }
  std::ostringstream j;
  j << "{\n  \"config\": " << config_json(o, 2) << ",\n  \"total_wall_ns\": " << r.res.total_wall_ns
    << ",\n  \"average_entropy_nats\": " << fmt17(r.res.average_entropy)
    << ",\n  \"per_device\": " << devices_json(o, r, 2) << ",\n  \"speedup_vs\": " << speedup << "\n}\n";
  write_file_atomic(out_dir / "report.json", j.str());
  write_file_atomic(out_dir / "trace.csv", trace_csv(o, r));
  if (o.kernel_log) write_file_atomic(out_dir / "kernels.csv", kernel_csv(o, r));
  std::printf("total_wall=%.6fs average_entropy=%.12f nats -> %s\n", r.res.total_wall_ns * 1e-9,
              r.res.average_entropy, (out_dir / "report.json").c_str());
  return 0;
}

// ------------------------------------------------------------------------------ verify
// The reference's suites (verify.cpp:33-162) restated for the device path: the checks run
// the device, the host arithmetic here is the independent comparison.
using cplx = std::complex<double>;

bool suite_gemm(uint64_t seed, std::string& detail) {  // verify.cpp:33-70
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> nd;
  tg_ctx* ctx = nullptr;
  check(tg_create(nullptr, 1, &ctx));
  double worst = 0.0;
  for (int t = 0; t < 60; ++t) {
    const int m = 1 + static_cast<int>(rng() % 24), n = 1 + static_cast<int>(rng() % 24),
              k = 1 + static_cast<int>(rng() % 24);
    std::vector<cplx> a(m * k), b(k * n), c(m * n), out(m * n);
    for (auto* v : {&a, &b, &c})
      for (auto& x : *v) x = cplx(nd(rng), nd(rng));
    const cplx al(nd(rng), nd(rng)), be(nd(rng), nd(rng));
    const double alv[2] = {al.real(), al.imag()}, bev[2] = {be.real(), be.imag()};
    const double* A = reinterpret_cast<double*>(a.data());
    const double* B = reinterpret_cast<double*>(b.data());
    const double* C = reinterpret_cast<double*>(c.data());
    double* O = reinterpret_cast<double*>(out.data());
    check(tg_zgemm_batched(ctx, 0, 1, m, n, k, alv, &A, &B, bev, &C, &O, nullptr, nullptr));
    double err = 0.0, mx = 0.0;
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) {
        cplx s = 0.0;
        for (int q = 0; q < k; ++q) s += a[i + q * m] * b[q + j * k];
        const cplx want = al * s + be * c[i + j * m];
        err = std::max(err, std::abs(out[i + j * m] - want));
        mx = std::max(mx, std::abs(want));
      }
    worst = std::max(worst, err / mx);
  }
  tg_destroy(ctx);
  detail = "60 random GEMMs (m,n,k <= 24), max relative error " + fmt17(worst);
  return worst <= 1e-13;
}

// Host check values for `verify entropy` (the reference's oracle.cpp:31-44 partial trace,
// then cyclic Jacobi for the spectrum): independent of the device's rho and eigen-solver.
std::vector<double> host_spectrum(const std::vector<cplx>& psi, uint32_t spins) {
  const size_t n = size_t{1} << spins, da = size_t{1} << (spins / 2), db = n / da;
  std::vector<cplx> w(da * da);
  for (size_t a1 = 0; a1 < da; ++a1)
    for (size_t a2 = 0; a2 < da; ++a2) {
      cplx s = 0.0;
      for (size_t b = 0; b < db; ++b) s += psi[a1 + b * da] * std::conj(psi[a2 + b * da]);
      w[a1 + a2 * da] = s;
    }
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (size_t p = 0; p < da; ++p)
      for (size_t q = 0; q < da; ++q)
        if (p != q) off += std::norm(w[p + q * da]);
    if (off < 1e-30) break;
    for (size_t p = 0; p + 1 < da; ++p)
      for (size_t q = p + 1; q < da; ++q) {
        const cplx b = w[p + q * da];
        const double ab = std::abs(b);
        if (ab == 0.0) continue;
        const cplx ph = b / ab;
        const double app = w[p + p * da].real(), aqq = w[q + q * da].real();
        const double tau = (aqq - app) / (2.0 * ab);
        const double t = (tau >= 0 ? 1.0 : -1.0) / (std::abs(tau) + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = t * c;
        for (size_t i = 0; i < da; ++i) {  // columns p, q: W G
          const cplx wp = w[i + p * da], wq = w[i + q * da];
          w[i + p * da] = c * ph * wp - sn * wq;
          w[i + q * da] = sn * ph * wp + c * wq;
        }
        for (size_t j = 0; j < da; ++j) {  // rows p, q: G^H (W G)
          const cplx wp = w[p + j * da], wq = w[q + j * da];
          w[p + j * da] = c * std::conj(ph) * wp - sn * wq;
          w[q + j * da] = sn * std::conj(ph) * wp + c * wq;
        }
      }
  }
  std::vector<double> lam(da);
  for (size_t i = 0; i < da; ++i) lam[i] = w[i + i * da].real();
  std::sort(lam.begin(), lam.end());
  return lam;
}

double device_entropy(const std::vector<cplx>& psi, uint32_t spins, int32_t kind) {
  double got = 0.0, norm = 0.0;
  check(tg_probe_entropy_kind(spins, 1, reinterpret_cast<const double*>(psi.data()), kind, &got, &norm));
  return got;
}

// verify.cpp:72-114: device von Neumann of random states vs a host partial trace, the
// product state (0) and GHZ(5) (ln 2, both kinds), on the rho path the anneal kernels use.
bool suite_entropy(uint64_t seed, std::string& detail) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> nd;
  double worst = 0.0;
  for (uint32_t spins : {2u, 4u, 6u, 8u}) {
    for (int trial = 0; trial < 8; ++trial) {
      const size_t n = size_t{1} << spins;
      std::vector<cplx> psi(n);
      double nrm = 0.0;
      for (auto& x : psi) {
        x = cplx(nd(rng), nd(rng));
        nrm += std::norm(x);
      }
      for (auto& x : psi) x /= std::sqrt(nrm);
      double want = 0.0;
      for (double l : host_spectrum(psi, spins))
        if (l > 1e-15) want -= l * std::log(l);
      worst = std::max(worst, std::abs(device_entropy(psi, spins, TG_VON_NEUMANN) - std::max(want, 0.0)));
    }
  }
  if (worst > 1e-9) {
    detail = "von Neumann entropy deviates from partial-trace oracle by " + fmt17(worst);
    return false;
  }
  std::vector<cplx> prod(64, 0.0);
  prod[0] = 1.0;
  const double pe = device_entropy(prod, 6, TG_VON_NEUMANN);
  if (std::abs(pe) > 1e-10) {
    detail = "product state entropy " + fmt17(pe) + " (expected 0)";
    return false;
  }
  std::vector<cplx> ghz(32, 0.0);
  ghz[0] = ghz[31] = 1.0 / std::sqrt(2.0);
  for (int32_t kind : {TG_VON_NEUMANN, TG_RENYI2}) {
    const double g = device_entropy(ghz, 5, kind);
    if (std::abs(g - std::log(2.0)) > 1e-10) {
      detail = "GHZ entropy " + fmt17(g) + " (expected ln 2)";
      return false;
    }
  }
  detail = "oracle agreement within " + fmt17(worst);
  return true;
}

bool suite_cross(uint64_t seed, std::string& detail) {  // verify.cpp:116-162
  tg_anneal_config c{};
  c.spins = 6;
  c.devices = 1;
  c.steps = 40;
  c.procedures = 4;
  c.seed = seed;
  c.entropy_kind = TG_VON_NEUMANN;  // verify.cpp:126
  c.t0 = 1.0;
  c.t_min = 1e-3;
  c.renormalize_interval = 1000;
  c.shard_count = 1;
  auto go = [&](const tg_anneal_config& cc, std::vector<double>& ent) {
    const uint64_t rows = tg_anneal_rows(&cc);
    std::vector<double> init(rows);
    std::vector<uint8_t> acc(rows * cc.steps);
    ent.assign(rows * cc.steps, 0.0);
    tg_anneal_result r{};
    r.initial_entropy = init.data();
    r.entropies = ent.data();
    r.accepted = acc.data();
    tg_ctx* ctx = nullptr;
    check(tg_create(nullptr, 1, &ctx));
    const tg_status st = tg_anneal_run(ctx, &cc, &r);
    tg_destroy(ctx);
    check(st);
  };
  std::vector<double> a, b, s1;
  go(c, a);
  go(c, b);
  c.shard_index = 1;
  c.shard_count = 2;
  go(c, s1);
  bool ok = a == b;
  for (size_t r = 0; r < 2; ++r)
    for (size_t s = 0; s < c.steps; ++s) ok = ok && s1[r * c.steps + s] == a[(1 + 2 * r) * c.steps + s];
  detail = "S=6, 40 steps, 4 procedures: rerun and shard {1,3} of 2 bitwise identical";
  return ok;
}

int do_verify(const std::vector<std::string>& suites, bool seed_given, uint64_t seed, bool fault) {
  if (!seed_given) seed = default_seed();
  if (fault) check(tg_set_perturb_gemm(1));  // taskgemm_main.cpp:119
  std::vector<std::string> names = suites.empty() ? std::vector<std::string>{"gemm", "entropy", "cross-executor"}
                                                  : suites;
  bool all = true;
  for (const auto& name : names) {
    std::string detail;
    bool ok;
    if (name == "gemm") ok = suite_gemm(seed, detail);
    else if (name == "entropy") ok = suite_entropy(seed, detail);
    else if (name == "cross-executor") ok = suite_cross(seed, detail);
    else throw ConfigError("unknown suite: " + name);
    std::printf("%s %s: %s\n", ok ? "PASS" : "FAIL", name.c_str(), detail.c_str());
    all = all && ok;
  }
  return all ? 0 : 1;
}

[[noreturn]] void usage_error(const std::string& msg) { throw ConfigError(msg); }

template <class T>
T parse_num(const std::string& flag, const std::string& v) {
  try {
    size_t pos = 0;
    T out;
    if constexpr (std::is_floating_point_v<T>) out = static_cast<T>(std::stod(v, &pos));
    else out = static_cast<T>(std::stoull(v, &pos));
    if (pos != v.size()) throw std::invalid_argument("trailing");
    if constexpr (!std::is_floating_point_v<T>)
      if (!v.empty() && v[0] == '-') throw std::invalid_argument("negative");
    return out;
  } catch (const std::exception&) {
    usage_error(flag + ": invalid value '" + v + "'");
  }
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) usage_error("a subcommand is required: run | verify");
    const std::string cmd = argv[1];
    std::vector<std::string> args(argv + 2, argv + argc);
    auto value = [&](size_t& i) -> std::string {
      if (i + 1 >= args.size()) usage_error(args[i] + " requires a value");
      return args[++i];
    };
    if (cmd == "run") {
      Options o;
      for (size_t i = 0; i < args.size(); ++i) {
        const std::string& a = args[i];
        if (a == "--spins") o.spins = parse_num<uint32_t>(a, value(i));
        else if (a == "--steps") o.steps = parse_num<uint64_t>(a, value(i));
        else if (a == "--procedures") o.procedures = parse_num<uint64_t>(a, value(i));
        else if (a == "--devices") o.devices = parse_num<uint32_t>(a, value(i));
        else if (a == "--procedures-per-device") o.procedures_per_device = parse_num<uint64_t>(a, value(i));
        else if (a == "--mode") o.mode = value(i);
        else if (a == "--device-mode") o.device_mode = value(i);
        else if (a == "--device-slots") o.device_slots = parse_num<uint64_t>(a, value(i));
        else if (a == "--entropy") o.entropy = value(i);
        else if (a == "--objective") o.objective = value(i);
        else if (a == "--t0") o.t0 = parse_num<double>(a, value(i));
        else if (a == "--t-min") o.t_min = parse_num<double>(a, value(i));
        else if (a == "--initial-state") o.initial_state = value(i);
        else if (a == "--seed") { o.seed = parse_num<uint64_t>(a, value(i)); o.seed_given = true; }
        else if (a == "--sweep-procedures") {
          std::stringstream ss(value(i));
          std::string tok;
          while (std::getline(ss, tok, ',')) o.sweep.push_back(parse_num<uint64_t>("--sweep-procedures", tok));
        } else if (a == "--repeats") o.repeats = parse_num<uint64_t>(a, value(i));
        else if (a == "--baseline") o.baseline = value(i);
        else if (a == "--out") o.out_dir = value(i);
        else if (a == "--kernel-log") o.kernel_log = true;
        else if (a == "--rho-half") o.rho_half = true;
        else if (a == "--help" || a == "-h") {
          std::printf("taskgemm_b200 run [--spins S] [--steps N] [--procedures P] [--devices G] "
                      "[--mode device] [--entropy renyi-2|von-neumann] [--objective max|min] [--t0 T] "
                      "[--t-min T] [--initial-state product|random] [--seed X] "
                      "[--sweep-procedures a,b,..] [--repeats R] [--baseline report.json] "
                      "[--out DIR] [--kernel-log] [--rho-half]\n");
          return 0;
        } else usage_error("unknown option: " + a);
      }
      return do_run(o);
    }
    if (cmd == "verify") {
      std::vector<std::string> suites;
      bool seed_given = false, fault = false;
      uint64_t seed = 0;
      for (size_t i = 0; i < args.size(); ++i) {
        const std::string& a = args[i];
        if (a == "--suite") suites.push_back(value(i));
        else if (a == "--seed") { seed = parse_num<uint64_t>(a, value(i)); seed_given = true; }
        else if (a == "--inject-fault") fault = true;
        else usage_error("unknown option: " + a);
      }
      return do_verify(suites, seed_given, seed, fault);
    }
    usage_error("unknown subcommand: " + cmd);
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "internal error: %s\n", e.what());
    return 1;
  }
}
