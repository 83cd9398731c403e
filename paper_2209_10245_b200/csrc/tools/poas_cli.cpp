// poas -- command-line front end of the B200 POAS path.
//
// Mirrors the reference CLI (proj/tools/poas.cpp:47-262) over real units:
//   poas profile  --units SPEC [--profiling k=v,..] [--bus true|false] --out FILE
//   poas plan     --profile FILE --dims MxNxK --out FILE [--policy reference|best-subset]
//   poas run      --schedule FILE --units SPEC [--repeats N] [--seed S] [--host]
//                 [--out-c FILE]   (C as raw fp32, row-major)
//   poas evaluate --units SPEC [--inputs FILE] [--repeats N] [--seed S]
//                 [--policy P] [--profiling k=v,..] [--adapt N] --out-dir DIR
//   poas adapt    --profile FILE --units SPEC --dims MxNxK [--iterations N]
//                 [--alpha A] [--threshold PCT] [--policy P] [--seed S] [--host]
//                 [--out-profile FILE] [--out FILE]
// Exit codes as the reference: 0 success, 1 domain or usage error (a
// poas::Error), 2 anything else -- CUDA failures included.
// `run` replaces `simulate` (poas.cpp:116-151): it executes the schedule on
// the box (inputs from the seeded counter generator) and writes
// <schedule>.report.json in the simulate report's shape.
#include <cuda_runtime.h>
#include <sys/stat.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../kernels/kernels.hpp"
#include "../planner/json_lite.hpp"
#include "../runtime/capi_util.hpp"
#include "../runtime/host_rng.hpp"
#include "../runtime/units.hpp"
#include "poas/dynamic.hpp"
#include "poas/error.hpp"
#include "poas/executor.hpp"
#include "poas/log.hpp"
#include "poas/policy.hpp"
#include "poas/profiler.hpp"
#include "poas/rng.hpp"
#include "poas/scheduler.hpp"

namespace poas_b200 {
poas::MachineProfile profile_units(const std::vector<std::unique_ptr<Unit>>& units,
                                   const poas::ProfilingConfig& cfg, bool bus);
}

namespace {

using poas::errc;
using poas::fail;
using poas_b200::AbType;
using poas_b200::parse_unit_list;
using poas_b200::Unit;
using poas_b200::UnitSpec;

struct Args {
  std::string cmd;
  std::map<std::string, std::string> kv;
  bool has(const std::string& k) const { return kv.count(k) != 0; }
  std::string get(const std::string& k, const std::string& def = "") const {
    const auto it = kv.find(k);
    return it == kv.end() ? def : it->second;
  }
  std::string need(const std::string& k) const {
    if (!has(k)) fail(errc::invalid_argument, "missing required option --" + k);
    return kv.at(k);
  }
};

Args parse_args(int argc, char** argv) {
  Args a;
  if (argc < 2) fail(errc::invalid_argument, "usage: poas {profile|plan|run|evaluate|adapt} [options]");
  a.cmd = argv[1];
  static const std::map<std::string, bool> flags = {{"host", true}};
  for (int i = 2; i < argc; ++i) {
    std::string s = argv[i];
    if (s.rfind("--", 0) != 0) fail(errc::invalid_argument, "unexpected argument '" + s + "'");
    s = s.substr(2);
    if (flags.count(s)) {
      a.kv[s] = "1";
      continue;
    }
    if (i + 1 >= argc) fail(errc::invalid_argument, "option --" + s + " needs a value");
    a.kv[s] = argv[++i];
  }
  return a;
}

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail(errc::io_failure, "cannot open '" + path + "'");
  std::ostringstream b;
  b << in.rdbuf();
  return b.str();
}

// tmp + rename, as the reference's report writer (poas.cpp:164-179).
void write_atomic(const std::string& path, const std::string& text) {
  const std::string tmp = path + ".tmp";
  {
    std::ofstream out(tmp, std::ios::binary);
    if (!out) fail(errc::io_failure, "cannot open '" + tmp + "' for writing");
    out << text;
    out.flush();
    if (!out) {
      std::remove(tmp.c_str());
      fail(errc::io_failure, "failed writing '" + tmp + "'");
    }
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0) {
    std::remove(tmp.c_str());
    fail(errc::io_failure, "cannot rename '" + tmp + "' to '" + path + "'");
  }
}

poas::ProfilingConfig profiling_from(const std::string& text) {
  poas::ProfilingConfig c;
  std::stringstream in(text);
  std::string item;
  while (std::getline(in, item, ',')) {
    if (item.empty()) continue;
    const auto eq = item.find('=');
    if (eq == std::string::npos) fail(errc::invalid_argument, "profiling: bad item " + item);
    const std::string k = item.substr(0, eq);
    const long long v = std::atoll(item.c_str() + eq + 1);
    if (k == "probes") c.probes = static_cast<int>(v);
    else if (k == "repetitions") c.repetitions = static_cast<int>(v);
    else if (k == "cpu_min_side") c.cpu_range.min_side = v;
    else if (k == "cpu_max_side") c.cpu_range.max_side = v;
    else if (k == "accel_min_side") c.accel_range.min_side = v;
    else if (k == "accel_max_side") c.accel_range.max_side = v;
    else if (k == "bandwidth_payload") c.bandwidth_payload = static_cast<std::uint64_t>(v);
    else fail(errc::invalid_argument, "profiling: unknown key " + k);
  }
  poas::validate_profiling_config(c);
  return c;
}

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Operands of one run: generated in place from the seeded counter stream,
// resident in HBM (default) or in pinned host memory (--host).
struct Operands {
  poas::GemmOperands io;
  std::vector<void*> dev, pinned, heap;
  ~Operands() {
    for (void* p : dev) cudaFree(p);
    for (void* p : pinned) cudaFreeHost(p);
    for (void* p : heap) std::free(p);
  }
};

std::unique_ptr<Operands> make_operands(const poas::MatrixDims& d, std::uint64_t seed, bool host,
                                        bool need_host, bool need_dev, bool need16, AbType t16) {
  auto o = std::make_unique<Operands>();
  const std::uint64_t sa = poas::Rng::for_stream(seed, "A").state();
  const std::uint64_t sb = poas::Rng::for_stream(seed, "B").state();
  poas::GemmOperands& io = o->io;
  io.m = d.m;
  io.n = d.n;
  io.k = d.k;
  io.resident = !host;
  auto dmalloc = [&](std::size_t bytes) {
    void* p = nullptr;
    cuda_ok(cudaMalloc(&p, bytes), "cudaMalloc");
    o->dev.push_back(p);
    return p;
  };
  auto hmalloc = [&](std::size_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) == cudaSuccess) {
      o->pinned.push_back(p);
      return p;
    }
    cudaGetLastError();  // no GPU/driver: a CPU-only run works on pageable memory
    p = std::aligned_alloc(64, (bytes + 63) / 64 * 64);
    if (!p) throw std::bad_alloc();
    o->heap.push_back(p);
    return p;
  };
  const std::size_t mk = static_cast<std::size_t>(d.m) * d.k, kn = static_cast<std::size_t>(d.k) * d.n,
                    mn = static_cast<std::size_t>(d.m) * d.n;
  if (host || need_host) {
    float* a = static_cast<float*>(hmalloc(mk * 4));
    float* b = static_cast<float*>(hmalloc(kn * 4));
    poas_b200::fill_uniform_host(a, d.k, d.m, d.k, 0, 0, d.k, sa);
    poas_b200::fill_uniform_host(b, d.n, d.k, d.n, 0, 0, d.n, sb);
    io.a_host = a;
    io.lda_host = d.k;
    io.b_host = b;
    io.ldb_host = d.n;
    io.c_host = static_cast<float*>(hmalloc(mn * 4));
    io.ldc_host = d.n;
  }
  if (!host && need_dev) {
    float* a = static_cast<float*>(dmalloc(mk * 4));
    float* b = static_cast<float*>(dmalloc(kn * 4));
    cuda_ok(poas_b200::fill_uniform(AbType::f32, a, d.k, d.m, d.k, 0, 0, d.k, sa, nullptr), "fill");
    cuda_ok(poas_b200::fill_uniform(AbType::f32, b, d.n, d.k, d.n, 0, 0, d.n, sb, nullptr), "fill");
    io.a_dev = a;
    io.lda_dev = d.k;
    io.b_dev = b;
    io.ldb_dev = d.n;
    io.c_dev = static_cast<float*>(dmalloc(mn * 4));
    io.ldc_dev = d.n;
    if (need16) {
      const std::int64_t lda = (d.k + 7) / 8 * 8, ldb = (d.n + 7) / 8 * 8;
      void* a16 = dmalloc(static_cast<std::size_t>(d.m) * lda * 2);
      void* b16 = dmalloc(static_cast<std::size_t>(d.k) * ldb * 2);
      cuda_ok(poas_b200::fill_uniform(t16, a16, lda, d.m, d.k, 0, 0, d.k, sa, nullptr), "fill");
      cuda_ok(poas_b200::fill_uniform(t16, b16, ldb, d.k, d.n, 0, 0, d.n, sb, nullptr), "fill");
      io.a16_dev = a16;
      io.lda16_dev = lda;
      io.b16_dev = b16;
      io.ldb16_dev = ldb;
    }
    cuda_ok(cudaDeviceSynchronize(), "fill sync");
  }
  return o;
}

// Operands every unit in `busy` can read.
std::unique_ptr<Operands> operands_for_units(const std::vector<const Unit*>& busy,
                                             const poas::MatrixDims& dims, std::uint64_t seed,
                                             bool host) {
  bool need_host = false, need_dev = false, need16 = false;
  AbType t16 = AbType::bf16;
  for (const Unit* u : busy) {
    if (!u->on_gpu()) need_host = true;
    else need_dev = true;
    if (u->spec().kind == poas::DeviceKind::xpu) {
      need16 = true;
      t16 = u->spec().dtype;
    }
  }
  return make_operands(dims, seed, host, need_host, need_dev, need16, t16);
}

std::unique_ptr<Operands> operands_for(const poas::Executor& ex, const poas::Schedule& s,
                                       std::uint64_t seed, bool host) {
  std::vector<const Unit*> busy;
  for (const poas::ScheduledDevice& d : s.devices) {
    if (d.rows == 0) continue;
    const Unit* u = ex.find(d.id);
    if (!u) fail(errc::missing_device, "no unit '" + d.id + "'");
    busy.push_back(u);
  }
  return operands_for_units(busy, s.dims, seed, host);
}

int cmd_profile(const Args& a) {
  bool bus = true;
  std::vector<std::unique_ptr<Unit>> units;
  for (const UnitSpec& s : parse_unit_list(a.need("units"), &bus)) units.push_back(std::make_unique<Unit>(s));
  if (a.has("bus")) bus = a.get("bus") == "true";
  const poas::MachineProfile m = poas_b200::profile_units(units, profiling_from(a.get("profiling")), bus);
  const std::string out = a.need("out");
  poas::save_profile(out, m);
  std::printf("profiled %zu unit(s), bus %s\n", m.devices.size(), m.bus ? "true" : "false");
  for (const poas::DeviceProfile& d : m.devices) {
    std::printf("%s (%s): slope %.6g s/op (%.1f TFLOP/s), intercept %.3g s", d.id.c_str(),
                poas::kind_name(d.kind), d.compute.slope, 2.0 / d.compute.slope / 1e12,
                d.compute.intercept);
    if (d.uses_bus()) std::printf(", link %.1f GB/s", d.bandwidth / 1e9);
    std::printf("\n");
  }
  std::printf("wrote %s\n", out.c_str());
  return 0;
}

int cmd_plan(const Args& a) {
  const poas::MachineProfile m = poas::load_profile(a.need("profile"));
  const poas::MatrixDims d = poas::parse_dims(a.need("dims"));
  const poas::Schedule s = poas::plan_with_policy(m, d, a.get("policy", "reference"));
  const std::string out = a.need("out");
  poas::save_schedule(out, s);
  std::printf("split:");
  for (std::size_t i = 0; i < s.devices.size(); ++i)
    std::printf("%s %s %.2f%%", i ? "," : "", s.devices[i].id.c_str(),
                100.0 * static_cast<double>(s.devices[i].rows) / static_cast<double>(d.m));
  std::printf("\npredicted makespan: %.9f s\nwrote %s\n", s.makespan, out.c_str());
  return 0;
}

void print_result(const poas::SimulationResult& r) {
  std::printf("%-14s %-9s %14s %14s %9s\n", "device", "phase", "predicted s", "measured s", "err %");
  for (const poas::DeviceOutcome& d : r.devices) {
    const struct {
      const char* n;
      const poas::PhaseError* p;
    } ph[] = {{"copy-in", &d.copy_in}, {"compute", &d.compute}, {"copy-out", &d.copy_out},
              {"finish", &d.finish}};
    for (const auto& x : ph)
      std::printf("%-14s %-9s %14.9f %14.9f %9.2f\n", d.id.c_str(), x.n, x.p->predicted,
                  x.p->measured, x.p->error_pct);
  }
  std::printf("makespan: predicted %.9f s, measured %.9f s, err %.2f%%\n", r.predicted_makespan,
              r.measured_makespan, r.makespan_error_pct);
  std::printf("rmse %%: finish %.2f, compute %.2f, copy %.2f\n", r.rmse_finish, r.rmse_compute,
              r.rmse_copy);
}

int cmd_run(const Args& a) {
  const std::string path = a.need("schedule");
  const poas::Schedule s = poas::load_schedule(path);
  poas::Executor ex(a.need("units"));
  if (s.machine_hash != ex.machine_hash())  // as cmd_simulate, proj/tools/poas.cpp:120-122
    fail(errc::hash_mismatch, "schedule was planned for machine " + s.machine_hash +
                                  ", the units describe " + ex.machine_hash());
  const int repeats = std::atoi(a.get("repeats", "3").c_str());
  const std::uint64_t seed = std::strtoull(a.get("seed", "20261017").c_str(), nullptr, 10);
  auto ops = operands_for(ex, s, seed, a.has("host"));
  ex.run(s, ops->io, 1);  // warm-up
  poas::SimulationResult r = ex.run(s, ops->io, repeats);
  r.seed = seed;
  std::printf("machine %s, seed %llu, repeats %d, %s operands\n", s.machine_hash.c_str(),
              static_cast<unsigned long long>(seed), repeats, a.has("host") ? "host" : "resident");
  print_result(r);
  std::string report = path;
  const auto dot = report.rfind('.');
  if (dot != std::string::npos && report.find('/', dot) == std::string::npos) report.resize(dot);
  report += ".report.json";
  write_atomic(report, poas::format_execution_report(s, r));
  std::printf("%.3f TFLOP/s\nwrote %s\n",
              2.0 * static_cast<double>(s.dims.total_ops()) / r.measured_makespan / 1e12,
              report.c_str());
  if (a.has("out-c")) {
    // C (fp32, row-major m x n) as the units left it: GPU units' rows in
    // device memory for resident runs, host-CPU units' (and every unit's,
    // for --host runs) in host memory; rows contiguous in schedule order
    const poas::MatrixDims& d = s.dims;
    std::vector<float> c(static_cast<std::size_t>(d.m) * static_cast<std::size_t>(d.n));
    const std::vector<std::int64_t> row0 = poas::row_offsets(s);
    for (std::size_t i = 0; i < s.devices.size(); ++i) {
      const std::int64_t r0 = row0[i], rows = s.devices[i].rows;
      if (rows == 0) continue;
      const Unit* u = ex.find(s.devices[i].id);
      float* dst = c.data() + r0 * d.n;
      const std::size_t bytes = static_cast<std::size_t>(rows) * static_cast<std::size_t>(d.n) * 4;
      if (ops->io.resident && u->on_gpu())
        cuda_ok(cudaMemcpy(dst, ops->io.c_dev + r0 * ops->io.ldc_dev, bytes, cudaMemcpyDeviceToHost), "copy C");
      else
        std::memcpy(dst, ops->io.c_host + r0 * ops->io.ldc_host, bytes);
    }
    write_atomic(a.get("out-c"), std::string(reinterpret_cast<const char*>(c.data()), c.size() * 4));
    std::printf("wrote %s\n", a.get("out-c").c_str());
  }
  return 0;
}

// Dynamic scheduling (paper §3.4.2; poas/dynamic.hpp): plan from the
// profile, run, re-fit the unit models from the measured phases, re-plan when
// the makespan error exceeds the threshold; writes the adapted profile and the
// last schedule.
int cmd_adapt(const Args& a) {
  poas::Executor ex(a.need("units"));
  const poas::MachineProfile prior = poas::load_profile(a.need("profile"));
  if (poas::machine_hash(prior) != ex.machine_hash())
    fail(errc::hash_mismatch, "profile describes machine " + poas::machine_hash(prior) +
                                  ", the units describe " + ex.machine_hash());
  const poas::MatrixDims dims = poas::parse_dims(a.need("dims"));
  const int iterations = std::atoi(a.get("iterations", "5").c_str());
  if (iterations < 1) fail(errc::invalid_argument, "--iterations must be >= 1");
  poas::DynamicOptions opt;
  opt.refit.alpha = std::atof(a.get("alpha", "0.5").c_str());
  opt.replan_threshold_pct = std::atof(a.get("threshold", "2").c_str());
  opt.policy = a.get("policy", "reference");
  const std::uint64_t seed = std::strtoull(a.get("seed", "20261017").c_str(), nullptr, 10);
  poas::DynamicScheduler dyn(prior, dims, opt);
  std::vector<const Unit*> all;
  for (const auto& u : ex.units()) all.push_back(u.get());
  auto ops = operands_for_units(all, dims, seed, a.has("host"));
  std::printf("%-5s %-8s %14s %14s %9s  rows\n", "iter", "replan", "predicted s", "measured s",
              "err %");
  bool replanned = false;
  for (int it = 0; it < iterations; ++it) {
    const poas::SimulationResult r = ex.run(dyn.schedule(), ops->io, 1);
    std::printf("%-5d %-8s %14.9f %14.9f %9.2f ", it, replanned ? "yes" : "no",
                r.predicted_makespan, r.measured_makespan, r.makespan_error_pct);
    for (const poas::DeviceOutcome& d : r.devices)
      std::printf(" %s=%lld", d.id.c_str(), static_cast<long long>(d.rows));
    std::printf("\n");
    replanned = dyn.observe(r);
  }
  std::printf("%d re-plan(s) in %d iteration(s)\n", dyn.replans(), iterations);
  if (a.has("out-profile")) {
    poas::save_profile(a.get("out-profile"), dyn.profile());
    std::printf("wrote %s\n", a.get("out-profile").c_str());
  }
  if (dyn.best_observation() >= 0)
    std::printf("fastest measured plan: iteration %d (%.9f s)\n", dyn.best_observation(),
                dyn.best_measured_makespan());
  if (a.has("out")) {
    poas::save_schedule(a.get("out"), dyn.best_schedule());
    std::printf("wrote %s\n", a.get("out").c_str());
  }
  return 0;
}

struct EvalInput {
  std::string name;
  poas::MatrixDims dims;
};

std::vector<EvalInput> load_inputs(const std::string& path) {
  const poas::json::Value j = poas::json::parse(read_file(path), "inputs");
  if (!j.is_array() || j.items.empty()) fail(errc::parse_failure, "inputs: expected a non-empty array");
  std::vector<EvalInput> out;
  for (const poas::json::Value& e : j.items) {
    if (!e.is_object() || e.size() != 4 || !e.get("name") || !e.get("m") || !e.get("n") || !e.get("k"))
      fail(errc::parse_failure, "inputs: each entry needs exactly name/m/n/k");
    if (!e.get("name")->is_string() || !e.get("m")->is_integer() || !e.get("n")->is_integer() ||
        !e.get("k")->is_integer())
      fail(errc::parse_failure, "inputs: name must be a string and m/n/k integers");
    EvalInput in{e.get("name")->s, {e.get("m")->as_int64(), e.get("n")->as_int64(), e.get("k")->as_int64()}};
    poas::validate_dims(in.dims);
    out.push_back(in);
  }
  return out;
}

// %.17g; JSON has no inf/nan: a phase that was not measured (a resident
// run's zero-length copies give e = 100 (0 - p) / 0) is written as null
std::string g(double v) {
  if (!std::isfinite(v)) return "null";
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

// evaluate_inputs over real hardware (reference proj/src/simulator.cpp:213-291):
// co-executed run per input, standalone run per unit (skipped when its
// predicted standalone makespan exceeds --max-standalone seconds), shares,
// speedups, per-device RMSE.
int cmd_evaluate(const Args& a) {
  const std::string units = a.need("units");
  const std::string out_dir = a.need("out-dir");
  const int repeats = std::atoi(a.get("repeats", "3").c_str());
  const std::uint64_t seed = std::strtoull(a.get("seed", "20261017").c_str(), nullptr, 10);
  const double max_alone = std::atof(a.get("max-standalone", "2.0").c_str());
  const std::string policy = a.get("policy", "reference");
  // --adapt N: dynamic scheduling (paper §3.4.2) -- N warm-up executions per
  // input re-fit the models (carried over to the next input) before the
  // measured run; 0 (default) is the reference's static evaluation.
  const int adapt = std::atoi(a.get("adapt", "0").c_str());
  std::vector<EvalInput> inputs;
  if (a.has("inputs")) {
    inputs = load_inputs(a.get("inputs"));
  } else {  // the reference's Table 3 shapes scaled to one B200 (1/4 per side)
    inputs = {{"i1", {7500, 7500, 7504}},   {"i2", {15000, 5000, 8752}},
              {"i3", {32496, 5000, 5000}},  {"i4", {10000, 20000, 5000}},
              {"i5", {10000, 7504, 15000}}, {"i6", {14000, 10000, 10000}}};
  }
  bool bus = true;
  std::vector<std::unique_ptr<Unit>> probe_units;
  for (const UnitSpec& s : parse_unit_list(units, &bus)) probe_units.push_back(std::make_unique<Unit>(s));
  const poas::MachineProfile prof = poas_b200::profile_units(probe_units, profiling_from(a.get("profiling")), bus);
  probe_units.clear();
  poas::Executor ex(units);
  poas::MachineProfile live = prof;  // re-fitted across inputs with --adapt
  std::vector<const Unit*> all_units;
  for (const auto& u : ex.units()) all_units.push_back(u.get());

  // report.json: the reference's evaluate report (format_report_json,
  // proj/src/simulator.cpp:448-490) key for key -- machine_hash, seed,
  // repeats, devices, inputs[{name, dims, tops, predicted/measured makespan,
  // makespan_error_pct, devices[{id, rows, share_pct, finish/compute/copy
  // error, standalone_makespan, speedup}]}], rmse[{id, finish, compute,
  // copy}] -- plus a "b200" object per input and at the top for what only
  // this implementation has (policy, dynamic re-fit, measured TFLOP/s, which
  // standalone runs were measured and which predicted).
  const auto q = [](const std::string& x) { return "\"" + poas_b200::capi::json_escape(x) + "\""; };
  std::string j = "{\n  \"machine_hash\": " + q(ex.machine_hash()) + ",\n  \"seed\": " +
                  std::to_string(seed) + ",\n  \"repeats\": " + std::to_string(repeats) +
                  ",\n  \"devices\": [";
  for (std::size_t i = 0; i < prof.devices.size(); ++i) j += (i ? ", " : "") + q(prof.devices[i].id);
  j += "],\n  \"inputs\": [\n";
  std::string txt = "machine " + ex.machine_hash() + "  seed " + std::to_string(seed) +
                    "  repeats " + std::to_string(repeats) + "  policy " + policy + "\n\n";
  char line[512];
  std::snprintf(line, sizeof line, "%-6s %-22s %8s %12s %12s %8s %10s %8s\n", "input", "dims",
                "TOps", "predicted s", "measured s", "err %", "TFLOP/s", "speedup");
  txt += line;
  std::map<std::string, std::vector<double>> e_fin, e_cp, e_cy;
  for (std::size_t ii = 0; ii < inputs.size(); ++ii) {
    const EvalInput& in = inputs[ii];
    poas::Schedule s = poas::plan_with_policy(live, in.dims, policy);
    auto ops = adapt > 0 ? operands_for_units(all_units, in.dims, seed + ii, false)
                         : operands_for(ex, s, seed + ii, false);
    double static_err = 0.0;
    if (adapt > 0) {
      poas::DynamicOptions o;
      o.policy = policy;
      o.refit.alpha = std::atof(a.get("alpha", "0.5").c_str());
      poas::DynamicScheduler dyn(live, in.dims, o);
      for (int it = 0; it < adapt; ++it) {  // same duty cycle as the measured run
        const poas::SimulationResult w = ex.run(dyn.schedule(), ops->io, repeats);
        if (it == 0) static_err = w.makespan_error_pct;
        dyn.observe(w);
      }
      live = dyn.profile();
      s = dyn.best_schedule();
    } else {
      ex.run(s, ops->io, 1);
    }
    const poas::SimulationResult r = ex.run(s, ops->io, repeats);
    // standalone run of every unit (evaluate_one, simulator.cpp:224-232):
    // measured when its predicted standalone makespan is at most
    // --max-standalone seconds, else its prediction stands in
    std::vector<double> alone(prof.devices.size(), 0.0);
    std::vector<char> alone_measured(prof.devices.size(), 0);
    double best_alone = 0.0;
    for (std::size_t di = 0; di < prof.devices.size(); ++di) {
      const poas::Schedule sa = poas::standalone_schedule(live, prof.devices[di].id, in.dims);
      alone[di] = sa.makespan;
      if (sa.makespan <= max_alone) {
        auto oa = operands_for(ex, sa, seed + ii, false);
        ex.run(sa, oa->io, 1);
        alone[di] = ex.run(sa, oa->io, repeats).measured_makespan;
        alone_measured[di] = 1;
      }
      if (best_alone == 0.0 || alone[di] < best_alone) best_alone = alone[di];
    }
    const double tops = static_cast<double>(in.dims.total_ops()) / 1e12;
    const double speedup = best_alone > 0 ? best_alone / r.measured_makespan : 0.0;
    std::snprintf(line, sizeof line, "%-6s %-22s %8.2f %12.6f %12.6f %8.2f %10.1f %7.3fx\n",
                  in.name.c_str(),
                  (std::to_string(in.dims.m) + "x" + std::to_string(in.dims.n) + "x" +
                   std::to_string(in.dims.k)).c_str(),
                  tops, r.predicted_makespan, r.measured_makespan, r.makespan_error_pct,
                  2 * tops / r.measured_makespan, speedup);
    txt += line;
    j += std::string(ii ? ",\n" : "") + "    {\n      \"name\": " + q(in.name) +
         ",\n      \"dims\": {\"m\": " + std::to_string(in.dims.m) + ", \"n\": " +
         std::to_string(in.dims.n) + ", \"k\": " + std::to_string(in.dims.k) + "},\n      \"tops\": " +
         g(tops) + ",\n      \"predicted_makespan\": " + g(r.predicted_makespan) +
         ",\n      \"measured_makespan\": " + g(r.measured_makespan) +
         ",\n      \"makespan_error_pct\": " + g(r.makespan_error_pct) + ",\n      \"devices\": [";
    std::string measured_ids;
    for (std::size_t di = 0; di < prof.devices.size(); ++di) {
      const std::string& id = prof.devices[di].id;
      const poas::DeviceOutcome* d = nullptr;
      for (const poas::DeviceOutcome& o : r.devices)
        if (o.id == id) d = &o;
      const std::int64_t rows = d ? d->rows : 0;
      j += std::string(di ? ", " : "") + "\n        {\"id\": " + q(id) + ", \"rows\": " +
           std::to_string(rows) + ", \"share_pct\": " +
           g(100.0 * static_cast<double>(rows) / static_cast<double>(in.dims.m)) +
           ", \"finish_error_pct\": " + g(d ? d->finish.error_pct : 0.0) +
           ", \"compute_error_pct\": " + g(d ? d->compute.error_pct : 0.0) +
           ", \"copy_error_pct\": " + g(d ? d->copy.error_pct : 0.0) +
           ", \"standalone_makespan\": " + g(alone[di]) +
           ", \"speedup\": " + g(alone[di] / r.measured_makespan) + "}";
      if (d) {  // the reference's RMSE takes every device of the co-executed run
        for (auto [vec, v] : {std::pair{&e_fin, d->finish.error_pct}, std::pair{&e_cp, d->compute.error_pct},
                              std::pair{&e_cy, d->copy.error_pct}})
          if (std::isfinite(v)) (*vec)[id].push_back(v);  // unmeasured phases (null) left out
      }
      if (alone_measured[di]) measured_ids += (measured_ids.empty() ? "" : ", ") + q(id);
    }
    j += "\n      ],\n      \"b200\": {\"tflops\": " + g(2 * tops / r.measured_makespan) +
         ", \"speedup_vs_best_single\": " + g(speedup) + ", \"standalone_measured\": [" + measured_ids +
         "]" + (adapt > 0 ? ", \"static_plan_error_pct\": " + g(static_err) : std::string()) + "}\n    }";
  }
  j += "\n  ],\n  \"rmse\": [";
  txt += "\nRMSE % across inputs, finish (compute, copy)\n";
  std::size_t idx = 0;
  for (const poas::DeviceProfile& d : prof.devices) {
    auto rms = [](const std::vector<double>& v) {
      double s = 0;
      for (double x : v) s += x * x;
      return v.empty() ? 0.0 : std::sqrt(s / static_cast<double>(v.size()));
    };
    const double f = rms(e_fin[d.id]), c = rms(e_cp[d.id]), y = rms(e_cy[d.id]);
    j += std::string(idx++ ? ", " : "") + "\n    {\"id\": " + q(d.id) + ", \"finish\": " + g(f) +
         ", \"compute\": " + g(c) + ", \"copy\": " + g(y) + "}";
    std::snprintf(line, sizeof line, "%-14s %.2f (%.2f, %.2f)\n", d.id.c_str(), f, c, y);
    txt += line;
  }
  j += "\n  ],\n  \"b200\": {\"policy\": " + q(policy) + ", \"adapt\": " + std::to_string(adapt) +
       ", \"max_standalone_s\": " + g(max_alone) + "}\n}\n";
  mkdir(out_dir.c_str(), 0755);
  write_atomic(out_dir + "/report.json", j);
  write_atomic(out_dir + "/report.txt", txt);
  std::fputs(txt.c_str(), stdout);
  std::printf("wrote %s/report.txt\nwrote %s/report.json\n", out_dir.c_str(), out_dir.c_str());
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (const char* env = std::getenv("POAS_LOG"); env && !poas::parse_log_level(env)) {
    std::fprintf(stderr, "poas: error: POAS_LOG must be quiet, info, or debug (got '%s')\n", env);
    return 1;
  }
  try {
    const Args a = parse_args(argc, argv);
    if (a.cmd == "profile") return cmd_profile(a);
    if (a.cmd == "plan") return cmd_plan(a);
    if (a.cmd == "run") return cmd_run(a);
    if (a.cmd == "evaluate") return cmd_evaluate(a);
    if (a.cmd == "adapt") return cmd_adapt(a);
    fail(errc::invalid_argument,
         "unknown subcommand '" + a.cmd + "' (profile|plan|run|evaluate|adapt)");
  } catch (const poas::Error& e) {
    std::fprintf(stderr, "poas: error: %s\n", e.what());
    return 1;
  } catch (const poas_b200::capi::AbiError& e) {
    // CUDA / internal failures are not domain errors: exit 2 as any other
    // non-poas::Error exception (proj/tools/poas.cpp:251-260)
    std::fprintf(stderr, "poas: internal error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "poas: internal error: %s\n", e.what());
    return 2;
  } catch (...) {
    std::fprintf(stderr, "poas: internal error\n");
    return 2;
  }
  return 2;
}
