// TEST INFRASTRUCTURE ONLY -- never linked into or called by the product.
//
// C entry points over the REFERENCE planner library, compiled from the
// read-only sources under /root/reference/proj/src by oracle/Makefile with
// -Dpoas=poasref (so it can sit in one process next to libpoas_b200.so).
// Output formats are identical to the product's C ABI (include/poas_b200.h)
// so parity tests compare bytes. Only tests/, bench.py's cpu_baseline /
// --impl reference leg and __graft_entry__.smoke() may load it.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "poas/adapter.hpp"
#include "poas/device_model.hpp"
#include "poas/error.hpp"
#include "poas/machine_config.hpp"
#include "poas/optimizer.hpp"
#include "poas/profiler.hpp"
#include "poas/rng.hpp"
#include "poas/scheduler.hpp"
#include "poas/simplex.hpp"
#include "poas/simulator.hpp"
#include "support.hpp"  // reference proj/tests/support.hpp: exact_profile, mach2_config

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const poas::Error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 101;
  }
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

std::string g17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

std::string iv(const poas::Interval& i) { return "[" + g17(i.start) + ", " + g17(i.end) + "]"; }

std::string split_json(const poas::WorkloadSplit& s) {
  std::string o = "{\"makespan\": " + g17(s.makespan) + ", \"lp_objective\": " +
                  g17(s.lp_objective) + ", \"lp_iterations\": " + std::to_string(s.lp_iterations) +
                  ", \"shares\": [";
  for (std::size_t i = 0; i < s.shares.size(); ++i) {
    const poas::DeviceShare& d = s.shares[i];
    o += (i ? ", " : "");
    o += "{\"id\": \"" + d.device_id + "\", \"rows\": " + std::to_string(d.rows) +
         ", \"ops\": " + std::to_string(d.ops) + ", \"fraction\": " + g17(d.fraction) +
         ", \"copy_in\": " + iv(d.timeline.copy_in) + ", \"compute\": " + iv(d.timeline.compute) +
         ", \"copy_out\": " + iv(d.timeline.copy_out) + ", \"finish\": " + g17(d.timeline.finish) +
         "}";
  }
  return o + "]}";
}

std::string tile_plan_json(const poas::TilePlan& p) {
  std::string o = "{\"devices\": [";
  for (std::size_t i = 0; i < p.devices.size(); ++i) {
    const poas::PlannedDevice& d = p.devices[i];
    o += (i ? ", " : "");
    o += "{\"id\": \"" + d.device_id + "\", \"rows\": " + std::to_string(d.rows) +
         ", \"k_prime\": " + std::to_string(d.tiling.k_prime) + ", \"sq\": " + g17(d.tiling.sq) +
         ", \"window_fallback\": " + (d.window_fallback ? "true" : "false") + ", \"tiles\": [";
    for (std::size_t t = 0; t < d.tiling.tiles.size(); ++t) {
      const poas::Tile& x = d.tiling.tiles[t];
      o += (t ? ", " : "");
      o += "[" + std::to_string(x.m) + ", " + std::to_string(x.k) + ", " + std::to_string(x.n) + "]";
    }
    o += "]}";
  }
  return o + "]}";
}

poas::MatrixDims dims(int64_t m, int64_t n, int64_t k) {
  poas::MatrixDims d{m, n, k};
  poas::validate_dims(d);
  return d;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

int ref_plan(const char* profile, int64_t m, int64_t n, int64_t k, char** out) {
  return guarded([&] {
    const poas::MachineProfile mp = poas::parse_profile(profile);
    const poas::MatrixDims d = dims(m, n, k);
    const poas::WorkloadSplit s = poas::solve_split(mp, d);
    *out = dup(poas::format_schedule(poas::build_schedule(poas::build_tile_plan(mp, d, s), mp)));
  });
}

int ref_plan_standalone(const char* profile, const char* id, int64_t m, int64_t n, int64_t k,
                        char** out) {
  return guarded([&] {
    const poas::MachineProfile mp = poas::parse_profile(profile);
    *out = dup(poas::format_schedule(poas::standalone_schedule(mp, id, dims(m, n, k))));
  });
}

int ref_split(const char* profile, int64_t m, int64_t n, int64_t k, char** out) {
  return guarded([&] {
    *out = dup(split_json(poas::solve_split(poas::parse_profile(profile), dims(m, n, k))));
  });
}

int ref_oracle_split(const char* profile, int64_t m, int64_t n, int64_t k, int64_t res,
                     int parallel, char** out) {
  return guarded([&] {
    const poas::MachineProfile mp = poas::parse_profile(profile);
    const poas::MatrixDims d = dims(m, n, k);
    *out = dup(split_json(parallel ? poas::oracle_grid_search(mp, d, res)
                                   : poas::oracle_grid_search_serial(mp, d, res)));
  });
}

int ref_tile_plan(const char* profile, int64_t m, int64_t n, int64_t k, const int64_t* rows,
                  size_t count, char** out) {
  return guarded([&] {
    const poas::MachineProfile mp = poas::parse_profile(profile);
    const poas::MatrixDims d = dims(m, n, k);
    const poas::WorkloadSplit s = poas::evaluate_rows(mp, d, std::vector<int64_t>(rows, rows + count));
    *out = dup(tile_plan_json(poas::build_tile_plan(mp, d, s)));
  });
}

int ref_schedule_roundtrip(const char* text, char** out) {
  return guarded([&] { *out = dup(poas::format_schedule(poas::parse_schedule(text))); });
}

int ref_profile_roundtrip(const char* text, char** out) {
  return guarded([&] { *out = dup(poas::format_profile(poas::parse_profile(text))); });
}

int ref_machine_hash(const char* profile, char out[17]) {
  return guarded([&] {
    const std::string h = poas::machine_hash(poas::parse_profile(profile));
    std::memcpy(out, h.c_str(), 17);
  });
}

int ref_fit_linear(const uint64_t* ops, const double* secs, size_t count, double* slope,
                   double* intercept) {
  return guarded([&] {
    std::vector<poas::ModelSample> s;
    for (size_t i = 0; i < count; ++i) s.push_back({ops[i], secs[i]});
    const poas::LinearModel m = poas::fit_linear(s);
    *slope = m.slope;
    *intercept = m.intercept;
  });
}

int ref_transfer_bytes(const char* profile, const char* id, uint64_t ops, int64_t m, int64_t n,
                       int64_t k, uint64_t* in, uint64_t* out) {
  return guarded([&] {
    const poas::MachineProfile mp = poas::parse_profile(profile);
    const poas::DeviceProfile* d = mp.find(id);
    if (!d) poas::fail(poas::errc::missing_device, "no device");
    const poas::TransferBytes tb = poas::transfer_bytes(*d, ops, dims(m, n, k));
    *in = tb.in;
    *out = tb.out;
  });
}

int ref_simplex(int nv, const double* obj, int neq, const double* eqa, const double* eqb, int nge,
                const double* gea, const double* geb, double* x, double* objective, long* iters) {
  return guarded([&] {
    poas::SimplexProblem p;
    p.num_vars = nv;
    p.objective.assign(obj, obj + nv);
    for (int i = 0; i < neq; ++i) {
      p.eq_a.emplace_back(eqa + (size_t)i * nv, eqa + (size_t)(i + 1) * nv);
      p.eq_b.push_back(eqb[i]);
    }
    for (int i = 0; i < nge; ++i) {
      p.ge_a.emplace_back(gea + (size_t)i * nv, gea + (size_t)(i + 1) * nv);
      p.ge_b.push_back(geb[i]);
    }
    const poas::SimplexSolution s = poas::solve_simplex(p);
    std::memcpy(x, s.x.data(), sizeof(double) * (size_t)nv);
    *objective = s.objective;
    *iters = s.iterations;
  });
}

// profile_machine over the reference's synthetic backends (noise from seed).
int ref_profile_synthetic(const char* machine_cfg, uint64_t seed, char** out) {
  return guarded([&] {
    *out = dup(poas::format_profile(
        poas::profile_machine(poas::parse_machine_config(machine_cfg), seed)));
  });
}

// Every measurement the reference's profile_machine (proj/src/simulator.cpp:
// 53-74) draws from its synthetic backends, in call order: the reference's
// own run_compute_probes / run_bandwidth_probe drive a recording wrapper
// around make_synthetic_backend(dev, seed). JSON: {"bus", "profiling":
// {...}, "devices": [{"id", "kind", "elem_size", "align", "cache_bytes",
// "priority" (-1 = none), "gemm": [[side, seconds], ...], "transfer":
// [[bytes, seconds], ...]}]}. Replaying it through another profiler must
// give ref_profile_synthetic's bytes.
int ref_probe_trace(const char* machine_cfg, uint64_t seed, char** out) {
  class Recording final : public poas::DeviceBackend {
   public:
    explicit Recording(poas::BackendPtr inner) : inner_(std::move(inner)) {}
    double time_gemm(std::int64_t side) override {
      const double t = inner_->time_gemm(side);
      gemm += (gemm.empty() ? "" : ", ") + ("[" + std::to_string(side) + ", " + g17(t) + "]");
      return t;
    }
    double time_transfer(std::uint64_t bytes) override {
      const double t = inner_->time_transfer(bytes);
      transfer += (transfer.empty() ? "" : ", ") + ("[" + std::to_string(bytes) + ", " + g17(t) + "]");
      return t;
    }
    bool has_transfers() const override { return inner_->has_transfers(); }
    std::string gemm, transfer;

   private:
    poas::BackendPtr inner_;
  };
  return guarded([&] {
    const poas::MachineConfig cfg = poas::parse_machine_config(machine_cfg);
    const poas::ProfilingConfig& pc = cfg.profiling;
    std::string js = std::string("{\"bus\": ") + (cfg.bus ? "true" : "false") +
                     ", \"profiling\": {\"probes\": " + std::to_string(pc.probes) +
                     ", \"repetitions\": " + std::to_string(pc.repetitions) +
                     ", \"cpu_min_side\": " + std::to_string(pc.cpu_range.min_side) +
                     ", \"cpu_max_side\": " + std::to_string(pc.cpu_range.max_side) +
                     ", \"accel_min_side\": " + std::to_string(pc.accel_range.min_side) +
                     ", \"accel_max_side\": " + std::to_string(pc.accel_range.max_side) +
                     ", \"bandwidth_payload\": " + std::to_string(pc.bandwidth_payload) +
                     "}, \"devices\": [";
    bool first = true;
    for (const poas::SyntheticDevice& dev : cfg.devices) {
      Recording rec(poas::make_synthetic_backend(dev, seed));
      poas::run_compute_probes(rec, pc.range_for(dev.kind), pc.probes, pc.repetitions);
      if (rec.has_transfers()) poas::run_bandwidth_probe(rec, pc.bandwidth_payload, pc.repetitions);
      js += std::string(first ? "" : ", ") + "{\"id\": \"" + dev.id + "\", \"kind\": \"" +
            poas::kind_name(dev.kind) + "\", \"elem_size\": " + std::to_string(dev.elem_size) +
            ", \"align\": " + std::to_string(dev.align) +
            ", \"cache_bytes\": " + std::to_string(dev.cache_bytes) +
            ", \"priority\": " + std::to_string(dev.priority ? *dev.priority : -1) +
            ", \"gemm\": [" + rec.gemm + "], \"transfer\": [" + rec.transfer + "]}";
      first = false;
    }
    *out = dup(js + "]}");
  });
}

// The reference's evaluate report (format_report_json, proj/src/simulator.cpp:
// 448-490) for a synthetic machine and "name:MxNxK;..." inputs -- the schema
// the B200 CLI's `poas evaluate` report follows.
int ref_evaluate_report(const char* machine_cfg, const char* inputs, int repeats, uint64_t seed,
                        char** out) {
  return guarded([&] {
    const poas::MachineConfig cfg = poas::parse_machine_config(machine_cfg);
    const poas::MachineProfile prof = poas::profile_machine(cfg, seed);
    std::vector<poas::EvalInput> in;
    std::string list(inputs);
    std::size_t at = 0;
    while (at < list.size()) {
      std::size_t end = list.find(';', at);
      if (end == std::string::npos) end = list.size();
      const std::string item = list.substr(at, end - at);
      const std::size_t colon = item.find(':');
      poas::EvalInput e;
      e.name = item.substr(0, colon);
      e.dims = poas::parse_dims(item.substr(colon + 1));
      in.push_back(e);
      at = end + 1;
    }
    poas::EvalOptions opt;
    opt.repeats = repeats;
    opt.seed = seed;
    *out = dup(poas::format_report_json(poas::evaluate_inputs(prof, cfg, in, opt)));
  });
}

// The reference test fixture's exact (noise-free) profile of a machine config.
int ref_exact_profile(const char* machine_cfg, char** out) {
  return guarded([&] {
    *out = dup(poas::format_profile(poas::test::exact_profile(poas::parse_machine_config(machine_cfg))));
  });
}

int ref_machine_config_roundtrip(const char* text, char** out) {
  return guarded([&] { *out = dup(poas::format_machine_config(poas::parse_machine_config(text))); });
}

uint64_t ref_rng_draw(uint64_t master, const char* name, int index, double* unit) {
  poas::Rng r = poas::Rng::for_stream(master, name);
  uint64_t v = 0;
  for (int i = 0; i <= index; ++i) v = r.next_u64();
  if (unit) *unit = double(v >> 11) * 0x1.0p-53;
  return v;
}

// Timed reference planner: `reps` full plans (solve_split -> build_tile_plan
// -> build_schedule -> format_schedule); returns seconds per plan.
int ref_time_plan(const char* profile, int64_t m, int64_t n, int64_t k, int reps, double* sec) {
  return guarded([&] {
    const poas::MachineProfile mp = poas::parse_profile(profile);
    const poas::MatrixDims d = dims(m, n, k);
    const auto t0 = std::chrono::steady_clock::now();
    std::size_t sink = 0;
    for (int r = 0; r < reps; ++r) {
      const poas::WorkloadSplit s = poas::solve_split(mp, d);
      sink += poas::format_schedule(poas::build_schedule(poas::build_tile_plan(mp, d, s), mp)).size();
    }
    const auto t1 = std::chrono::steady_clock::now();
    *sec = std::chrono::duration<double>(t1 - t0).count() / reps + (sink == 0 ? 1e-30 : 0.0);
  });
}

}  // extern "C"
