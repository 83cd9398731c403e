// TEST HARNESS for the reference-side binding snippets of INTEGRATION.md.
//
// tests/test_integration_snippets.py extracts every "<!-- snippet: NAME -->"
// block of INTEGRATION.md verbatim into snippet_NAME.inc next to a copy of
// this file and compiles it against the REFERENCE sources (oracle/_ref/obj,
// built from /root/reference/proj/src with -Dpoas=poasref, so `poas::` here is
// the reference library) plus libpoas_b200.so. Each snippet runs in a
// function that declares the caller variables it uses, on a host-CPU unit:
//
//   backend  -- the reference profile_machine loop (proj/src/simulator.cpp:
//               53-74) with B200Backend in place of make_synthetic_backend
//   execute  -- a CPU-unit schedule planned by the reference planner,
//               executed through poas_b200_execute (C checked by the test)
//   dynamic  -- poas_b200_run_dynamic on the same executor
//   overlap  -- planner policy "overlap" + executor overlap=1;pipeline=1
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <string>
#include <vector>

#include <unistd.h>

#include "poas/adapter.hpp"
#include "poas/backend.hpp"
#include "poas/device_model.hpp"
#include "poas/error.hpp"
#include "poas/optimizer.hpp"
#include "poas/profiler.hpp"
#include "poas/scheduler.hpp"
#include "poas_b200.h"

#include "snippet_backend.inc"

namespace {

std::string profile_with_backend(const char* spec, const char* id) {
  poas::ProfilingConfig config;
  config.probes = 3;
  config.repetitions = 1;
  config.cpu_range = {96, 192};
  B200Backend backend(spec);
  poas::DeviceProbeData data;
  data.id = id;
  data.kind = poas::DeviceKind::cpu;
  data.elem_size = 4;
  data.samples = poas::run_compute_probes(backend, config.cpu_range, config.probes, config.repetitions);
  if (backend.has_transfers())
    data.bandwidth = poas::run_bandwidth_probe(backend, config.bandwidth_payload, config.repetitions);
  data.cache_bytes = 32ULL << 20;
  return poas::format_profile(poas::fit_machine({data}, true, config));
}

std::string run_execute(const char* units, const poas::MatrixDims& dims, const float* A,
                        const float* B, float* C, const std::string& schedule_text, int repeats) {
#include "snippet_execute.inc"
  return report_json;
}

std::string run_dynamic(poas_executor_t ex, const std::string& profile_text,
                        const poas::MatrixDims& dims, const poas_gemm_io& io, int iterations) {
#include "snippet_dynamic.inc"
  return dynamic_json;
}

void run_overlap(const char* units, const std::string& profile_text, const poas::MatrixDims& dims,
                 const poas_gemm_io& io, int repeats) {
#include "snippet_overlap.inc"
}

// the caller's JSON reader for the snippet: a flat array of strings
std::vector<std::string> parse_string_array(const char* json) {
  std::vector<std::string> out;
  std::string cur;
  bool in = false, esc = false;
  for (const char* p = json; *p; ++p) {
    const char ch = *p;
    if (!in) {
      if (ch == '"') in = true, cur.clear();
      continue;
    }
    if (esc) {
      cur += ch == 'n' ? '\n' : ch;
      esc = false;
    } else if (ch == '\\') {
      esc = true;
    } else if (ch == '"') {
      in = false;
      out.push_back(cur);
    } else {
      cur += ch;
    }
  }
  return out;
}

std::string run_sharded(const char* job_token, int rank, int world, int device, const std::string& profile_text,
                        const poas::MatrixDims& dims) {
#include "snippet_sharded.inc"
  return sharded_json;
}

}  // namespace

// argv: out_dir m n k. Writes profile.txt, schedule.json, report.json,
// dynamic.json, A.bin, B.bin, C.bin, C_ovl.bin for the test to check.
int main(int argc, char** argv) {
  if (argc != 5) return 2;
  const std::string dir = argv[1];
  const poas::MatrixDims dims{std::atoll(argv[2]), std::atoll(argv[3]), std::atoll(argv[4])};
  const char* units = "cpu0=cpu:threads=2";
  auto put = [&](const std::string& name, const void* p, std::size_t bytes) {
    FILE* f = std::fopen((dir + "/" + name).c_str(), "wb");
    if (!f || std::fwrite(p, 1, bytes, f) != bytes) std::exit(3);
    std::fclose(f);
  };
  try {
    const std::string profile_text = profile_with_backend(units, "cpu0");
    put("profile.txt", profile_text.data(), profile_text.size());
    // the reference planner plans for the profiled machine
    const poas::MachineProfile machine = poas::parse_profile(profile_text);
    const poas::WorkloadSplit split = poas::solve_split(machine, dims);
    const std::string schedule_text =
        poas::format_schedule(poas::build_schedule(poas::build_tile_plan(machine, dims, split), machine));
    put("schedule.json", schedule_text.data(), schedule_text.size());

    const std::size_t na = dims.m * dims.k, nb = dims.k * dims.n, nc = dims.m * dims.n;
    std::vector<float> A(na), B(nb), C(nc, -1.0f), C2(nc, -1.0f);
    std::uint64_t s = 12345;
    auto next = [&] {
      s = s * 6364136223846793005ULL + 1442695040888963407ULL;
      return static_cast<float>(static_cast<double>(s >> 40) / 16777216.0 * 2.0 - 1.0);
    };
    for (auto& x : A) x = next();
    for (auto& x : B) x = next();
    put("A.bin", A.data(), na * 4);
    put("B.bin", B.data(), nb * 4);

    const std::string report = run_execute(units, dims, A.data(), B.data(), C.data(), schedule_text, 2);
    put("report.json", report.data(), report.size());
    put("C.bin", C.data(), nc * 4);

    poas_executor_t ex = nullptr;
    if (poas_b200_executor_create(units, &ex) != POAS_OK) return 4;
    poas_gemm_io io{};
    io.m = dims.m; io.n = dims.n; io.k = dims.k;
    io.a_host = A.data(); io.lda_host = dims.k; io.b_host = B.data(); io.ldb_host = dims.n;
    io.c_host = C2.data(); io.ldc_host = dims.n;
    const std::string dyn = run_dynamic(ex, profile_text, dims, io, 2);
    poas_b200_executor_destroy(ex);
    put("dynamic.json", dyn.data(), dyn.size());

    std::fill(C2.begin(), C2.end(), -1.0f);
    run_overlap(units, profile_text, dims, io, 2);
    put("C_ovl.bin", C2.data(), nc * 4);

    // a one-GPU box's profile (tensor + CUDA-core units) for the sharded plan
    const std::string gpu_profile =
        "poas-profile v1\n\nbus true\n\ndevice gpu0.tc\nkind xpu\nslope 7e-16\nintercept 2e-05\n"
        "bandwidth 6500000000000\nelem_size 2\npriority 0\nalign 1\nops_min 1000000\n"
        "ops_max 4398046511104\n\ndevice gpu0.simt\nkind gpu\nslope 3.5e-14\nintercept 2e-05\n"
        "bandwidth 107000000000\nelem_size 4\npriority 1\nops_min 134217728\nops_max 8589934592\n";
    const std::string token = "harness_" + std::to_string(::getpid());
    const std::string sharded = run_sharded(token.c_str(), 0, 1, -1, gpu_profile, dims);
    put("sharded.json", sharded.data(), sharded.size());
  } catch (const std::exception& e) {
    std::cerr << "harness: " << e.what() << "\n";
    return 1;
  }
  std::cout << "ok\n";
  return 0;
}
