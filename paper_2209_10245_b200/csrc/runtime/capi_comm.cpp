// C-ABI: the multi-GPU entry points (include/poas_b200.h "Multi-GPU").
#include <cstring>
#include <string>
#include <vector>

#include "capi_util.hpp"
#include "comm.hpp"
#include "poas/error.hpp"
#include "poas/profiler.hpp"
#include "poas/scheduler.hpp"
#include "poas/sharded.hpp"
#include "poas_b200.h"

using poas_b200::capi::dup_string;
using poas_b200::capi::guard;
using poas_b200::capi::json_escape;
using poas_b200::capi::raise;

namespace {

poas_b200::Comm& need_comm(poas_comm_t c) {
  if (!c || !c->comm) raise(POAS_E_INVALID_ARGUMENT, "comm is NULL");
  return *c->comm;
}

}  // namespace

extern "C" {

int poas_b200_comm_create(const char* name, int rank, int world, int device, poas_comm_t* out) {
  return guard([&] {
    if (!out || !name) raise(POAS_E_INVALID_ARGUMENT, "name / out is NULL");
    auto h = std::make_unique<poas_comm_s>();
    h->comm = std::make_unique<poas_b200::Comm>(name, rank, world, device);
    *out = h.release();
  });
}

void poas_b200_comm_destroy(poas_comm_t comm) { delete comm; }

int poas_b200_comm_barrier(poas_comm_t comm) {
  return guard([&] { need_comm(comm).barrier(); });
}

int poas_b200_comm_allgather(poas_comm_t comm, const char* text, char** json_array) {
  return guard([&] {
    if (!text || !json_array) raise(POAS_E_INVALID_ARGUMENT, "text / out is NULL");
    const std::vector<std::string> all = need_comm(comm).allgather(text);
    std::string o = "[";
    for (std::size_t i = 0; i < all.size(); ++i) o += (i ? ", \"" : "\"") + json_escape(all[i]) + "\"";
    *json_array = dup_string(o + "]");
  });
}

int poas_b200_comm_max(poas_comm_t comm, double value, double* out) {
  return guard([&] {
    if (!out) raise(POAS_E_INVALID_ARGUMENT, "out is NULL");
    *out = need_comm(comm).allreduce_max(value);
  });
}

int poas_b200_nccl_unique_id(unsigned char* id, size_t capacity, size_t* length) {
  return guard([&] {
    if (!id || !length) raise(POAS_E_INVALID_ARGUMENT, "id / length is NULL");
    const std::vector<unsigned char> v = poas_b200::Comm::nccl_unique_id();
    if (capacity < v.size()) raise(POAS_E_INVALID_ARGUMENT, "id buffer too small");
    std::memcpy(id, v.data(), v.size());
    *length = v.size();
  });
}

int poas_b200_comm_init_nccl(poas_comm_t comm, const unsigned char* id, size_t length) {
  return guard([&] {
    if (!id) raise(POAS_E_INVALID_ARGUMENT, "id is NULL");
    need_comm(comm).init_nccl(id, length);
  });
}

int poas_b200_comm_register_b(poas_comm_t comm, const void* b16, const float* b32, int64_t k, int64_t n,
                              int panels) {
  return guard([&] { need_comm(comm).register_b(b16, b32, k, n, panels); });
}

int poas_b200_comm_time_broadcast(poas_comm_t comm, const char* transport, uint64_t bytes, int repetitions,
                                  double* seconds) {
  return guard([&] {
    if (!seconds) raise(POAS_E_INVALID_ARGUMENT, "seconds is NULL");
    *seconds = need_comm(comm).time_broadcast(poas_b200::parse_transport(transport ? transport : ""), bytes,
                                              repetitions);
  });
}

int poas_b200_plan_sharded(const char* const* gpu_profiles, const double* link_bandwidth, int gpus, int64_t m,
                           int64_t n, int64_t k, const char* policy, char** out_json) {
  return guard([&] {
    if (!gpu_profiles || !link_bandwidth || !out_json || gpus < 1)
      raise(POAS_E_INVALID_ARGUMENT, "gpu_profiles / link_bandwidth / out is NULL or gpus < 1");
    std::vector<poas::MachineProfile> profs;
    for (int g = 0; g < gpus; ++g) {
      if (!gpu_profiles[g]) raise(POAS_E_INVALID_ARGUMENT, "gpu profile is NULL");
      profs.push_back(poas::parse_profile(gpu_profiles[g]));
    }
    const std::vector<double> bw(link_bandwidth, link_bandwidth + gpus);
    const poas::ShardedPlan p =
        poas::plan_sharded(profs, bw, poas::MatrixDims{m, n, k}, policy ? policy : "reference");
    std::string o = "{\"level1_profile\": \"" + json_escape(poas::format_profile(p.level1)) +
                    "\", \"level1\": " + poas::format_schedule(p.level1_schedule) + ", \"rows\": [";
    for (std::size_t g = 0; g < p.rows.size(); ++g) o += (g ? ", " : "") + std::to_string(p.rows[g]);
    o += "], \"row0\": [";
    for (std::size_t g = 0; g < p.row0.size(); ++g) o += (g ? ", " : "") + std::to_string(p.row0[g]);
    o += "], \"plans\": [";
    for (std::size_t g = 0; g < p.plans.size(); ++g)
      o += std::string(g ? ", " : "") + (p.plans[g] ? poas::format_schedule(*p.plans[g]) : "null");
    *out_json = dup_string(o + "]}");
  });
}

}  // extern "C"
