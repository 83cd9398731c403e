#include "units.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <sstream>

#include "capi_util.hpp"
#include "host_gemm.hpp"
#include "host_rng.hpp"
#include "poas/error.hpp"

namespace poas_b200 {

using capi::cuda_check;

namespace {

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  std::istringstream in(s);
  while (std::getline(in, cur, sep)) {
    // trim spaces
    const auto b = cur.find_first_not_of(" \t\n");
    const auto e = cur.find_last_not_of(" \t\n");
    if (b == std::string::npos) continue;
    out.push_back(cur.substr(b, e - b + 1));
  }
  return out;
}

long to_long(const std::string& v, const std::string& key) {
  char* end = nullptr;
  const long x = std::strtol(v.c_str(), &end, 10);
  if (v.empty() || *end != '\0')
    poas::fail(poas::errc::invalid_argument, "unit spec: bad integer for '" + key + "': " + v);
  return x;
}

std::int64_t round_up(std::int64_t x, std::int64_t a) { return (x + a - 1) / a * a; }

}  // namespace

UnitSpec parse_unit_spec(const std::string& text) {
  const auto eq = text.find('=');
  if (eq == std::string::npos || eq == 0)
    poas::fail(poas::errc::invalid_argument, "unit spec '" + text + "': expected <id>=<kind>[:k=v]*");
  UnitSpec u;
  u.id = text.substr(0, eq);
  const std::vector<std::string> parts = split(text.substr(eq + 1), ':');
  if (parts.empty()) poas::fail(poas::errc::invalid_argument, "unit spec '" + text + "': no kind");
  const auto kind = poas::kind_from_name(parts[0]);
  if (!kind) poas::fail(poas::errc::invalid_argument, "unit spec '" + text + "': unknown kind");
  u.kind = *kind;
  u.elem = 4;
  for (size_t i = 1; i < parts.size(); ++i) {
    const auto kv = parts[i].find('=');
    if (kv == std::string::npos)
      poas::fail(poas::errc::invalid_argument, "unit spec '" + text + "': bad option " + parts[i]);
    const std::string k = parts[i].substr(0, kv), v = parts[i].substr(kv + 1);
    if (k == "dev") u.device = static_cast<int>(to_long(v, k));
    else if (k == "sms") u.sms = static_cast<int>(to_long(v, k));
    else if (k == "exclusive") u.exclusive = to_long(v, k) != 0;
    else if (k == "threads") u.threads = static_cast<int>(to_long(v, k));
    else if (k == "elem") u.elem = static_cast<std::uint32_t>(to_long(v, k));
    else if (k == "align") u.align = to_long(v, k);
    else if (k == "preroll") u.preroll_ms = static_cast<double>(to_long(v, k));
    else if (k == "dtype") {
      if (v == "bf16") u.dtype = AbType::bf16;
      else if (v == "f16" || v == "fp16") u.dtype = AbType::f16;
      else poas::fail(poas::errc::invalid_argument, "unit spec: dtype must be bf16 or f16");
    } else if (k == "probe") {
      const auto dash = v.find('-');
      if (dash == std::string::npos)
        poas::fail(poas::errc::invalid_argument, "unit spec: probe must be MIN-MAX");
      u.probe_min = to_long(v.substr(0, dash), k);
      u.probe_max = to_long(v.substr(dash + 1), k);
      if (u.probe_min < 1 || u.probe_max < u.probe_min)
        poas::fail(poas::errc::invalid_argument, "unit spec: bad probe range " + v);
    } else if (k == "link") {
      if (v == "pcie") u.link = Link::pcie;
      else if (v == "hbm") u.link = Link::hbm;
      else if (v == "fused") u.link = Link::fused;
      else poas::fail(poas::errc::invalid_argument, "unit spec: link must be pcie, hbm or fused");
    } else {
      poas::fail(poas::errc::invalid_argument, "unit spec '" + text + "': unknown option " + k);
    }
  }
  if (u.kind == poas::DeviceKind::cpu && u.link != Link::pcie) u.link = Link::pcie;
  return u;
}

std::vector<UnitSpec> parse_unit_list(const std::string& text, bool* bus, bool* lend,
                                      bool* overlap, bool* pipeline) {
  std::vector<UnitSpec> out;
  if (bus) *bus = true;
  if (lend) *lend = true;
  if (overlap) *overlap = false;
  if (pipeline) *pipeline = false;
  for (const std::string& item : split(text, ';')) {
    if (item.rfind("bus=", 0) == 0) {
      if (bus) *bus = item.substr(4) != "0" && item.substr(4) != "false";
      continue;
    }
    if (item.rfind("lend=", 0) == 0) {
      if (lend) *lend = item.substr(5) != "0" && item.substr(5) != "false";
      continue;
    }
    if (item.rfind("overlap=", 0) == 0) {
      if (overlap) *overlap = item.substr(8) != "0" && item.substr(8) != "false";
      continue;
    }
    if (item.rfind("pipeline=", 0) == 0) {
      if (pipeline) *pipeline = item.substr(9) != "0" && item.substr(9) != "false";
      continue;
    }
    out.push_back(parse_unit_spec(item));
  }
  if (out.empty()) poas::fail(poas::errc::invalid_argument, "no units in '" + text + "'");
  return out;
}

DeviceBuffer::~DeviceBuffer() {
  if (ptr_) cudaFree(ptr_);
}

void* DeviceBuffer::ensure(std::size_t bytes) {
  if (bytes <= bytes_ && ptr_) return ptr_;
  if (ptr_) cudaFree(ptr_);
  ptr_ = nullptr;
  bytes_ = 0;
  cuda_check(cudaMalloc(&ptr_, bytes), "cudaMalloc");
  bytes_ = bytes;
  return ptr_;
}

PinnedBuffer::~PinnedBuffer() {
  if (ptr_) cudaFreeHost(ptr_);
}

void* PinnedBuffer::ensure(std::size_t bytes) {
  if (bytes <= bytes_ && ptr_) return ptr_;
  if (ptr_) cudaFreeHost(ptr_);
  ptr_ = nullptr;
  bytes_ = 0;
  cuda_check(cudaMallocHost(&ptr_, bytes), "cudaMallocHost");
  bytes_ = bytes;
  return ptr_;
}

DeviceGuard::DeviceGuard(int dev) {
  cudaGetDevice(&prev_);
  if (dev != prev_) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
}

DeviceGuard::~DeviceGuard() { cudaSetDevice(prev_); }

Unit::Unit(UnitSpec spec) : spec_(std::move(spec)) {
  if (on_gpu()) {
    DeviceGuard g(spec_.device);
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    cuda_check(cudaEventCreate(&ev0_), "cudaEventCreate");
    cuda_check(cudaEventCreate(&ev1_), "cudaEventCreate");
  }
}

Unit::~Unit() {
  if (on_gpu()) {
    DeviceGuard g(spec_.device);
    if (stream_) cudaStreamSynchronize(stream_);
    if (ev0_) cudaEventDestroy(ev0_);
    if (ev1_) cudaEventDestroy(ev1_);
    if (stream_) cudaStreamDestroy(stream_);
  }
}

void Unit::gemm(std::int64_t m, std::int64_t n, std::int64_t k, const void* a, std::int64_t lda,
                const void* b, std::int64_t ldb, float* c, std::int64_t ldc, bool accumulate,
                int extra_sms) {
  const int sms = spec_.sms > 0 ? spec_.sms + extra_sms : 0;
  switch (spec_.kind) {
    case poas::DeviceKind::cpu:
      host_gemm(m, n, k, static_cast<const float*>(a), lda, static_cast<const float*>(b), ldb, c,
                ldc, accumulate, spec_.threads);
      return;
    case poas::DeviceKind::gpu:
      cuda_check(simt_gemm(m, n, k, static_cast<const float*>(a), lda,
                           static_cast<const float*>(b), ldb, c, ldc, accumulate, sms,
                           spec_.exclusive, stream_),
                 "simt_gemm");
      return;
    case poas::DeviceKind::xpu:
      cuda_check(tc_gemm(spec_.dtype, m, n, k, a, lda, b, ldb, c, ldc, accumulate, sms, stream_),
                 "tc_gemm");
      return;
  }
}

void Unit::gemm_panels(std::int64_t m, std::int64_t n, std::int64_t k, const void* a,
                       std::int64_t lda, const void* b, std::int64_t ldb, float* c, std::int64_t ldc,
                       int panels, const int* flags, int epoch, int extra_sms) {
  if (spec_.kind != poas::DeviceKind::xpu)
    poas::fail(poas::errc::invalid_argument, "gemm_panels: tensor units only");
  const int sms = spec_.sms > 0 ? spec_.sms + extra_sms : 0;
  TcPanels ps;
  ps.panels = panels;
  ps.flags = flags;
  ps.epoch = epoch;
  cuda_check(tc_gemm_panels(spec_.dtype, m, n, k, a, lda, b, ldb, c, ldc, false, sms, ps, stream_),
             "tc_gemm_panels");
}

void Unit::gemm_stream(std::int64_t m, std::int64_t n, std::int64_t k, const void* a,
                       std::int64_t lda, const void* b, std::int64_t ldb, float* c, std::int64_t ldc,
                       const TcStream& s, int extra_sms) {
  if (spec_.kind != poas::DeviceKind::xpu)
    poas::fail(poas::errc::invalid_argument, "gemm_stream: tensor units only");
  const int sms = spec_.sms > 0 ? spec_.sms + extra_sms : 0;
  cuda_check(tc_gemm_stream(spec_.dtype, m, n, k, a, lda, b, ldb, c, ldc, sms, s, stream_),
             "tc_gemm_stream");
}

double Unit::time_gemm(std::int64_t side) {
  if (side < 1) poas::fail(poas::errc::invalid_argument, "time_gemm: side must be positive");
  if (!on_gpu()) {
    const std::size_t elems = static_cast<std::size_t>(side) * static_cast<std::size_t>(side);
    if (probe_side_ != side) {
      host_a_.resize(elems);
      host_b_.resize(elems);
      host_c_.resize(elems);
      fill_uniform_host(host_a_.data(), side, side, side, 0, 0, side, 0x5eedA);
      fill_uniform_host(host_b_.data(), side, side, side, 0, 0, side, 0x5eedB);
      probe_side_ = side;
      gemm(side, side, side, host_a_.data(), side, host_b_.data(), side, host_c_.data(), side,
           false);  // warm-up: page in, spin up threads
    }
    const auto t0 = std::chrono::steady_clock::now();
    gemm(side, side, side, host_a_.data(), side, host_b_.data(), side, host_c_.data(), side, false);
    const auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
  }

  DeviceGuard g(spec_.device);
  const bool tensor = spec_.kind == poas::DeviceKind::xpu;
  // A tensor unit whose link carries fp32 (elem 4) receives fp32 operands
  // and converts them to 16-bit inside its compute phase (executor.cpp);
  // the probe times exactly that.
  const bool converts = tensor && spec_.elem == 4;
  // 16-bit operands need a 16-byte row pitch for TMA: pad the leading dim.
  const std::int64_t ld = tensor ? round_up(side, 8) : side;
  const std::size_t esz = tensor ? 2 : 4;
  if (probe_side_ != side) {
    const std::size_t bytes = static_cast<std::size_t>(side) * ld * esz;
    void* a = probe_a_.ensure(bytes);
    void* b = probe_b_.ensure(bytes);
    probe_c_.ensure(static_cast<std::size_t>(side) * side * 4);
    const AbType t = tensor ? spec_.dtype : AbType::f32;
    cuda_check(fill_uniform(t, a, ld, side, side, 0, 0, side, 0x5eedA, stream_), "fill");
    cuda_check(fill_uniform(t, b, ld, side, side, 0, 0, side, 0x5eedB, stream_), "fill");
    if (converts) {
      const std::size_t f32 = static_cast<std::size_t>(side) * side * 4;
      cuda_check(fill_uniform(AbType::f32, probe_a32_.ensure(f32), side, side, side, 0, 0, side,
                              0x5eedA, stream_), "fill");
      cuda_check(fill_uniform(AbType::f32, probe_b32_.ensure(f32), side, side, side, 0, 0, side,
                              0x5eedB, stream_), "fill");
    }
    probe_side_ = side;
    gemm(side, side, side, a, ld, b, ld, static_cast<float*>(probe_c_.get()), side, false);
  }
  const auto one = [&] {  // the probed operation: (conversions +) the GEMM
    if (converts) {
      cuda_check(convert_f32(spec_.dtype, static_cast<const float*>(probe_a32_.get()), side,
                             probe_a_.get(), ld, side, side, stream_), "convert");
      cuda_check(convert_f32(spec_.dtype, static_cast<const float*>(probe_b32_.get()), side,
                             probe_b_.get(), ld, side, side, stream_), "convert");
    }
    gemm(side, side, side, probe_a_.get(), ld, probe_b_.get(), ld,
         static_cast<float*>(probe_c_.get()), side, false);
  };
  // Pre-roll ("preroll=<ms>", B200 extension): the timed launch follows
  // back-to-back launches of the same operation worth >= preroll ms, so it
  // runs in the continuous-load regime a co-executed step runs in (under
  // the power cap a launch after an idle gap sees a boost clock the
  // sustained run never gets, profiles/r01_warmup); 0 = one cold launch.
  // In that regime a short GEMM is also timed the way the executor replays
  // back-to-back steps (one event pair around consecutive launches, each
  // launch staged while the previous runs): the mean of `reps` launches
  // spanning >= ~100 us (1 once a launch alone lasts that long).
  int reps = 1;
  if (spec_.preroll_ms > 0.0) {
    // one launch's time: the previous probe, scaled by ops to this side
    double est = 0.0;
    if (last_probe_s_ > 0.0 && last_probe_side_ > 0) {
      const double r = static_cast<double>(side) / static_cast<double>(last_probe_side_);
      est = last_probe_s_ * r * r * r;
    }
    const int pre = std::min(est > 0.0 ? static_cast<int>(spec_.preroll_ms * 1e-3 / est) + 1 : 2, 4096);
    // the pre-roll's own back-to-back launches give this side's launch time
    // (the cubic extrapolation above misses by far for short, latency-bound
    // GEMMs: from a 512^3 probe it puts 2048^3 at ~0.5 ms, ~25x too long,
    // and the probe would time one isolated launch instead of the
    // back-to-back regime the steps run in)
    cuda_check(cudaEventRecord(ev0_, stream_), "cudaEventRecord");
    for (int i = 0; i < pre; ++i) one();
    cuda_check(cudaEventRecord(ev1_, stream_), "cudaEventRecord");
    cuda_check(cudaEventSynchronize(ev1_), "cudaEventSynchronize");
    float pre_ms = 0.f;
    cuda_check(cudaEventElapsedTime(&pre_ms, ev0_, ev1_), "cudaEventElapsedTime");
    const double per = static_cast<double>(pre_ms) * 1e-3 / pre;
    if (per > 0.0) est = per;
    // a pre-roll shorter than asked (an over-estimate above): top it up
    if (est > 0.0 && pre * est < spec_.preroll_ms * 1e-3)
      for (int i = 0, more = std::min(static_cast<int>((spec_.preroll_ms * 1e-3 - pre * est) / est) + 1, 4096);
           i < more; ++i)
        one();
    if (est > 0.0) reps = std::clamp(static_cast<int>(100e-6 / est) + 1, 1, 32);
  }
  float ms = 0.f;
  if (reps > 1 && std::getenv("POAS_PROBE_GRAPH") == nullptr) {
    // A short GEMM is timed as the executor runs a resident plan's steps:
    // consecutive launches replayed as one CUDA graph (host launch cost off
    // the GPU's critical path), >= ~1 ms of them. POAS_PROBE_GRAPH (set)
    // times stream launches instead.
    const int greps = std::clamp(static_cast<int>(reps * 10), 2, 512);
    if (tensor) cuda_check(tc_prepare_stream(stream_), "tc_prepare_stream");
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cuda_check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeRelaxed), "cudaStreamBeginCapture");
    try {
      for (int i = 0; i < greps; ++i) one();
    } catch (...) {
      cudaStreamEndCapture(stream_, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    cuda_check(cudaStreamEndCapture(stream_, &graph), "cudaStreamEndCapture");
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    cuda_check(ie, "cudaGraphInstantiate (probe)");
    cuda_check(cudaGraphLaunch(exec, stream_), "cudaGraphLaunch");  // upload, steady state
    cuda_check(cudaEventRecord(ev0_, stream_), "cudaEventRecord");
    cuda_check(cudaGraphLaunch(exec, stream_), "cudaGraphLaunch");
    cuda_check(cudaEventRecord(ev1_, stream_), "cudaEventRecord");
    const cudaError_t se = cudaEventSynchronize(ev1_);
    cudaGraphExecDestroy(exec);
    cuda_check(se, "cudaEventSynchronize");
    reps = greps;
  } else {
    cuda_check(cudaEventRecord(ev0_, stream_), "cudaEventRecord");
    for (int i = 0; i < reps; ++i) one();
    cuda_check(cudaEventRecord(ev1_, stream_), "cudaEventRecord");
    cuda_check(cudaEventSynchronize(ev1_), "cudaEventSynchronize");
  }
  cuda_check(cudaEventElapsedTime(&ms, ev0_, ev1_), "cudaEventElapsedTime");
  last_probe_s_ = static_cast<double>(ms) * 1e-3 / reps;
  last_probe_side_ = side;
  return last_probe_s_;
}

double Unit::time_transfer(std::uint64_t bytes) {
  if (!on_gpu()) poas::fail(poas::errc::backend_failure, "cpu unit has no link");
  // The operand stream is inside the probed GEMM: a nominal 1 PB/s keeps
  // the model's copy phases (and the LP's bandwidth terms) at ~zero while
  // staying a valid positive bandwidth of the reference profile format.
  if (spec_.link == Link::fused) return static_cast<double>(bytes) / 1e15;
  DeviceGuard g(spec_.device);
  // Buffers first: allocation must stay outside the timed interval.
  if (spec_.link == Link::pcie) {
    // Pinned host -> device over the unit's PCIe link (what execute() copies).
    void* dst = xfer_dev_.ensure(bytes);
    const void* src = xfer_host_.ensure(bytes);
    cuda_check(cudaEventRecord(ev0_, stream_), "cudaEventRecord");
    cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, stream_), "cudaMemcpyAsync");
  } else {
    // Resident operands: the unit's "link" is its own path from HBM into its
    // SMs -- a streaming read on exactly its SM budget. A 2-SM CUDA-core
    // unit sees ~1/70 of what the 146-SM tensor unit sees, which is what
    // makes receiving all of B (the model's copy-in) expensive for it.
    const std::size_t rounded = (bytes + 15) / 16 * 16;
    void* src = xfer_dev2_.ensure(rounded);
    if (spec_.kind == poas::DeviceKind::gpu) {
      // A CUDA-core unit's operand path for the few rows a co-executed share
      // gives it IS its skinny GEMM streaming all of B (each B element feeds
      // only those rows): time exactly that -- 8 rows against a B of `bytes`
      // (16384 columns) -- rather than a bare streaming read, which it
      // outruns (a 4-row share at 32768^3 read B at 0.6x the bare rate).
      const std::int64_t n = 16384;
      const std::int64_t k = std::max<std::int64_t>(1, static_cast<std::int64_t>(rounded / 4 / n));
      const std::int64_t rows = 8;
      float* a = static_cast<float*>(xfer_dev_.ensure(static_cast<std::size_t>(rows * k) * 4 +
                                                      static_cast<std::size_t>(rows * n) * 4));
      float* c = a + rows * k;
      const float* b = static_cast<const float*>(src);
      const int sms = spec_.sms > 0 ? spec_.sms : 0;
      if (xfer_warm_bytes_ != rounded) {  // one untimed pass: clocks, L2 and TLB state
        cuda_check(simt_gemm(rows, n, k, a, k, b, n, c, n, false, sms, spec_.exclusive, stream_), "simt_gemm");
        xfer_warm_bytes_ = rounded;
      }
      cuda_check(cudaEventRecord(ev0_, stream_), "cudaEventRecord");
      cuda_check(simt_gemm(rows, n, k, a, k, b, n, c, n, false, sms, spec_.exclusive, stream_), "simt_gemm");
      cuda_check(cudaEventRecord(ev1_, stream_), "cudaEventRecord");
      cuda_check(cudaEventSynchronize(ev1_), "cudaEventSynchronize");
      float ms = 0.f;
      cuda_check(cudaEventElapsedTime(&ms, ev0_, ev1_), "cudaEventElapsedTime");
      // scaled to exactly `bytes` (B was k * 16384 fp32 elements)
      return static_cast<double>(ms) * 1e-3 * static_cast<double>(bytes) /
             static_cast<double>(k * n * 4);
    }
    float* sink = static_cast<float*>(xfer_dev_.ensure(64));
    cuda_check(cudaEventRecord(ev0_, stream_), "cudaEventRecord");
    cuda_check(stream_read(src, rounded, spec_.sms, sink, stream_), "stream_read");
  }
  cuda_check(cudaEventRecord(ev1_, stream_), "cudaEventRecord");
  cuda_check(cudaEventSynchronize(ev1_), "cudaEventSynchronize");
  float ms = 0.f;
  cuda_check(cudaEventElapsedTime(&ms, ev0_, ev1_), "cudaEventElapsedTime");
  return static_cast<double>(ms) * 1e-3;
}

}  // namespace poas_b200
