// C-ABI entry points for the raw unit kernels (device pointers, caller's
// stream). The plan/profile/execute entry points live in capi.cpp.
#include <cuda_runtime.h>

#include "../kernels/kernels.hpp"
#include "capi_util.hpp"
#include "poas_b200.h"

using poas_b200::AbType;

namespace {

AbType ab_type(int dtype) {
  switch (dtype) {
    case POAS_DTYPE_F32: return AbType::f32;
    case POAS_DTYPE_F16: return AbType::f16;
    case POAS_DTYPE_BF16: return AbType::bf16;
  }
  return AbType::f32;
}

bool valid_dtype(int d) { return d == POAS_DTYPE_F32 || d == POAS_DTYPE_F16 || d == POAS_DTYPE_BF16; }

}  // namespace

extern "C" {

int poas_b200_tc_gemm(int dtype, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda,
                      const void* b, int64_t ldb, float* c, int64_t ldc, int accumulate,
                      int num_ctas, void* stream) {
  return poas_b200::capi::guard([&] {
    if (dtype != POAS_DTYPE_F16 && dtype != POAS_DTYPE_BF16)
      poas_b200::capi::raise(POAS_E_INVALID_ARGUMENT, "tc_gemm: dtype must be f16 or bf16");
    poas_b200::capi::cuda_check(
        poas_b200::tc_gemm(ab_type(dtype), m, n, k, a, lda, b, ldb, c, ldc, accumulate != 0,
                           num_ctas, static_cast<cudaStream_t>(stream)),
        "tc_gemm launch");
  });
}

int poas_b200_tc_gemm_panels(int dtype, int64_t m, int64_t n, int64_t k, const void* a, int64_t lda,
                             const void* b, int64_t ldb, float* c, int64_t ldc, int accumulate,
                             int num_ctas, int panels, const int* flags, int epoch, void* stream) {
  return poas_b200::capi::guard([&] {
    if (dtype != POAS_DTYPE_F16 && dtype != POAS_DTYPE_BF16)
      poas_b200::capi::raise(POAS_E_INVALID_ARGUMENT, "tc_gemm_panels: dtype must be f16 or bf16");
    if (panels < 1 || n % panels != 0 || (panels > 1 && (n / panels) % 256 != 0))
      poas_b200::capi::raise(POAS_E_INVALID_ARGUMENT,
                             "tc_gemm_panels: n must split into panels of a multiple of 256 columns");
    poas_b200::TcPanels ps;
    ps.panels = panels;
    ps.flags = flags;
    ps.epoch = epoch;
    poas_b200::capi::cuda_check(
        poas_b200::tc_gemm_panels(ab_type(dtype), m, n, k, a, lda, b, ldb, c, ldc, accumulate != 0,
                                  num_ctas, ps, static_cast<cudaStream_t>(stream)),
        "tc_gemm_panels launch");
  });
}

int poas_b200_signal_flag(int* flag, int value, void* stream) {
  return poas_b200::capi::guard([&] {
    poas_b200::capi::cuda_check(
        poas_b200::signal_flag(flag, value, static_cast<cudaStream_t>(stream)), "signal_flag");
  });
}

int poas_b200_wait_flag(const int* flag, int value, void* stream) {
  return poas_b200::capi::guard([&] {
    poas_b200::capi::cuda_check(
        poas_b200::wait_flag(flag, value, static_cast<cudaStream_t>(stream)), "wait_flag");
  });
}

const char* poas_b200_tc_kernel_name(int64_t m, int64_t n, int64_t k) {
  return poas_b200::tc_gemm_kernel_name(m, n, k);
}

const char* poas_b200_tc_scheduler_name(int64_t m, int64_t n, int64_t k) {
  return poas_b200::tc_gemm_scheduler_name(m, n, k);
}

int poas_b200_simt_gemm(int64_t m, int64_t n, int64_t k, const float* a, int64_t lda,
                        const float* b, int64_t ldb, float* c, int64_t ldc, int accumulate,
                        int num_ctas, int exclusive_sm, void* stream) {
  return poas_b200::capi::guard([&] {
    poas_b200::capi::cuda_check(
        poas_b200::simt_gemm(m, n, k, a, lda, b, ldb, c, ldc, accumulate != 0, num_ctas,
                             exclusive_sm != 0, static_cast<cudaStream_t>(stream)),
        "simt_gemm launch");
  });
}

int poas_b200_fill_uniform(int dtype, void* dst, int64_t ld, int64_t rows, int64_t cols,
                           int64_t row0, int64_t col0, int64_t total_cols, uint64_t seed,
                           void* stream) {
  return poas_b200::capi::guard([&] {
    if (!valid_dtype(dtype)) poas_b200::capi::raise(POAS_E_INVALID_ARGUMENT, "bad dtype");
    poas_b200::capi::cuda_check(
        poas_b200::fill_uniform(ab_type(dtype), dst, ld, rows, cols, row0, col0, total_cols,
                                seed, static_cast<cudaStream_t>(stream)),
        "fill_uniform launch");
  });
}

int poas_b200_convert_f32(int dtype, const float* src, int64_t ld_src, void* dst, int64_t ld_dst,
                          int64_t rows, int64_t cols, void* stream) {
  return poas_b200::capi::guard([&] {
    if (dtype != POAS_DTYPE_F16 && dtype != POAS_DTYPE_BF16)
      poas_b200::capi::raise(POAS_E_INVALID_ARGUMENT, "convert: dtype must be f16 or bf16");
    poas_b200::capi::cuda_check(
        poas_b200::convert_f32(ab_type(dtype), src, ld_src, dst, ld_dst, rows, cols,
                               static_cast<cudaStream_t>(stream)),
        "convert launch");
  });
}

int poas_b200_sm_count(void) { return poas_b200::device_sm_count(); }

}  // extern "C"
