#pragma once
#include <cstdint>

namespace poas_b200 {

// Host fp32 GEMM over `threads` OpenMP threads (0 = all online cores).
void host_gemm(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
               int64_t ldb, float* C, int64_t ldc, bool accumulate, int threads);

int host_threads_default();

}  // namespace poas_b200
