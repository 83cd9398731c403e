// Host CPU unit: fp32 GEMM on the box's own cores.
//
//   C[m x n] (=|+=) A[m x k] . B[k x n]      row-major fp32
//
// Replaces the CPU-kind synthetic law (reference proj/src/simulator.cpp:30-34).
// Goto-style blocking: B is packed once per (kc x nc) block into 32-column
// panels shared by all threads; threads split the rows; a 6 x 32 AVX-512
// register tile (12 zmm accumulators) runs the inner product. Hosts without
// AVX-512 take a portable 4 x 16 path the compiler vectorises.
#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

#include "host_gemm.hpp"

namespace poas_b200 {
namespace {

constexpr int64_t kKC = 256;   // k-block: one packed B panel of 256 x 32 floats = 32 KiB (L1/L2)
constexpr int64_t kNC = 2048;  // n-block: packed B block 256 x 2048 x 4 B = 2 MiB (L2/L3)
constexpr int64_t kNR = 32;    // panel width (two zmm)
constexpr int64_t kMR = 6;     // register-tile rows

// Pack B[k0:k0+kc, n0:n0+nc] into panels of kNR columns, zero-padded.
void pack_b(const float* B, int64_t ldb, int64_t k0, int64_t kc, int64_t n0, int64_t nc,
            float* out) {
  const int64_t panels = (nc + kNR - 1) / kNR;
#pragma omp for schedule(static)
  for (int64_t p = 0; p < panels; ++p) {
    float* dst = out + p * kc * kNR;
    const int64_t c0 = n0 + p * kNR;
    const int64_t w = std::min<int64_t>(kNR, n0 + nc - c0);
    for (int64_t kk = 0; kk < kc; ++kk) {
      const float* src = B + (k0 + kk) * ldb + c0;
      float* d = dst + kk * kNR;
      if (w == kNR) {
        std::memcpy(d, src, kNR * sizeof(float));
      } else {
        std::memcpy(d, src, static_cast<size_t>(w) * sizeof(float));
        std::memset(d + w, 0, static_cast<size_t>(kNR - w) * sizeof(float));
      }
    }
  }
}

__attribute__((target("avx512f,fma"))) void micro_avx512(int64_t mr, int64_t nr, int64_t kc,
                                                          const float* A, int64_t lda,
                                                          const float* Bp, float* C, int64_t ldc,
                                                          bool load_c) {
  __m512 acc[kMR][2];
  for (int i = 0; i < kMR; ++i) acc[i][0] = acc[i][1] = _mm512_setzero_ps();
  const float* a[kMR];
  for (int i = 0; i < kMR; ++i) a[i] = A + std::min<int64_t>(i, mr - 1) * lda;
  for (int64_t kk = 0; kk < kc; ++kk) {
    const __m512 b0 = _mm512_loadu_ps(Bp + kk * kNR);
    const __m512 b1 = _mm512_loadu_ps(Bp + kk * kNR + 16);
#pragma GCC unroll 6
    for (int i = 0; i < kMR; ++i) {
      const __m512 av = _mm512_set1_ps(a[i][kk]);
      acc[i][0] = _mm512_fmadd_ps(av, b0, acc[i][0]);
      acc[i][1] = _mm512_fmadd_ps(av, b1, acc[i][1]);
    }
  }
  const __mmask16 m0 = nr >= 16 ? 0xFFFF : static_cast<__mmask16>((1u << nr) - 1);
  const __mmask16 m1 =
      nr >= 32 ? 0xFFFF : (nr <= 16 ? 0 : static_cast<__mmask16>((1u << (nr - 16)) - 1));
  for (int64_t i = 0; i < mr; ++i) {
    float* c = C + i * ldc;
    __m512 v0 = acc[i][0], v1 = acc[i][1];
    if (load_c) {
      v0 = _mm512_add_ps(v0, _mm512_maskz_loadu_ps(m0, c));
      v1 = _mm512_add_ps(v1, _mm512_maskz_loadu_ps(m1, c + 16));
    }
    _mm512_mask_storeu_ps(c, m0, v0);
    _mm512_mask_storeu_ps(c + 16, m1, v1);
  }
}

void micro_portable(int64_t mr, int64_t nr, int64_t kc, const float* A, int64_t lda,
                    const float* Bp, float* C, int64_t ldc, bool load_c) {
  float acc[kMR][kNR] = {};
  for (int64_t kk = 0; kk < kc; ++kk) {
    const float* b = Bp + kk * kNR;
    for (int64_t i = 0; i < mr; ++i) {
      const float av = A[i * lda + kk];
      for (int j = 0; j < kNR; ++j) acc[i][j] += av * b[j];
    }
  }
  for (int64_t i = 0; i < mr; ++i)
    for (int64_t j = 0; j < nr; ++j) C[i * ldc + j] = (load_c ? C[i * ldc + j] : 0.f) + acc[i][j];
}

// Skinny-M path (a co-executed CPU share is often a handful of residue rows):
// no packing -- every B element is streamed from memory exactly once per
// 8-row group. Threads split the columns in 1024-wide strips (one 4 KB page
// of each B row per k, so the walk down B stays page-friendly); a strip
// keeps its 8 x 1024 partial C in an L1-resident buffer.
constexpr int64_t kSkinnyRows = 8;
constexpr int64_t kSkinnyCols = 1024;

__attribute__((target("avx512f,fma"))) void skinny_block_avx512(
    int64_t mr, int64_t c0, int64_t nc, int64_t k, const float* A, int64_t lda, const float* B,
    int64_t ldb, float* C, int64_t ldc, bool accumulate) {
  alignas(64) float acc[kSkinnyRows][kSkinnyCols];
  const int64_t vecs = (nc + 15) / 16;
  const __mmask16 tail =
      nc % 16 == 0 ? static_cast<__mmask16>(0xFFFF) : static_cast<__mmask16>((1u << (nc % 16)) - 1);
  for (int64_t i = 0; i < mr; ++i)
    for (int64_t v = 0; v < vecs; ++v) _mm512_store_ps(&acc[i][16 * v], _mm512_setzero_ps());
  for (int64_t kk = 0; kk < k; ++kk) {
    const float* b = B + kk * ldb + c0;
    __m512 av[kSkinnyRows];
    for (int64_t i = 0; i < mr; ++i) av[i] = _mm512_set1_ps(A[i * lda + kk]);
    for (int64_t v = 0; v < vecs; ++v) {
      const __m512 bv = _mm512_maskz_loadu_ps(v + 1 == vecs ? tail : 0xFFFF, b + 16 * v);
#pragma GCC unroll 8
      for (int64_t i = 0; i < kSkinnyRows; ++i) {
        if (i >= mr) break;
        _mm512_store_ps(&acc[i][16 * v],
                        _mm512_fmadd_ps(av[i], bv, _mm512_load_ps(&acc[i][16 * v])));
      }
    }
  }
  for (int64_t i = 0; i < mr; ++i) {
    float* c = C + i * ldc + c0;
    for (int64_t v = 0; v < vecs; ++v) {
      const __mmask16 mk = v + 1 == vecs ? tail : 0xFFFF;
      __m512 x = _mm512_load_ps(&acc[i][16 * v]);
      if (accumulate) x = _mm512_add_ps(x, _mm512_maskz_loadu_ps(mk, c + 16 * v));
      _mm512_mask_storeu_ps(c + 16 * v, mk, x);
    }
  }
}

bool have_avx512() {
  static const bool yes = __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("fma");
  return yes;
}

}  // namespace

int host_threads_default() { return omp_get_num_procs(); }

void host_gemm(int64_t m, int64_t n, int64_t k, const float* A, int64_t lda, const float* B,
               int64_t ldb, float* C, int64_t ldc, bool accumulate, int threads) {
  if (m <= 0 || n <= 0) return;
  if (k <= 0) {
    if (!accumulate)
      for (int64_t i = 0; i < m; ++i) std::memset(C + i * ldc, 0, static_cast<size_t>(n) * 4);
    return;
  }
  const int nt = threads > 0 ? threads : omp_get_num_procs();
  const bool wide = have_avx512();
  if (wide && m <= 4 * kSkinnyRows) {
    const int64_t groups = (m + kSkinnyRows - 1) / kSkinnyRows;
    const int64_t blocks = (n + kSkinnyCols - 1) / kSkinnyCols;
#pragma omp parallel for num_threads(nt) schedule(static) collapse(2)
    for (int64_t g = 0; g < groups; ++g)
      for (int64_t cb = 0; cb < blocks; ++cb) {
        const int64_t r0 = g * kSkinnyRows;
        const int64_t c0 = cb * kSkinnyCols;
        skinny_block_avx512(std::min(kSkinnyRows, m - r0), c0, std::min(kSkinnyCols, n - c0), k,
                            A + r0 * lda, lda, B, ldb, C + r0 * ldc, ldc, accumulate);
      }
    return;
  }
  const int64_t nc_max = std::min<int64_t>(kNC, (n + kNR - 1) / kNR * kNR);
  std::unique_ptr<float[]> packed(new float[static_cast<size_t>(kKC * nc_max)]);
  float* Bp = packed.get();

#pragma omp parallel num_threads(nt)
  {
    for (int64_t n0 = 0; n0 < n; n0 += kNC) {
      const int64_t nc = std::min(kNC, n - n0);
      for (int64_t k0 = 0; k0 < k; k0 += kKC) {
        const int64_t kc = std::min(kKC, k - k0);
        const bool load_c = accumulate || k0 > 0;
        pack_b(B, ldb, k0, kc, n0, nc, Bp);  // implicit barrier at the end of omp for
        const int64_t row_tiles = (m + kMR - 1) / kMR;
        const int64_t panels = (nc + kNR - 1) / kNR;
#pragma omp for schedule(static) collapse(2)
        for (int64_t rt = 0; rt < row_tiles; ++rt) {
          for (int64_t p = 0; p < panels; ++p) {
            const int64_t i0 = rt * kMR;
            const int64_t mr = std::min(kMR, m - i0);
            const int64_t c0 = p * kNR;
            const int64_t nr = std::min(kNR, nc - c0);
            const float* a = A + i0 * lda + k0;
            float* c = C + i0 * ldc + n0 + c0;
            const float* bp = Bp + p * kc * kNR;
            if (wide)
              micro_avx512(mr, nr, kc, a, lda, bp, c, ldc, load_c);
            else
              micro_portable(mr, nr, kc, a, lda, bp, c, ldc, load_c);
          }
        }
        // implicit barrier: Bp is repacked next iteration
      }
    }
  }
}

}  // namespace poas_b200
