// host_narrow.cpp -- host-side narrowing of int64 neighbour ids to int32 for the
// host-buffer drop-in (gsvr_train_step_backward_host): the caller's (P, K)
// int64 lists (kernels.py:81, `nbr`) are halved before they cross PCIe, with
// the id range check [0, N) folded into the same pass.  Streaming (non-temporal)
// stores into the pinned staging slot: no read-for-ownership of the
// destination, which the copy engine reads right after.
#include <immintrin.h>
#include <omp.h>

#include <cstdint>
#include <cstring>

namespace gsvr {

__attribute__((target("avx2"))) static int narrow_avx2(const int64_t *src, int32_t *dst, int64_t n, int64_t N) {
  const __m256i zero = _mm256_setzero_si256(), top = _mm256_set1_epi64x(N - 1);
  __m256i badv = zero;
  int bad = 0;
  int64_t i = 0;
  for (; i < n && (reinterpret_cast<uintptr_t>(dst + i) & 31); ++i) {  // head up to 32-byte alignment
    const int64_t v = src[i];
    bad |= (uint64_t)v >= (uint64_t)N;
    dst[i] = (int32_t)v;
  }
  for (; i + 8 <= n; i += 8) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 4));
    badv = _mm256_or_si256(badv, _mm256_or_si256(_mm256_cmpgt_epi64(zero, a), _mm256_cmpgt_epi64(a, top)));
    badv = _mm256_or_si256(badv, _mm256_or_si256(_mm256_cmpgt_epi64(zero, b), _mm256_cmpgt_epi64(b, top)));
    // low words: [a0 a1 b0 b1 | a2 a3 b2 b3] -> [a0 a1 a2 a3 b0 b1 b2 b3]
    const __m256 lo = _mm256_shuffle_ps(_mm256_castsi256_ps(a), _mm256_castsi256_ps(b), _MM_SHUFFLE(2, 0, 2, 0));
    const __m256i packed = _mm256_permute4x64_epi64(_mm256_castps_si256(lo), _MM_SHUFFLE(3, 1, 2, 0));
    _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i), packed);
  }
  bad |= !_mm256_testz_si256(badv, badv);
  for (; i < n; ++i) {
    const int64_t v = src[i];
    bad |= (uint64_t)v >= (uint64_t)N;
    dst[i] = (int32_t)v;
  }
  _mm_sfence();
  return bad;
}

static int narrow_scalar(const int64_t *src, int32_t *dst, int64_t n, int64_t N) {
  int bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t v = src[i];
    bad |= (uint64_t)v >= (uint64_t)N;
    dst[i] = (int32_t)v;
  }
  return bad;
}

int narrow_ids_host(const int64_t *src, int32_t *dst, int64_t n, int64_t N, int threads) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  int bad = 0;
#pragma omp parallel num_threads(threads) reduction(| : bad)
  {
    const int nt = omp_get_num_threads(), t = omp_get_thread_num();
    const int64_t per = ((n + nt - 1) / nt + 7) / 8 * 8;  // 8-id (32-byte) aligned pieces
    const int64_t lo = (int64_t)t * per < n ? (int64_t)t * per : n;
    const int64_t hi = lo + per < n ? lo + per : n;
    if (hi > lo) bad |= avx2 ? narrow_avx2(src + lo, dst + lo, hi - lo, N) : narrow_scalar(src + lo, dst + lo, hi - lo, N);
  }
  return bad;
}

// streaming copy: 32-byte non-temporal stores once the destination is aligned
// (no read-for-ownership of the destination lines: one third less memory traffic)
__attribute__((target("avx2"))) static void copy_stream_avx2(char *dst, const char *src, int64_t n) {
  int64_t i = 0;
  const int64_t head = (int64_t)((32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31);
  if (head) {
    const int64_t h = head < n ? head : n;
    std::memcpy(dst, src, (size_t)h);
    i = h;
  }
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 64));
    const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(src + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i *>(dst + i + 96), d);
  }
  if (i < n) std::memcpy(dst + i, src + i, (size_t)(n - i));
  _mm_sfence();
}

// Parallel host copy (pageable caller buffers <-> pinned staging of the
// host-buffer drop-in): the driver's own pageable path stages through one
// bounce buffer at single-thread memcpy speed; host threads move the bytes at
// the host's memory bandwidth instead, with streaming stores.
void copy_host_parallel(void *dst, const void *src, int64_t bytes, int threads) {
  if (bytes <= 0) return;
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (bytes < (1 << 20) || threads <= 1) {
    std::memcpy(dst, src, (size_t)bytes);
    return;
  }
#pragma omp parallel num_threads(threads)
  {
    const int nt = omp_get_num_threads(), t = omp_get_thread_num();
    const int64_t per = ((bytes + nt - 1) / nt + 63) / 64 * 64;
    const int64_t lo = (int64_t)t * per < bytes ? (int64_t)t * per : bytes;
    const int64_t hi = lo + per < bytes ? lo + per : bytes;
    char *d = static_cast<char *>(dst) + lo;
    const char *s = static_cast<const char *>(src) + lo;
    if (hi > lo) {
      if (avx2) copy_stream_avx2(d, s, hi - lo);
      else std::memcpy(d, s, (size_t)(hi - lo));
    }
  }
}

}  // namespace gsvr
