// Host side of the API edge: staging pageable caller arrays into page-locked
// buffers for the upload DMA.
//
// Measured on the B200 host (tools/microbench/h2d_bench2.py, 40 MB float64):
// a threaded cached copy into pinned memory takes ~0.9 ms and a DMA from a
// clean pinned buffer 0.73 ms, but copy + DMA back to back take 2.7 ms: the
// freshly written lines sit dirty in the CPU caches and the DMA reads them
// through snoops.  Non-temporal (streaming) stores write around the caches,
// so the DMA reads DRAM at full rate.  Threads split the copy; each thread
// ends with an sfence so the stores are globally visible before the caller
// queues the DMA.
#include <emmintrin.h>
#include <xmmintrin.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

// dst must be 16-byte aligned (page-locked buffers are page aligned); src any.
void stream_copy(char* dst, const char* src, size_t bytes) {
  size_t i = 0;
  for (; i + 64 <= bytes; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  if (i < bytes) std::memcpy(dst + i, src + i, bytes - i);
  _mm_sfence();
}

// float64 -> float32 (round to nearest, as numpy's astype), streaming stores.
void stream_narrow(float* dst, const double* src, size_t n) {
  size_t i = 0;
  for (; i + 8 <= n; i += 8) {
    const __m128 a = _mm_movelh_ps(_mm_cvtpd_ps(_mm_loadu_pd(src + i)), _mm_cvtpd_ps(_mm_loadu_pd(src + i + 2)));
    const __m128 b = _mm_movelh_ps(_mm_cvtpd_ps(_mm_loadu_pd(src + i + 4)), _mm_cvtpd_ps(_mm_loadu_pd(src + i + 6)));
    _mm_stream_ps(dst + i, a);
    _mm_stream_ps(dst + i + 4, b);
  }
  for (; i < n; ++i) dst[i] = (float)src[i];
  _mm_sfence();
}

template <class F>
void split(size_t n, size_t grain, int threads, F f) {
  threads = std::max(1, std::min<int>(threads, (int)((n + grain - 1) / grain)));
  if (threads == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> pool;
  const size_t per = ((n + threads - 1) / threads + grain - 1) / grain * grain;
  for (int t = 0; t < threads; ++t) {
    const size_t a = std::min(n, per * t), b = std::min(n, a + per);
    if (a < b) pool.emplace_back(f, a, b);
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

// dst: 16-byte aligned page-locked buffer; copies `bytes` from src.
int pab_host_stage_copy(void* dst, const void* src, size_t bytes, int threads) {
  if (!dst || !src) return 1;
  if (reinterpret_cast<uintptr_t>(dst) & 15) return 1;
  split(bytes, 64 * 1024, threads, [&](size_t a, size_t b) {
    stream_copy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
  });
  return 0;
}

// dst[i] = (float)src[i], i < n; dst 16-byte aligned.
int pab_host_stage_narrow(float* dst, const double* src, size_t n, int threads) {
  if (!dst || !src) return 1;
  if (reinterpret_cast<uintptr_t>(dst) & 15) return 1;
  split(n, 16 * 1024, threads, [&](size_t a, size_t b) { stream_narrow(dst + a, src + a, b - a); });
  return 0;
}

}  // extern "C"
