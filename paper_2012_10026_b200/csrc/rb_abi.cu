// rb_abi.cu -- error plumbing of the C ABI (include/rcmbfs_b200.h).
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif

#include <thread>
#include <vector>

#include "rb_error.h"

static thread_local char g_err[1024] = "";

extern "C" void rb_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* rb_last_error(void) { return g_err; }

extern "C" int rb_version(void) { return 1; }

// Host-side fill of a result array's tail (the isolated vertices' -1 entries,
// engine.py:598): streaming (non-temporal) stores from a few threads.  The fill
// runs while the parents are DMA'd into the head of the same array; ordinary
// stores read every line before writing it and take host memory bandwidth from
// the DMA (measured: BfsEngine.run 3.18 ms per scale-26 root with a cached
// 16-thread fill against 2.72 ms of traversal + DMA).
static void fill_range(int32_t* p, int64_t n, int32_t value) {
#if defined(__x86_64__)
  while (n > 0 && (reinterpret_cast<uintptr_t>(p) & 15)) {
    *p++ = value;
    --n;
  }
  const __m128i v = _mm_set1_epi32(value);
  int64_t i = 0;
  for (; i + 16 <= n; i += 16) {
    _mm_stream_si128(reinterpret_cast<__m128i*>(p + i), v);
    _mm_stream_si128(reinterpret_cast<__m128i*>(p + i + 4), v);
    _mm_stream_si128(reinterpret_cast<__m128i*>(p + i + 8), v);
    _mm_stream_si128(reinterpret_cast<__m128i*>(p + i + 12), v);
  }
  for (; i < n; ++i) p[i] = value;
  _mm_sfence();
#else
  for (int64_t i = 0; i < n; ++i) p[i] = value;
#endif
}

extern "C" int rb_host_fill_i32(int32_t* h_dst, int64_t n, int32_t value, int threads) {
  if (n <= 0) return RB_OK;
  if (!h_dst || threads < 1 || threads > 256) {
    rb_set_error("rb_host_fill_i32: bad argument (n=%lld threads=%d)", (long long)n, threads);
    return RB_ERR_ARG;
  }
  const int64_t kMin = 1 << 20;  // entries per thread worth a thread
  int t = (int)((n + kMin - 1) / kMin);
  if (t > threads) t = threads;
  if (t <= 1) {
    fill_range(h_dst, n, value);
    return RB_OK;
  }
  const int64_t per = ((n + t - 1) / t + 15) & ~(int64_t)15;
  std::vector<std::thread> th;
  for (int k = 1; k < t; ++k) {
    const int64_t a = k * per, b = a + per < n ? a + per : n;
    if (a < b) th.emplace_back(fill_range, h_dst + a, b - a, value);
  }
  fill_range(h_dst, per < n ? per : n, value);
  for (auto& x : th) x.join();
  return RB_OK;
}
