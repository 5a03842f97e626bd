// Host-side staging for the end-to-end path: a caller's pageable numpy inputs are copied into the
// engine's pinned buffers before the H2D DMA.  Two things make a plain memcpy slow here, both
// measured on the GPU box (tools/copy_bw_probe.py, tools/e2e_gpu_trace.py --numpy): one core
// moves ~5 GB/s into pinned memory, and the DMA engine then reads freshly written lines that are
// still dirty in the CPU caches at about half its normal rate (X* from a just-staged buffer:
// 1.4 ms instead of 0.45 ms for 24 MB).  fagp_host_copy splits the copy over threads and writes
// with non-temporal (streaming) stores, which bypass the caches: the data is in DRAM, not dirty
// in L2/L3, when the copy engine reads it.
#include <emmintrin.h>

#include <cstdint>
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "fagp_b200.h"

namespace {

void stream_copy(char* dst, const char* src, size_t n) {
  // align the destination to 16 bytes with a plain copy, stream the body, plain copy the tail
  const size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
  if (head >= n) {
    std::memcpy(dst, src, n);
    return;
  }
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  const size_t body = n & ~size_t(63);
  for (size_t i = 0; i < body; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
  }
  std::memcpy(dst + body, src + body, n - body);
  _mm_sfence();
}

// A small persistent worker pool: thread creation (~10-20 us each) would otherwise dominate the
// per-chunk staging copies of the host pipeline.  run(n, f) calls f(0) .. f(n-1), f(0) on the
// calling thread, and returns when all are done; calls are serialised.
class Pool {
 public:
  void run(int n, const std::function<void(int)>& f) {
    if (n <= 1) {
      if (n == 1) f(0);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);
    ensure(n - 1);
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &f;
      next_ = 1;
      total_ = n;
      pending_ = n - 1;
      ++gen_;
    }
    cv_.notify_all();
    f(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  void ensure(int workers) {
    while (int(threads_.size()) < workers) threads_.emplace_back([this] { loop(); });
  }
  void loop() {
    unsigned long long seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return gen_ != seen && next_ < total_; });
      seen = gen_;
      while (next_ < total_) {
        const int i = next_++;
        const std::function<void(int)>* f = fn_;
        lk.unlock();
        (*f)(i);
        lk.lock();
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> threads_;
  const std::function<void(int)>* fn_ = nullptr;
  int next_ = 0, total_ = 0, pending_ = 0;
  unsigned long long gen_ = 0;
};

Pool& pool() {
  static Pool* p = new Pool();  // never destroyed: workers live for the process
  return *p;
}

}  // namespace

// height rows of width bytes (dst / src row pitches in bytes), rows split over the threads
extern "C" int fagp_host_copy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                                 size_t height, int32_t threads) {
  if (width == 0 || height == 0) return FAGP_OK;
  if (dst == nullptr || src == nullptr || dpitch < width || spitch < width) return FAGP_EINVAL;
  if (threads < 1) threads = 1;
  const size_t min_chunk = size_t(256) << 10;
  const size_t nt = std::max<size_t>(1, std::min<size_t>(std::min<size_t>(size_t(threads), height), width * height / min_chunk));
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  pool().run(int(nt), [&](int t) {
    for (size_t r = height * size_t(t) / nt; r < height * size_t(t + 1) / nt; ++r)
      stream_copy(d + r * dpitch, s + r * spitch, width);
  });
  return FAGP_OK;
}

extern "C" int fagp_host_copy(void* dst, const void* src, size_t bytes, int32_t threads) {
  if (bytes == 0) return FAGP_OK;
  if (dst == nullptr || src == nullptr) return FAGP_EINVAL;
  if (threads < 1) threads = 1;
  const size_t min_chunk = size_t(256) << 10;  // below ~256 KB per thread the hand-off costs more
  const size_t nt = std::max<size_t>(1, std::min<size_t>(size_t(threads), bytes / min_chunk));
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  if (nt == 1) {
    stream_copy(d, s, bytes);
    return FAGP_OK;
  }
  auto cut = [&](size_t i) { return i == nt ? bytes : (bytes * i / nt) & ~size_t(63); };
  pool().run(int(nt), [&](int t) { stream_copy(d + cut(t), s + cut(t), cut(t + 1) - cut(t)); });
  return FAGP_OK;
}

// 1 when the device can write the host range [p, p + bytes) through the same address (pinned and
// mapped: cudaHostAlloc'd memory under unified addressing), else 0.  No device work.
extern "C" int fagp_host_mapped(const void* p, size_t bytes) {
  if (p == nullptr) return 0;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (at.type != cudaMemoryTypeHost || at.devicePointer != p) return 0;
  const char* last = static_cast<const char*>(p) + (bytes ? bytes - 1 : 0);
  cudaPointerAttributes at2{};
  if (cudaPointerGetAttributes(&at2, last) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return at2.type == cudaMemoryTypeHost && at2.devicePointer == last ? 1 : 0;
}
