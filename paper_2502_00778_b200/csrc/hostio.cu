// hostio.cu -- host <-> device copies of the C-ABI's host buffers.
//
// The C++ drop-in API (mesh.hpp / metrics.hpp) hands the library plain
// std::vector storage: pageable memory.  A cudaMemcpy from or to pageable
// memory runs at a few GB/s (the driver stages it through its own small
// pinned buffer, one thread), so a C5 result (2.8 GB of navs) took ~0.75 s to
// come back.  Here pageable transfers are chunked through two pinned staging
// buffers owned by the context: while chunk i crosses PCIe, chunk i-1 is
// copied between the staging buffer and the caller's memory by a small pool
// of host threads.  Pinned (or registered) caller buffers go straight to
// cudaMemcpyAsync.  Both calls return once the host buffer may be reused
// (H2D: the data sits in staging or on the device, in stream order; D2H: the
// data is in the caller's buffer).
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "dm_internal.cuh"

namespace dm {
namespace {

constexpr size_t kStageBytes = size_t(64) << 20;  // per staging buffer

// Fixed pool of memcpy workers: parallel_copy splits [0, n) into one slice
// per worker and returns when every slice is done.
class CopyPool {
 public:
  CopyPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    n_ = static_cast<int>(std::min(16u, hw));
    for (int i = 1; i < n_; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void copy(void* dst, const void* src, size_t n) {
    if (n < (size_t(1) << 20) || n_ == 1) {
      std::memcpy(dst, src, n);
      return;
    }
    std::unique_lock<std::mutex> g(mu_);
    dst_ = static_cast<char*>(dst);
    src_ = static_cast<const char*>(src);
    len_ = n;
    pending_ = n_ - 1;
    ++gen_;
    g.unlock();
    cv_.notify_all();
    slice(0);
    g.lock();
    done_.wait(g, [this] { return pending_ == 0; });
  }

 private:
  void slice(int i) {
    const size_t per = ((len_ + n_ - 1) / n_ + 63) & ~size_t(63);  // n_ slices cover len_
    const size_t a = std::min(len_, per * static_cast<size_t>(i));
    const size_t b = std::min(len_, a + per);
    if (b > a) std::memcpy(dst_ + a, src_ + a, b - a);
  }
  void loop(int i) {
    unsigned long seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> g(mu_);
      cv_.wait(g, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      g.unlock();
      slice(i);
      g.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int n_ = 1;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  unsigned long gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t len_ = 0;
};

CopyPool& pool() {
  static CopyPool* p = new CopyPool;  // lives for the process (frees may run at exit)
  return *p;
}

bool pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

int ensure_stage(dm_ctx* c) {
  if (c->stage[0]) return DM_OK;
  for (int i = 0; i < 2; ++i) {
    DM_CK(c, cudaMallocHost(&c->stage[i], kStageBytes));
    DM_CK(c, cudaEventCreateWithFlags(&c->stage_ev[i], cudaEventDisableTiming));
  }
  return DM_OK;
}

}  // namespace

int copy_h2d(dm_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return DM_OK;
  if (bytes <= (size_t(4) << 20) || pinned(src)) {
    DM_CK(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
    return DM_OK;
  }
  if (int st = ensure_stage(c)) return st;
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  for (size_t off = 0, i = 0; off < bytes; off += kStageBytes, ++i) {
    const int b = static_cast<int>(i & 1);
    const size_t n = std::min(kStageBytes, bytes - off);
    // the buffer's previous transfer (this call's chunk i - 2, or the last
    // chunks of an earlier call still queued) must have left it
    DM_CK(c, cudaEventSynchronize(c->stage_ev[b]));
    pool().copy(c->stage[b], s + off, n);
    DM_CK(c, cudaMemcpyAsync(d + off, c->stage[b], n, cudaMemcpyHostToDevice, c->stream));
    DM_CK(c, cudaEventRecord(c->stage_ev[b], c->stream));
  }
  return DM_OK;
}

int copy_d2h(dm_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return DM_OK;
  if (bytes <= (size_t(4) << 20) || pinned(dst)) {
    DM_CK(c, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    return DM_OK;
  }
  if (int st = ensure_stage(c)) return st;
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  const size_t nchunk = (bytes + kStageBytes - 1) / kStageBytes;
  auto issue = [&](size_t i) -> int {
    const int b = static_cast<int>(i & 1);
    const size_t off = i * kStageBytes, n = std::min(kStageBytes, bytes - off);
    // (stream order puts this copy after any earlier transfer of the buffer;
    // the host copies out of it below are synchronous)
    DM_CK(c, cudaMemcpyAsync(c->stage[b], s + off, n, cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaEventRecord(c->stage_ev[b], c->stream));
    return DM_OK;
  };
  if (int st = issue(0)) return st;
  for (size_t i = 0; i < nchunk; ++i) {
    // chunk i + 1 crosses PCIe while chunk i is copied out of staging
    if (i + 1 < nchunk)
      if (int st = issue(i + 1)) return st;
    const int b = static_cast<int>(i & 1);
    const size_t off = i * kStageBytes, n = std::min(kStageBytes, bytes - off);
    DM_CK(c, cudaEventSynchronize(c->stage_ev[b]));
    pool().copy(d + off, c->stage[b], n);
  }
  return DM_OK;
}

void release_stage(dm_ctx* c) {
  for (int i = 0; i < 2; ++i) {
    if (c->stage[i]) cudaFreeHost(c->stage[i]);
    if (c->stage_ev[i]) cudaEventDestroy(c->stage_ev[i]);
    c->stage[i] = nullptr;
    c->stage_ev[i] = nullptr;
  }
}

}  // namespace dm
