// devmem.cu -- device memory for every buffer of the library (DevBuf, Arena).
//
// A cold cudaMalloc / cudaFree costs 2-80 ms each on a fresh process (measured
// on the B200 boxes: `DUALMESH_ALLOC_TRACE=1`), independent of the size, and a
// C5 context holds ~45 buffers, so first calls spent more time in the driver
// than in kernels.  Buffers are therefore carved out of large chunks (>= 2
// GB, or the request) with best-fit placement and coalescing frees; a chunk
// goes back to the driver when its last buffer is freed.  A free first
// synchronises the device -- the semantics of cudaFree, so a block can never
// be handed out again while a kernel on any stream still uses it.
#include <mutex>
#include <map>
#include <unordered_map>
#include <vector>

#include "dm_internal.cuh"

namespace dm {
namespace {

constexpr size_t kAlign = 512;
constexpr size_t kChunk = size_t(2) << 30;
constexpr size_t kGranule = size_t(2) << 20;

struct Chunk {
  char* base = nullptr;
  size_t size = 0;
  int device = 0;
  size_t used = 0;
  std::map<size_t, size_t> free;  // offset -> length, coalesced
};

struct Pool {
  std::mutex mu;
  std::vector<Chunk*> chunks;
  std::unordered_map<void*, std::pair<Chunk*, size_t>> live;
};

Pool& pool() {
  static Pool* p = new Pool;  // never destroyed: frees may run from static destructors
  return *p;
}

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

cudaError_t dev_alloc(void** out, size_t bytes) {
  *out = nullptr;
  bytes = round_up(bytes ? bytes : 1, kAlign);
  int dev = 0;
  cudaError_t st = cudaGetDevice(&dev);
  if (st != cudaSuccess) return st;
  Pool& P = pool();
  std::lock_guard<std::mutex> lock(P.mu);
  Chunk* bc = nullptr;
  size_t boff = 0, blen = ~size_t(0);
  for (Chunk* c : P.chunks) {
    if (c->device != dev) continue;
    for (const auto& [off, len] : c->free)
      if (len >= bytes && len < blen) {
        bc = c;
        boff = off;
        blen = len;
      }
  }
  if (!bc) {
    size_t sz = std::max(round_up(bytes, kGranule), kChunk);
    char* base = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    st = cudaMalloc(reinterpret_cast<void**>(&base), sz);
    if (st != cudaSuccess && sz > round_up(bytes, kGranule)) {  // tight memory: exact size
      cudaGetLastError();
      sz = round_up(bytes, kGranule);
      st = cudaMalloc(reinterpret_cast<void**>(&base), sz);
    }
    alloc_trace("cudaMalloc(chunk)", sz, t0);
    if (st != cudaSuccess) return st;
    bc = new Chunk;
    bc->base = base;
    bc->size = sz;
    bc->device = dev;
    bc->free[0] = sz;
    P.chunks.push_back(bc);
    boff = 0;
    blen = sz;
  }
  bc->free.erase(boff);
  if (blen > bytes) bc->free[boff + bytes] = blen - bytes;
  bc->used += bytes;
  void* p = bc->base + boff;
  P.live[p] = {bc, bytes};
  *out = p;
  return cudaSuccess;
}

void dev_free(void* p) {
  if (!p) return;
  cudaDeviceSynchronize();
  Pool& P = pool();
  std::lock_guard<std::mutex> lock(P.mu);
  auto it = P.live.find(p);
  if (it == P.live.end()) return;
  Chunk* c = it->second.first;
  size_t off = static_cast<char*>(p) - c->base, len = it->second.second;
  P.live.erase(it);
  c->used -= len;
  if (c->used == 0) {
    const auto t0 = std::chrono::steady_clock::now();
    cudaFree(c->base);
    alloc_trace("cudaFree(chunk)", c->size, t0);
    for (size_t i = 0; i < P.chunks.size(); ++i)
      if (P.chunks[i] == c) {
        P.chunks.erase(P.chunks.begin() + static_cast<long>(i));
        break;
      }
    delete c;
    return;
  }
  auto next = c->free.lower_bound(off);
  if (next != c->free.end() && next->first == off + len) {  // merge with the block after
    len += next->second;
    next = c->free.erase(next);
  }
  if (next != c->free.begin()) {  // merge with the block before
    auto prev = std::prev(next);
    if (prev->first + prev->second == off) {
      prev->second += len;
      return;
    }
  }
  c->free[off] = len;
}

}  // namespace dm
