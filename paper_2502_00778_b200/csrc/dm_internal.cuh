// dm_internal.cuh -- context, device buffers and shared device helpers of
// libdualmesh.so.  Everything here is sm_100a-only; the library is compiled
// with -fmad=false so fp64 expressions round exactly like the serial oracle
// built with -ffp-contract=off.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include <type_traits>
#include <cstdio>
#include <string>

#include "dm_capi.h"

namespace dm {

using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i64 = std::int64_t;

// ---------------------------------------------------------------- buffers
// env DUALMESH_ALLOC_TRACE=1: print driver allocations / frees slower than 2 ms
inline void alloc_trace(const char* what, size_t bytes, std::chrono::steady_clock::time_point t0) {
  static const bool on = [] {
    const char* e = std::getenv("DUALMESH_ALLOC_TRACE");
    return e && e[0] == '1';
  }();
  if (!on) return;
  const double ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (ms > 2.0) std::fprintf(stderr, "[alloc] %s %.1f MB %.2f ms\n", what, bytes / 1e6, ms);
}

// devmem.cu: every device buffer is carved out of large pooled chunks.
cudaError_t dev_alloc(void** out, size_t bytes);
void dev_free(void* p);

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;  // elements allocated
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) dev_free(p);
    p = nullptr;
    n = 0;
  }
  void swap(DevBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
  }
  // (Re)allocate to exactly hold `count` elements; keeps the buffer when it
  // is already large enough.
  cudaError_t ensure(size_t count) {
    if (count <= n && p) return cudaSuccess;
    release();
    size_t bytes = (count ? count : 1) * sizeof(T);
    cudaError_t st = dev_alloc(reinterpret_cast<void**>(&p), bytes);
    if (st == cudaSuccess) n = count;
    else p = nullptr;
    return st;
  }
};

// Scratch arena for the temporaries of the plan builders: a few large
// device blocks reused across calls (a cold cudaMalloc / cudaFree costs
// 2-60 ms each on a fresh process, and the ring plan needs ~15
// temporaries).  Bump allocation, released by ArenaScope on exit; all users
// run on the context stream, so reuse is stream-ordered.
struct Arena {
  struct Block {
    char* p;
    size_t size;
  };
  Block blocks[16] = {};
  int nblocks = 0, cur = 0;
  size_t off = 0;
  Arena() = default;
  Arena(const Arena&) = delete;
  Arena& operator=(const Arena&) = delete;
  ~Arena() {
    for (int b = 0; b < nblocks; ++b) dev_free(blocks[b].p);
  }
  cudaError_t take(size_t bytes, void** out, size_t min_block) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    while (cur < nblocks) {
      if (off + bytes <= blocks[cur].size) {
        *out = blocks[cur].p + off;
        off += bytes;
        return cudaSuccess;
      }
      ++cur;
      off = 0;
    }
    if (nblocks == 16) return cudaErrorMemoryAllocation;
    const size_t sz = bytes > min_block ? bytes : min_block;
    char* p = nullptr;
    cudaError_t st = dev_alloc(reinterpret_cast<void**>(&p), sz);
    if (st != cudaSuccess) return st;
    blocks[nblocks++] = {p, sz};
    cur = nblocks - 1;
    off = bytes;
    *out = p;
    return cudaSuccess;
  }
};

struct ArenaScope {
  Arena& a;
  int cur;
  size_t off;
  explicit ArenaScope(Arena& arena) : a(arena), cur(arena.cur), off(arena.off) {}
  ~ArenaScope() {
    a.cur = cur;
    a.off = off;
  }
};

// Arena-backed stand-in for a local DevBuf: same .p / .ensure() surface.
template <typename T>
struct ScratchBuf {
  Arena& a;
  size_t min_block;
  T* p = nullptr;
  size_t n = 0;
  ScratchBuf(Arena& arena, size_t min_block_bytes) : a(arena), min_block(min_block_bytes) {}
  cudaError_t ensure(size_t count) {
    if (count <= n && p) return cudaSuccess;
    void* q = nullptr;
    cudaError_t st = a.take((count ? count : 1) * sizeof(T), &q, min_block);
    if (st == cudaSuccess) {
      p = static_cast<T*>(q);
      n = count;
    }
    return st;
  }
};

// 3D node coordinates padded to one 32-byte sector per node; loaded with a
// single 256-bit LDG (LDG.E.ENL2.256 on sm_100a).
struct __align__(32) d4 {
  double x, y, z, w;
};

}  // namespace dm

// ---------------------------------------------------------------- context
struct dm_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;

  int dim = 0;
  dm::i64 nv = 0, nE = 0, nB = 0;
  dm::DevBuf<double> coords;  // caller layout, dim doubles per node
  dm::DevBuf<dm::d4> x4;      // 3D padded copy (lazy: built from coords on demand)
  bool x4_fresh = false;      // x4 matches coords
  dm::DevBuf<int32_t> elems, bnd;

  // edge structures (K1)
  bool have_edges = false;
  dm::i64 ne = 0;
  dm::DevBuf<int2> edges;
  dm::DevBuf<dm::u32> os;  // origin_start (32-bit on device)
  dm::DevBuf<int32_t> e2l, inc_ptr, inc;
  bool have_ifl = false;
  dm::DevBuf<int2> ifl;  // face-list incidence, same order as inc (edges.cu, built on demand)
  // derived: incoming-edge CSR per node, boundary (edge,facet) pairs, node->element CSR
  bool have_in = false;
  dm::DevBuf<dm::u32> in_ptr;
  dm::DevBuf<int32_t> in_list;
  bool have_bedge = false;
  dm::i64 n_bedge = 0;
  dm::DevBuf<dm::u64> bedge;
  dm::DevBuf<dm::u32> tile_bptr;  // bedge slice per kTileEdges-edge tile
  bool have_tables = false, table_ok = false;
  dm::DevBuf<dm::u32> adj_ptr;
  dm::DevBuf<int32_t> adj;
  dm::DevBuf<uint16_t> codes;  // tables.cu
  dm::DevBuf<int4> tile_meta;  // 2 per tile: {A0,A1,P0,P1}, {j0,jl,0,0}
  bool have_rings = false, ring_ok = false;
  dm::i64 ring_max_nodes = 0, ring_fail = 0;
  dm::DevBuf<int32_t> tnodes;      // kTileNodeCap per tile (rings.cu)
  dm::DevBuf<dm::u32> tnode_cnt;
  dm::DevBuf<uint8_t> rcodes;      // lane-transposed warp blocks (rings.cu), bytes
  int code_width = 2;              // 1: 8-bit slots + per-lane header, 2: 16-bit words
  bool plan_colored = false;       // tile tables recoloured against bank conflicts
  dm::DevBuf<int4> ring_meta;      // per tile {C0, NC, NU | nbnd << 16, bptr}, offsets
  dm::DevBuf<int32_t> eperm;       // tile position p -> edge id (Morton origin order)
  dm::DevBuf<int32_t> morder;      // Morton rank -> node id
  dm::DevBuf<dm::u32> rpstart;     // rank r's outgoing edges at positions [rpstart[r], rpstart[r+1])
  dm::DevBuf<dm::u32> rin_ptr;     // rank r's incoming edges, as positions, in
  dm::DevBuf<int32_t> rin_list;    //   ascending edge id (rin_list[rin_ptr[r] ..])
  bool vol_by_rank = false;        // node ids lack locality: s in position order,
                                   // volume pass in Morton rank order
  dm::DevBuf<double2> mxy;         // coordinates in Morton rank order: (x, y)
  dm::DevBuf<double> mz;           //                                    z
  dm::DevBuf<dm::u64> bedge_p;     // (p << 32 | facet), sorted
  dm::DevBuf<dm::u32> tile_bptr_p; // bedge_p slice per tile
  dm::i64 n_bseg = 0;              // boundary edges (segments of bedge_p)
  dm::DevBuf<int4> bseg;           // per boundary edge {e, j, k, p}
  dm::DevBuf<dm::u32> bseg_start;  // its facets: bedge_p[bseg_start[i] .. bseg_start[i+1])
  // side list of the ring path: edges the ring codes cannot describe (more
  // than kRingMax incidences, a non-manifold or inconsistently oriented fan)
  // as {edge id, position}; the ring kernels give them a zero row and
  // k_navs_side recomputes them from the element list inside the same step
  dm::DevBuf<int2> side;
  dm::i64 n_side = 0;
  // row-tile plan (rowplan.cu), chosen over the Morton tiles for node
  // numberings whose id-contiguous edge ranges have small node tables
  bool row_plan = false;
  dm::i64 rt_ntiles = 0;
  dm::DevBuf<int4> rt_meta;         // per tile {code offset (32 B units), code bytes, runs, run block}
  dm::DevBuf<int2> rt_runs;         // kRowRuns per tile {first node, nodes | slot << 16}
  unsigned long long rt_bytes[3] = {0, 0, 0};  // per step: codes, table fill, meta + runs
  bool have_n2e = false;
  dm::DevBuf<dm::u32> n2e_ptr;
  dm::DevBuf<int32_t> n2e;

  // metrics
  bool have_navs = false, have_vols = false;
  int navs_algo = -1;
  dm::DevBuf<double> navs, svals, vols, velem;
  bool svals_pos = false;  // svals indexed by ring position p (rings.cu), not edge id

  // verify / reductions scratch
  dm::DevBuf<double> red;
  dm::DevBuf<dm::u64> redu;

  // generic scratch
  dm::DevBuf<dm::u32> cnt, fill;
  dm::DevBuf<dm::u64> tmp64;
  dm::DevBuf<dm::u32> seg_big;  // segment_sort: ids of segments longer than a warp's
  dm::DevBuf<dm::u32> seg_med;  // segment_sort (u32): ids of segments longer than a lane's
  dm::Arena arena;              // plan temporaries (rings.cu)
  dm::DevBuf<dm::u32> scan_tmp;
  dm::DevBuf<dm::u64> scan_tmp64;
  // K1 (edge_extract.cu): packed per-origin counts -> exclusive scan
  // (items << 32 | entries), entries (element ids bucketed by origin node),
  // look-back status per warp chunk, and the long-bucket side path
  dm::DevBuf<dm::u64> k1_cs;
  dm::DevBuf<dm::u32> k1_ent;
  dm::DevBuf<dm::u64> k1_status;
  dm::DevBuf<dm::u32> k1_bscan, k1_blist, k1_bseg, k1_bd;
  dm::DevBuf<dm::u64> k1_bitems;
  dm::DevBuf<int> flag;

  // derived boundary / validation
  dm::i64 n_derived = 0;
  dm::DevBuf<int32_t> derived;
  dm::DevBuf<dm::i64> vlist;  // first offending ids per class
  dm::i64 vlist_n[DM_VCOUNT] = {0};
  dm::i64 vlist_cap = 0;

  // tuning knob for the GATHER kernel shape (env DUALMESH_GATHER_CFG)
  int gather_cfg = 0;

  // pipelined host steps (dm_metrics_host_async): coordinates arrive on
  // s_h2d, results leave on s_d2h, the kernels stay on `stream`; navs / vols
  // alternate between two device buffers so step i+1 computes while step i
  // is still being copied out (PCIe is full duplex)
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_h2d = nullptr, ev_comp = nullptr, ev_out[2] = {nullptr, nullptr};
  int out_slot = 0;
  dm::DevBuf<double> navs_alt, vols_alt;

  // pinned staging buffers of the pageable host copies (hostio.cu)
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};

  // timing
  bool timing = false;
  // ring of per-step phase events (dm_set_timing(enable > 1)): 4 per step
  std::vector<cudaEvent_t> ev_ring;
  int ring_steps = 0;
  long long ring_pos = 0;  // steps recorded so far (slot = ring_pos % ring_steps)
  cudaEvent_t ev[8] = {nullptr};
  float last_ms[4] = {0, 0, 0, 0};
  dm::i64 launches = 0;
};

namespace dm {

// ---------------------------------------------------------------- errors
inline int fail(dm_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define DM_CK(ctx, call)                                                              \
  do {                                                                                \
    cudaError_t _st = (call);                                                         \
    if (_st != cudaSuccess)                                                           \
      return ::dm::fail((ctx), _st == cudaErrorMemoryAllocation ? DM_ERR_OOM : DM_ERR_CUDA, \
                        std::string(#call) + ": " + cudaGetErrorString(_st));         \
  } while (0)

// Launch with bookkeeping: counts the launch and checks the launch error.
#define DM_LAUNCH(ctx, kern, grid, block, smem, ...)                                  \
  do {                                                                                \
    if ((grid) > 0) {                                                                 \
      kern<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);                  \
      (ctx)->launches++;                                                              \
      cudaError_t _le = cudaGetLastError();                                           \
      if (_le != cudaSuccess)                                                         \
        return ::dm::fail((ctx), _le == cudaErrorMemoryAllocation ? DM_ERR_OOM : DM_ERR_CUDA, \
                          std::string("launch of " #kern ": ") + cudaGetErrorString(_le)); \
    }                                                                                 \
  } while (0)

// Edges per CTA tile of the edge-owned kernels (navs gather / finalize).
constexpr int kTileEdges = 256;
// Ring path (rings.cu): unique nodes per tile, incidences per edge.
constexpr int kTileNodeCap = 1536;
// 8-bit (256-node) plans keep, behind a tile's slot table in its tnodes row,
// the tile's ranks in ascending order (kTileFillRanks, -1 padded) and their
// recoloured slots as bytes (kTileFillSlots): the ring kernel's fill then
// reads its sources in rank order (rings.cu k_tile_color_warp)
constexpr int kTileFillRanks = 256;
constexpr int kTileFillSlots = 512;
constexpr int kRingMax = 24;
constexpr int kSideCap = 1 << 20;  // side-list entries (more: the ring plan is not used)
// Row-tile plan (rowplan.cu): tiles are contiguous edge-id ranges of at most
// kRowTile edges (7 warps) whose node table -- node-id runs copied straight
// from the caller's coordinates -- holds at most kRowSlots records.
constexpr int kRowTile = 224;
constexpr int kRowSlots = 256;
constexpr int kRowRuns = 32;       // node runs per tile (TMA bulk copies)
constexpr int kRowCodeCap = 4096;  // code bytes per tile (tile header + warp blocks)

inline unsigned grid_for(i64 n, int per_block) {
  return static_cast<unsigned>((n + per_block - 1) / per_block);
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ d4 ld_d4(const d4* p) {
  d4 r;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
               : "l"(p));
  return r;
}
// x, y, z of a padded node without the pad word (6 registers instead of 8).
__device__ __forceinline__ d4 ld_d3(const d4* p) {
  d4 r;
  asm("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  asm("ld.global.nc.f64 %0, [%1+16];" : "=d"(r.z) : "l"(p));
  r.w = 0.0;
  return r;
}
__device__ __forceinline__ double2 ld_d2(const double2* p) { return __ldg(p); }

// cp.async (LDGSTS) helpers: global -> shared without a register round trip.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem));
}
// L1-bypassing 16-byte copy (cp.async.cg: cached in L2 only)
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
// mbarrier helpers (shared::cta): per-buffer full / empty phases of the ring
// kernel's tile pipeline
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(a) : "memory");
}
// arrives on `bar` once every cp.async this thread issued so far has landed
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  unsigned done = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
// TMA bulk copy global -> shared (no tensor map): `bytes` (multiple of 16,
// both addresses 16-byte aligned) complete_tx on `bar`; the issuing thread
// first registers them with an arrive + expect_tx.
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1; }" ::"r"(a),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes,
                                         uint64_t* bar) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s),
      "l"(gmem), "r"(bytes), "r"(b)
      : "memory");
}
// TMA bulk copy shared -> global (bulk-group completion); the source must be
// made visible to the async proxy first (fence_async_smem).
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, unsigned bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"(s),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

__device__ __forceinline__ int4 ld_i4(const int4* p) { return __ldg(p); }

// Select el[i] for a runtime i in 0..3 without local-memory indexing.
__device__ __forceinline__ int sel4(int a0, int a1, int a2, int a3, int i) {
  return i == 0 ? a0 : (i == 1 ? a1 : (i == 2 ? a2 : a3));
}
__device__ __forceinline__ int sel3(int a0, int a1, int a2, int i) {
  return i == 0 ? a0 : (i == 1 ? a1 : a2);
}

// ref mesh.cpp:15 tet_opposite_face = {{1,2,3},{0,3,2},{0,1,3},{0,2,1}},
// packed as 2-bit local ids, 6 bits per face.
constexpr unsigned kOppPacked = (1u | 2u << 2 | 3u << 4) | (0u | 3u << 2 | 2u << 4) << 6 |
                                (0u | 1u << 2 | 3u << 4) << 12 | (0u | 2u << 2 | 1u << 4) << 18;
// ref mesh.cpp:17 tet_local_edges = {01,02,03,12,13,23}; 2D mesh.cpp:263-265 = {01,12,20}.
constexpr unsigned kTetEdgePacked =
    (0u | 1u << 2) | (0u | 2u << 2) << 4 | (0u | 3u << 2) << 8 | (1u | 2u << 2) << 12 |
    (1u | 3u << 2) << 16 | (2u | 3u << 2) << 20;
constexpr unsigned kTriEdgePacked = (0u | 1u << 2) | (1u | 2u << 2) << 4 | (2u | 0u << 2) << 8;

__device__ __forceinline__ void cross3(double u0, double u1, double u2, double v0, double v1,
                                       double v2, double& c0, double& c1, double& c2) {
  // ref mesh.cpp:25-27, same operation order
  c0 = u1 * v2 - u2 * v1;
  c1 = u2 * v0 - u0 * v2;
  c2 = u0 * v1 - u1 * v0;
}

// Warp-level inclusive scan of an int.
__device__ __forceinline__ int warp_incl_scan(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// ---------------------------------------------------------------- host-side primitives
// Exclusive scan of n u32 counts into out[0..n] (out[n] = total) on the ctx
// stream.  in and out may alias.  Returns DM_OK or an error code.
int scan_exclusive(dm_ctx* c, const u32* in, u32* out, i64 n);
int scan_exclusive_u64(dm_ctx* c, const u64* in, u64* out, i64 n);

// Sort each segment [seg[s], seg[s+1]) of data ascending; segments up to
// 4096 keys (larger ones set *flag = 1).  Keys are u32 or u64.
int segment_sort_u64(dm_ctx* c, u64* data, const u32* seg, i64 nseg);
// Keys unique within each segment (K1 payloads, boundary pairs); with ucnt,
// ucnt[s] := number of distinct high words in segment s.
int segment_sort_unique_u64(dm_ctx* c, u64* data, const u32* seg, i64 nseg, u32* ucnt);
// u32 keys must be unique within each segment (edge / element ids).
int segment_sort_u32(dm_ctx* c, u32* data, const u32* seg, i64 nseg);
// (key, value) pairs sorted lexicographically within each segment.
int segment_sort_kv(dm_ctx* c, u64* keys, u32* vals, const u32* seg, i64 nseg);
// Global sort of n u64 keys into keys_out; with vals, (key, value) pairs
// lexicographically (stable-sort order for values entering ascending);
// without, the keys must be unique.
int sort_u64(dm_ctx* c, const u64* keys, const u32* vals, i64 n, u64* keys_out, u32* vals_out);

__global__ void k_tile_bptr(const u64* bedge, u32 n, i64 ne, i64 ntiles, u32* tile_bptr);

// Derived structures, built lazily.
int ensure_incoming(dm_ctx* c);
int ensure_bedge(dm_ctx* c);
int ensure_n2e(dm_ctx* c);
int ensure_ifl(dm_ctx* c);  // face-list incidence for the FACES / traditional fallbacks
int ensure_tables(dm_ctx* c);
int ensure_rings(dm_ctx* c);
// rowplan.cu: builds the row-tile plan if the node numbering allows it
// (sets c->row_plan); called by ensure_rings before the Morton plan.
int try_row_plan(dm_ctx* c);
int build_edges_impl(dm_ctx* c);
// edge_extract.cu: the entry-bucket K1; returns DM_OK, an error, or
// kK1Unsupported when the mesh needs the generic item-sort path
// (repeated nodes in an element, more than 2^25 nodes).
constexpr int kK1Unsupported = -1000;
int build_edges_buckets(dm_ctx* c);
int navs_impl(dm_ctx* c, int algo, int variant);
int volumes_impl(dm_ctx* c, int algo);
// Coordinate-derived layouts.  coords_changed marks them stale (set-time
// entry points); pad_x4 rebuilds the padded copy; ensure_x4 rebuilds it only
// if stale (plan building, verification); refresh_ring_coords rebuilds the
// ring path's Morton-order copy from the raw coordinates.  Every metrics
// call rebuilds the layout its kernels read from the raw coordinates
// (navs_impl), so a timed step consumes the caller's coordinate array.
int coords_changed(dm_ctx* c);
int pad_x4(dm_ctx* c);
int ensure_x4(dm_ctx* c);
int refresh_ring_coords(dm_ctx* c);
int compute_element_volumes(dm_ctx* c);
int svals_from_navs(dm_ctx* c);

// Host phase timer of the plan (env DUALMESH_PLAN_TIMING=1): synchronises the
// stream at each mark and prints the wall time since the previous one.
struct PlanClock {
  dm_ctx* c;
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit PlanClock(dm_ctx* ctx) : c(ctx) {
    const char* e = std::getenv("DUALMESH_PLAN_TIMING");
    on = e && std::atoi(e) == 1;
    if (on) cudaStreamSynchronize(c->stream);
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(c->stream);
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[plan] %-22s %8.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// hostio.cu: copies between device buffers and caller host memory on the ctx
// stream -- pinned host memory directly, pageable memory chunked through two
// pinned staging buffers with multi-threaded host copies.  copy_h2d returns
// once `src` may be reused; copy_d2h once `dst` is filled.
int copy_h2d(dm_ctx* c, void* dst, const void* src, size_t bytes);
int copy_d2h(dm_ctx* c, void* dst, const void* src, size_t bytes);
void release_stage(dm_ctx* c);

// Read a device int flag (synchronises the stream).
int read_flag(dm_ctx* c, int* value);

// Timing helpers: record event slot i when timing is enabled.
inline void tmark(dm_ctx* c, int i) {
  if (!c->timing) return;
  if (c->ring_steps > 0) {
    // marks 0..2 come from dm_navs, 2 (again) and 3 from dm_volumes: the
    // step's row is complete at mark 3
    const size_t slot = static_cast<size_t>(c->ring_pos % c->ring_steps);
    cudaEventRecord(c->ev_ring[4 * slot + i], c->stream);
    if (i == 3) ++c->ring_pos;
  }
  cudaEventRecord(c->ev[i], c->stream);
}

}  // namespace dm
