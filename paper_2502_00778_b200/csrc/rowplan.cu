// rowplan.cu -- the row-tile plan of the GATHER path (3D) for node numberings
// with spatial coherence (lexicographic structured grids, RCM-ordered
// unstructured ones).
//
// The ring walk of rings.cu evaluates one edge per thread from a
// shared-memory table of the tile's nodes.  With Morton tiles (rings.cu) the
// tile's edges are scattered over the edge list (a permutation eperm), the
// table is filled node by node from a per-call Morton-order copy of the
// coordinates, and the rows go out as scattered per-lane stores.  Here a tile
// is instead a contiguous edge-id range [e0, e0 + cnt), cnt <= kRowTile
// (split in halves until its table fits), and
//   * its node table is a handful of contiguous node-id runs (a row of
//     origins and its neighbour rows), copied by TMA bulk copies straight
//     from the caller's coordinate array (24-byte records; runs are padded to
//     even node ids so every copy is 16-byte aligned) -- no coordinate copy
//     per call, no per-node fill instructions;
//   * the lanes of the tile take its edges sorted by ring length, then by
//     the edge's index inside its origin row, then by origin: a warp's lanes
//     walk rings of one length (a Kuhn grid's even and odd cubes give one
//     edge direction 4- and 6-rings), and for a structured grid they hold
//     the same edge direction of consecutive origins, so a ring step reads
//     consecutive table slots (few bank conflicts);
//   * the rows are staged in shared memory and leave as two TMA bulk stores
//     per tile (navs rows, s terms) -- contiguous, no per-lane stores.
// The plan is used when the tiles split little (<= 25 % more tiles than
// ne / kRowTile); otherwise the Morton plan of rings.cu.
//
// Code block of a tile (32-byte units, contiguous, at a fixed kRowCodeCap
// stride -- the builder writes every tile in one pass, no size scan):
//   [tile header 32 B: e0 (i32), cnt (i32), eight u16 byte offsets of the
//    warp blocks from the tile's code start]
//   per warp w: [32 B: n | sign << 5 | closed << 7 per lane]
//               [32 B: edge offset e - e0 per lane]
//               [S_w steps x 32 B: slot(j), slot(k), slot(m_0), slot(m_1) ..]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include "dm_internal.cuh"
#include "ring_encode.cuh"

namespace dm {
namespace {

constexpr int kRTThreads = 256;   // plan kernel: one CTA per tile
constexpr int kRTHash = 2048;  // <= 512 unique nodes: load factor <= 1/4
constexpr int kRTUniqCap = 512;
constexpr int kRTCodeUnits = kRowCodeCap / 32;

// infeasibility bits of a candidate tile
constexpr int kRTTooManyNodes = 1;
constexpr int kRTTooManyRuns = 2;
constexpr int kRTTooManyCodes = 4;

constexpr int kBitPairs = 4096 * 32;  // pair bitmap: a tile's node-pair span up to 131072

struct RTShared {
  union {
    struct {
      int hs[kRTHash];
      int uq[kRTUniqCap];
    } h;                       // node set as a hash set (wide node spans)
    unsigned bm[kBitPairs / 32];  // node pairs as a bitmap over the tile's span
  } u;
  unsigned key[kRTThreads], ktmp[kRTThreads];
  int vmin[8], vmax[8], hcount[8];
  int2 heads[kRowRuns];  // run heads {first pair, pairs}, unsorted
  int n_uniq;
  int nruns, nslots;
  int2 runs[kRowRuns];
  int wmax[8];
  int woff[8];
};

// Sorts the kRTThreads unique keys a[t] ascending in place: each warp sorts
// its 32 keys with a shuffle bitonic network (no block barriers), then every
// key's rank is its rank in its warp plus, per other warp, the number of
// that warp's keys below it (binary search in the warp's sorted run).
__device__ __forceinline__ void warp_merge_sort_u32(unsigned* a, unsigned* tmp, int t) {
  const int lane = t & 31, w = t >> 5;
  unsigned x = a[t];
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const unsigned y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = (lane & k) == 0, lower = (lane & j) == 0;
      x = (lower == up) ? min(x, y) : max(x, y);
    }
  tmp[t] = x;  // warp w's sorted run at tmp[32w .. 32w + 32)
  __syncthreads();
  int r = lane;
#pragma unroll
  for (int v = 0; v < kRTThreads / 32; ++v) {
    if (v == w) continue;
    const unsigned* run = tmp + 32 * v;
    int lo = 0;  // keys of run v below x
#pragma unroll
    for (int step = 16; step > 0; step >>= 1)
      if (run[lo + step - 1] < x) lo += step;
    r += lo + (run[31] < x && lo == 31 ? 1 : 0);
  }
  __syncthreads();
  a[r] = x;
  __syncthreads();
}

// One CTA per candidate tile {e0, cnt} (tile index p = base + blockIdx.x):
// the tile's node set (shared-memory hash set), sorted; its runs of node-id
// pairs (a run covers pairs [a, b], i.e. nodes [2a, 2b + 2): every copy is
// 16-byte aligned; consecutive or equal pairs extend a run); the
// lane order (ring length, then direction); and, if the tile fits (<= kRowRuns runs,
// <= kRowSlots slots, <= kRowCodeCap code bytes), its runs and its code block
// at codes + p * kRowCodeCap.  Otherwise bad[p] says why (the host splits it).
__global__ void __launch_bounds__(kRTThreads)
    k_rt_build(const int2* __restrict__ cand, int base, const int2* __restrict__ edges,
               const u32* __restrict__ os, const int32_t* __restrict__ inc_ptr,
               const int32_t* __restrict__ inc, const int32_t* __restrict__ el,
               uint8_t* __restrict__ bad, int2* __restrict__ runs_out, int* __restrict__ nruns_out,
               int* __restrict__ bytes_out, uint8_t* __restrict__ codes, int by_len) {
  __shared__ RTShared S;
  const int t = threadIdx.x, lane = t & 31;
  const i64 p = static_cast<i64>(base) + blockIdx.x;
  const int2 cd = cand[blockIdx.x];
  const int e0 = cd.x, cnt = cd.y;
  if (t == 0) {
    S.n_uniq = 0;
    S.nruns = 0;
  }
  if (t < 8) S.wmax[t] = 0;
  auto insert = [&](int v) {
    unsigned h = (static_cast<unsigned>(v) * 2654435761u) >> 21;  // 11 bits
    for (int probe = 0; probe < kRTHash; ++probe, h = (h + 1) & (kRTHash - 1)) {
      const int old = atomicCAS(&S.u.h.hs[h], -1, v);
      if (old == -1) {
        const int q = atomicAdd(&S.n_uniq, 1);
        if (q < kRTUniqCap) S.u.h.uq[q] = v;
        return;
      }
      if (old == v) return;
    }
  };
  int n_inc = 0, pb = 0, nq = 0;
  int2 jk = make_int2(0, 0);
  unsigned key = 0xffffff00u | static_cast<unsigned>(t);  // idle lanes: unique, after every edge
  if (t < cnt) {
    const int e = e0 + t;
    jk = edges[e];
    pb = inc_ptr[e];
    n_inc = inc_ptr[e + 1] - pb;
    // the ring nodes: the two others of each element (a side-list edge, more
    // than kRingMax incidences, needs only j and k in the table)
    nq = n_inc > kRingMax ? 0 : n_inc;
    // direction-major: index of the edge inside its origin row, then origin
    key = (static_cast<unsigned>(e - static_cast<int>(os[jk.x])) << 8) | static_cast<unsigned>(t);
    if (by_len)  // ring length first (warps of equal trip counts: on the Kuhn grids the
                 // even/odd cube orientation splits a direction into 4- and 6-rings)
      key = static_cast<unsigned>(min(n_inc, 31)) << 27 |
            min(static_cast<unsigned>(e - static_cast<int>(os[jk.x])), (1u << 19) - 1u) << 8 |
            static_cast<unsigned>(t);
  }
  S.key[t] = key;
  // this edge's table nodes: j, k and its ring's nodes (element ids and rows
  // loaded eight at a time: two round trips per batch)
  auto for_nodes = [&](auto&& fn) {
    if (t >= cnt) return;
    fn(jk.x);
    fn(jk.y);
    int last = -1;
    for (int q0 = 0; q0 < nq; q0 += 8) {
      int id[8];
      int4 rows[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) id[u] = q0 + u < nq ? __ldg(inc + pb + q0 + u) : -1;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        rows[u] = id[u] >= 0 ? __ldg(reinterpret_cast<const int4*>(el) + id[u])
                             : make_int4(jk.x, jk.x, jk.x, jk.x);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int vs[4] = {rows[u].x, rows[u].y, rows[u].z, rows[u].w};
#pragma unroll
        for (int a = 0; a < 4; ++a)
          if (vs[a] != jk.x && vs[a] != jk.y && vs[a] != last) {
            fn(vs[a]);
            last = vs[a];
          }
      }
    }
  };
  // the tile's node-pair span: a bitmap when it fits, else the hash set
  {
    int lo = 0x7fffffff, hi = -1;
    for_nodes([&](int v) {
      lo = min(lo, v);
      hi = max(hi, v);
    });
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0) {
      S.vmin[t >> 5] = lo;
      S.vmax[t >> 5] = hi;
    }
  }
  __syncthreads();
  int vlo = 0x7fffffff, vhi = -1;
#pragma unroll
  for (int w = 0; w < kRTThreads / 32; ++w) {
    vlo = min(vlo, S.vmin[w]);
    vhi = max(vhi, S.vmax[w]);
  }
  const int pmin = vlo >> 1;
  const int npairs = vhi >= vlo ? (vhi >> 1) - pmin + 1 : 0;
  const bool bits = npairs <= kBitPairs;
  const int nw = (npairs + 31) >> 5;
  if (bits) {
    for (int i = t; i < nw; i += kRTThreads) S.u.bm[i] = 0u;
  } else {
    for (int i = t; i < kRTHash; i += kRTThreads) S.u.h.hs[i] = -1;
  }
  __syncthreads();
  if (bits) {
    for_nodes([&](int v) {
      const int q = (v >> 1) - pmin;
      atomicOr(&S.u.bm[q >> 5], 1u << (q & 31));
    });
  } else {
    for_nodes(insert);
  }
  __syncthreads();
  int badbits = 0;
  if (bits) {
    // runs: a set pair after a clear one opens a run; a thread scans a slice
    // of words, runs are numbered in pair order by a block scan of the heads
    const int W = (nw + kRTThreads - 1) / kRTThreads;
    const int w0 = min(nw, t * W), w1 = min(nw, w0 + W);
    auto heads_of = [&](int i) -> unsigned {
      const unsigned x = S.u.bm[i], prev = i > 0 ? S.u.bm[i - 1] >> 31 : 0u;
      return x & ~((x << 1) | prev);
    };
    int c = 0;
    for (int i = w0; i < w1; ++i) c += __popc(heads_of(i));
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) S.hcount[t >> 5] = incl;
    __syncthreads();
    int r = incl - c;
    for (int w = 0; w < (t >> 5); ++w) r += S.hcount[w];
    if (t == kRTThreads - 1) S.nruns = r + c;
    for (int i = w0; i < w1; ++i) {
      unsigned h = heads_of(i);
      while (h) {
        const int b = __ffs(h) - 1;
        h &= h - 1;
        if (r < kRowRuns) {
          // the run ends at the next clear pair
          int wi = i;
          unsigned z = ~S.u.bm[wi] & (0xffffffffu << b);
          while (!z && ++wi < nw) z = ~S.u.bm[wi];
          const int end = z ? 32 * wi + __ffs(z) - 1 : 32 * nw;
          S.heads[r] = make_int2(pmin + 32 * i + b, end - (32 * i + b));
        }
        ++r;
      }
    }
  } else {
    const int nu = S.n_uniq;
    if (nu > kRTUniqCap) badbits = kRTTooManyNodes;
    if (!badbits) {
      // runs of node pairs straight from the hash set (no sorted node list): a
      // present pair p (node 2p or 2p + 1 in the tile) opens a run iff pair
      // p - 1 is absent; the run extends while the next pairs are present.
      auto present = [&](int v) -> bool {
        if (v < 0) return false;
        unsigned h = (static_cast<unsigned>(v) * 2654435761u) >> 21;
        for (int probe = 0; probe < kRTHash; ++probe, h = (h + 1) & (kRTHash - 1)) {
          const int x = S.u.h.hs[h];
          if (x == v) return true;
          if (x == -1) return false;
        }
        return false;
      };
      for (int i = t; i < nu; i += kRTThreads) {
        const int v = S.u.h.uq[i], pr = v >> 1;
        const bool rep = !(v & 1) || !present(v - 1);  // one representative per pair
        if (rep && !present(2 * pr - 2) && !present(2 * pr - 1)) {
          int len = 1;
          while (present(2 * (pr + len)) || present(2 * (pr + len) + 1)) ++len;
          const int r = atomicAdd(&S.nruns, 1);
          if (r < kRowRuns) S.heads[r] = make_int2(pr, len);
        }
      }
    }
  }
  if (__syncthreads_or(badbits)) {
    if (t == 0) bad[p] = static_cast<uint8_t>(kRTTooManyNodes);
    return;
  }
  warp_merge_sort_u32(S.key, S.ktmp, t);  // lane order (its barriers also publish the heads)
  if (t < 32) {  // order the heads by pair, then slot offsets
    const int nr = min(S.nruns, kRowRuns);
    const int2 hd = t < nr ? S.heads[t] : make_int2(0x7fffffff, 0);
    int rank = 0;
    for (int q = 0; q < nr; ++q) rank += __shfl_sync(0xffffffffu, hd.x, q) < hd.x;
    int x = t < nr ? 2 * hd.y : 0;  // exclusive scan in pair order: by rank
    int off = 0;
    for (int q = 0; q < nr; ++q) {
      const int rq = __shfl_sync(0xffffffffu, rank, q);
      const int lq = __shfl_sync(0xffffffffu, x, q);
      off += rq < rank ? lq : 0;
    }
    const int tot = __reduce_add_sync(0xffffffffu, x);
    __syncwarp();
    if (t < nr) S.runs[rank] = make_int2(2 * hd.x, (2 * hd.y) | off << 16);
    if (t == 0) S.nslots = tot;
  }
  __syncthreads();
  const unsigned kq = S.key[t];
  const int q = static_cast<int>(kq & 0xffu);
  const int e = e0 + q;
  if (t < cnt) {
    const int n = inc_ptr[e + 1] - inc_ptr[e];
    atomicMax(&S.wmax[t >> 5], (n > kRingMax ? 0 : n) + 3);  // side edges: 3 steps
  }
  __syncthreads();
  if (S.nruns > kRowRuns) badbits |= kRTTooManyRuns;
  else if (S.nslots > kRowSlots) badbits |= kRTTooManyNodes;
  if (t == 0) {  // warp block byte offsets (S.woff[7]: the tile's code bytes)
    int units = 1;  // tile header
    for (int w = 0; w < kRowTile / 32; ++w) {
      S.woff[w] = 32 * units;
      if (w * 32 < cnt) units += 2 + S.wmax[w];
    }
    S.woff[kRowTile / 32] = 32 * units;
  }
  __syncthreads();
  const int units = S.woff[kRowTile / 32] / 32;
  if (units > kRTCodeUnits) badbits |= kRTTooManyCodes;
  if (t == 0) bad[p] = static_cast<uint8_t>(badbits);
  if (badbits) return;
  if (t < kRowRuns) runs_out[p * kRowRuns + t] = t < S.nruns ? S.runs[t] : make_int2(0, 0);
  if (t == 0) {
    nruns_out[p] = S.nruns;
    bytes_out[p] = 32 * units;
  }
  uint8_t* tb = codes + p * kRowCodeCap;
  if (t == 0) {  // tile header: e0, cnt, warp block offsets
    int* h = reinterpret_cast<int*>(tb);
    h[0] = e0;
    h[1] = cnt;
    uint16_t* wo = reinterpret_cast<uint16_t*>(h + 2);
    for (int w = 0; w < 8; ++w) wo[w] = static_cast<uint16_t>(S.woff[w]);
  }
  if (t < cnt) tb[S.woff[t >> 5] + 32 + lane] = static_cast<uint8_t>(q);  // lane -> edge
}

// Ring codes (k_rt_build has written the tile header and each lane's edge
// offset): one CTA per tile, the runs in shared memory, one thread per lane.
// An edge the walk cannot encode (more than kRingMax incidences, a
// non-manifold or inconsistently oriented fan) gets an empty ring (header n =
// 0, slots j, k, k: the kernel writes a zero row) and goes to the side list
// {e, e}; flag[0] collects the kRing* reasons, flag[1] counts the list.
__global__ void __launch_bounds__(kRowTile)
    k_rt_codes(const int* __restrict__ order, const int2* __restrict__ edges,
               const int32_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc,
               const int32_t* __restrict__ el, const int2* __restrict__ runs,
               const int* __restrict__ nruns, uint8_t* __restrict__ codes,
               int* __restrict__ flag, int2* __restrict__ side) {
  __shared__ int2 R[kRowRuns];
  const int t = threadIdx.x, lane = t & 31;
  const i64 p = order[blockIdx.x];
  const int nr = nruns[p];
  if (t < nr) R[t] = runs[p * kRowRuns + t];
  __syncthreads();
  uint8_t* tb = codes + p * kRowCodeCap;
  const int* h = reinterpret_cast<const int*>(tb);
  const int e0 = h[0], cnt = h[1];
  if (t >= cnt) return;
  auto slot = [&](int v) -> int {  // the runs ascend by first node: binary search
    if (nr == 0 || v < R[0].x) return -1;
    int lo = 0, hi = nr - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (R[mid].x <= v) lo = mid;
      else hi = mid - 1;
    }
    const int2 x = R[lo];
    return v < x.x + (x.y & 0xffff) ? (x.y >> 16) + (v - x.x) : -1;
  };
  uint8_t* blk = tb + reinterpret_cast<const uint16_t*>(h + 2)[t >> 5];
  const int e = e0 + blk[32 + lane];
  const int2 jk = edges[e];
  const int pb = inc_ptr[e], n = inc_ptr[e + 1] - pb;
  int miss = 0;
  const RingWalk rw = ring_walk_encode(jk.x, jk.y, pb, n, inc, el, [&](int step, int v) {
    const int sl = slot(v);
    miss |= sl < 0;
    blk[64 + (2 + step) * 32 + lane] = static_cast<uint8_t>(sl);
  });
  const int sj = slot(jk.x), sk = slot(jk.y);
  if (sj < 0 || sk < 0) {  // cannot happen for a plan built from this edge list
    atomicOr(flag, 1);
    return;
  }
  blk[64 + lane] = static_cast<uint8_t>(sj);
  blk[64 + 32 + lane] = static_cast<uint8_t>(sk);
  if (rw.fail || miss) {
    blk[64 + 64 + lane] = static_cast<uint8_t>(sk);  // m_0 := k, no ring steps
    blk[lane] = 0;
    atomicOr(flag, rw.fail | (miss ? 64 : 0));
    const int q = atomicAdd(flag + 1, 1);
    if (q < kSideCap) side[q] = make_int2(e, e);
    return;
  }
  blk[lane] = static_cast<uint8_t>(n | (rw.sign < 0 ? 32 : 0) | (rw.closed ? 128 : 0));
}

// meta[f] = {code offset (32 B units), code bytes, runs, provisional index}
// for the tiles in ascending e0 order
// (+ the plan's per-step stream sizes in sums[0..2]: code bytes, node-table
// fill bytes, metadata + run bytes -- the element loop's design bytes)
__global__ void k_rt_meta(const int* __restrict__ order, const int* __restrict__ nruns,
                          const int* __restrict__ bytes, const int2* __restrict__ runs, i64 ntiles,
                          int4* __restrict__ meta, unsigned long long* __restrict__ sums) {
  const i64 f = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long cb = 0, fb = 0, mb = 0;
  if (f < ntiles) {
    const int p = order[f];
    meta[f] = make_int4(p * (kRowCodeCap / 32), bytes[p], nruns[p], p);
    cb = static_cast<unsigned long long>(bytes[p]);
    for (int r = 0; r < nruns[p]; ++r)
      fb += 24ull * static_cast<unsigned long long>(runs[static_cast<i64>(p) * kRowRuns + r].y & 0xffff);
    mb = 16ull + 8ull * static_cast<unsigned long long>(nruns[p]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    cb += __shfl_xor_sync(0xffffffffu, cb, o);
    fb += __shfl_xor_sync(0xffffffffu, fb, o);
    mb += __shfl_xor_sync(0xffffffffu, mb, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(sums, cb);
    atomicAdd(sums + 1, fb);
    atomicAdd(sums + 2, mb);
  }
}

__global__ void k_rt_cand(i64 ne, i64 n, int ct, int2* __restrict__ cand) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const i64 e0 = i * ct;
  cand[i] = make_int2(static_cast<int>(e0), static_cast<int>(ne - e0 < ct ? ne - e0 : ct));
}

// boundary segments with positions = edge ids
__global__ void k_rt_bseg_fill(const u64* __restrict__ b, i64 n, const u32* __restrict__ idx,
                               const int2* __restrict__ edges, int4* __restrict__ seg,
                               u32* __restrict__ start) {
  const i64 q = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  if (q == n - 1) start[idx[n]] = static_cast<u32>(n);
  if (idx[q + 1] == idx[q]) return;  // not a segment start
  const int e = static_cast<int>(b[q] >> 32);
  const int2 jk = edges[e];
  seg[idx[q]] = make_int4(e, jk.x, jk.y, e);
  start[idx[q]] = static_cast<u32>(q);
}

__global__ void k_rt_bflag(const u64* __restrict__ b, i64 n, u32* __restrict__ flag) {
  const i64 q = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < n) flag[q] = (q == 0 || (b[q] >> 32) != (b[q - 1] >> 32)) ? 1u : 0u;
}

size_t rt_block(const dm_ctx* c) { return static_cast<size_t>(16 * c->ne) + (64u << 20); }

}  // namespace

int try_row_plan(dm_ctx* c) {
  c->row_plan = false;
  if (c->dim != 3 || c->ne == 0) return DM_OK;
  if (const char* ev = std::getenv("DUALMESH_ROW_PLAN"))
    if (std::atoi(ev) == 0) return DM_OK;
  ArenaScope scratch(c->arena);
  PlanClock clk(c);
  const i64 ne = c->ne;
  int ct = kRowTile;  // candidate tile (edges), env DUALMESH_ROW_CAND
  if (const char* cs = std::getenv("DUALMESH_ROW_CAND")) ct = std::max(2, std::min(kRowTile, std::atoi(cs) & ~1));
  const i64 n0 = (ne + ct - 1) / ct;
  // provisional tiles: the level-0 ranges p < n0, then the halves of tiles
  // that did not fit, appended level by level (about 2 % of tiles at C5)
  double split_max = 1.25;  // tiles after splitting / (ne / kRowTile), env DUALMESH_ROW_SPLIT_MAX
  if (const char* sm = std::getenv("DUALMESH_ROW_SPLIT_MAX")) split_max = std::atof(sm);
  int by_len = 1;  // lane order: ring length first; env DUALMESH_ROW_BYLEN=0: direction only
  if (const char* bl = std::getenv("DUALMESH_ROW_BYLEN")) by_len = std::atoi(bl);
  const i64 cap = static_cast<i64>(split_max * static_cast<double>(n0)) + 1024;
  ScratchBuf<int2> cand(c->arena, rt_block(c));
  ScratchBuf<uint8_t> bad(c->arena, rt_block(c));
  ScratchBuf<int> nruns(c->arena, rt_block(c)), bytes(c->arena, rt_block(c));
  DM_CK(c, cand.ensure(n0));
  DM_CK(c, bad.ensure(cap));
  DM_CK(c, nruns.ensure(cap));
  DM_CK(c, bytes.ensure(cap));
  DM_CK(c, c->rt_runs.ensure(static_cast<size_t>(cap * kRowRuns)));
  DM_CK(c, c->rcodes.ensure(static_cast<size_t>(cap) * kRowCodeCap));
  DM_CK(c, c->flag.ensure(4));
  DM_CK(c, cudaMemsetAsync(c->flag.p, 0, 2 * sizeof(int), c->stream));
  DM_LAUNCH(c, k_rt_cand, grid_for(n0, 256), 256, 0, ne, n0, ct, cand.p);
  // provisional tiles: p < n0 the level-0 ranges (by formula, as k_rt_cand
  // writes them), then the halves of tiles that did not fit (host list)
  std::vector<int2> extra;
  auto tile_of = [&](i64 p) -> int2 {
    if (p >= n0) return extra[static_cast<size_t>(p - n0)];
    const i64 e0 = p * ct;
    return make_int2(static_cast<int>(e0), static_cast<int>(ne - e0 < ct ? ne - e0 : ct));
  };
  clk.mark("row tiles: setup");
  std::vector<uint8_t> hb;
  std::vector<int> child(static_cast<size_t>(n0), -1);  // first of the two halves
  std::vector<int> split0;                               // split level-0 tiles, ascending
  i64 base = 0, np = n0;
  for (int level = 0; np > 0; ++level) {
    if (level > 0)
      DM_CK(c, cudaMemcpyAsync(cand.p, extra.data() + (base - n0), np * sizeof(int2),
                               cudaMemcpyHostToDevice, c->stream));
    DM_LAUNCH(c, k_rt_build, static_cast<unsigned>(np), kRTThreads, 0, cand.p,
              static_cast<int>(base), c->edges.p, c->os.p, c->inc_ptr.p, c->inc.p, c->elems.p,
              bad.p, c->rt_runs.p, nruns.p, bytes.p, c->rcodes.p, by_len);
    hb.resize(static_cast<size_t>(np));
    DM_CK(c, cudaMemcpyAsync(hb.data(), bad.p + base, np, cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    clk.mark(level == 0 ? "row tiles: build level 0" : "row tiles: build level >0");
    i64 nbad = 0;
    const i64 next = base + np;
    if (static_cast<i64>(child.size()) < next) child.resize(static_cast<size_t>(next), -1);
    // the flagged tiles (mostly none: the scan skips eight zero flags at a time)
    const uint8_t* q = hb.data();
    const uint8_t* const end = q + np;
    for (;;) {
      while (q + 8 <= end) {
        std::uint64_t w;
        std::memcpy(&w, q, 8);
        if (w) break;
        q += 8;
      }
      while (q < end && !*q) ++q;
      if (q >= end) break;
      const i64 i = q - hb.data();
      ++q;
      ++nbad;
      const int2 tl = tile_of(base + i);
      if (tl.y < 2) return DM_OK;  // one edge does not fit: Morton plan
      const int h = tl.y >= 4 ? (tl.y / 2 + 1) & ~1 : 1;  // even splits keep e0 even
      child[static_cast<size_t>(base + i)] = static_cast<int>(n0 + static_cast<i64>(extra.size()));
      if (level == 0) split0.push_back(static_cast<int>(i));
      extra.push_back(make_int2(tl.x, h));
      extra.push_back(make_int2(tl.x + h, tl.y - h));
    }
    if (level == 0 && static_cast<double>(nbad) > (split_max - 1.0) * static_cast<double>(n0))
      return DM_OK;  // tables too large: Morton plan
    if (n0 + static_cast<i64>(extra.size()) > cap) return DM_OK;  // (cap: the split budget below)
    base = next;
    np = n0 + static_cast<i64>(extra.size()) - next;
    DM_CK(c, cand.ensure(np > 0 ? np : 1));
  }
  clk.mark("row tiles: build + split");
  child.resize(static_cast<size_t>(n0) + extra.size(), -1);
  // final order: every level-0 tile, or its halves in place, depth first;
  // runs of unsplit level-0 tiles are written as ranges, only the split
  // tiles (their ids are ascending in split0) walk the stack
  std::vector<int> order(static_cast<size_t>(n0) + extra.size());
  size_t w = 0;
  std::vector<int> stack;
  i64 prev = 0;
  auto expand = [&](int root) {
    stack.push_back(root);
    while (!stack.empty()) {
      const int pv = stack.back();
      stack.pop_back();
      const int ch = child[static_cast<size_t>(pv)];
      if (ch < 0) {
        order[w++] = pv;
      } else {
        stack.push_back(ch + 1);
        stack.push_back(ch);
      }
    }
  };
  for (const int sp : split0) {
    std::iota(order.begin() + static_cast<std::ptrdiff_t>(w),
              order.begin() + static_cast<std::ptrdiff_t>(w + (sp - prev)), static_cast<int>(prev));
    w += static_cast<size_t>(sp - prev);
    expand(sp);
    prev = sp + 1;
  }
  std::iota(order.begin() + static_cast<std::ptrdiff_t>(w),
            order.begin() + static_cast<std::ptrdiff_t>(w + (n0 - prev)), static_cast<int>(prev));
  w += static_cast<size_t>(n0 - prev);
  order.resize(w);
  const i64 nt = static_cast<i64>(order.size());
  clk.mark("row tiles: host order");
  if (static_cast<double>(nt) > split_max * static_cast<double>(n0)) return DM_OK;
  ScratchBuf<int> dorder(c->arena, rt_block(c));
  DM_CK(c, dorder.ensure(nt));
  DM_CK(c, cudaMemcpyAsync(dorder.p, order.data(), nt * sizeof(int), cudaMemcpyHostToDevice,
                           c->stream));
  DM_CK(c, c->rt_meta.ensure(static_cast<size_t>(nt)));
  DM_CK(c, c->side.ensure(kSideCap));
  DM_CK(c, cudaMemsetAsync(c->flag.p, 0, 2 * sizeof(int), c->stream));
  clk.mark("row tiles: order upload");
  DM_LAUNCH(c, k_rt_codes, static_cast<unsigned>(nt), kRowTile, 0, dorder.p, c->edges.p,
            c->inc_ptr.p, c->inc.p, c->elems.p, c->rt_runs.p, nruns.p, c->rcodes.p, c->flag.p,
            c->side.p);
  ScratchBuf<unsigned long long> sums(c->arena, rt_block(c));
  DM_CK(c, sums.ensure(3));
  DM_CK(c, cudaMemsetAsync(sums.p, 0, 3 * sizeof(unsigned long long), c->stream));
  DM_LAUNCH(c, k_rt_meta, grid_for(nt, 256), 256, 0, dorder.p, nruns.p, bytes.p, c->rt_runs.p, nt,
            c->rt_meta.p, sums.p);
  DM_CK(c, cudaMemcpyAsync(c->rt_bytes, sums.p, sizeof(c->rt_bytes), cudaMemcpyDeviceToHost,
                           c->stream));
  {
    int fl[2] = {0, 0};
    DM_CK(c, cudaMemcpyAsync(fl, c->flag.p, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    if ((fl[0] & 1) || fl[1] > kSideCap) return DM_OK;  // not for this plan: Morton tiles
    c->ring_fail = fl[0];  // reasons the side list exists (informational)
    c->n_side = fl[1];
  }
  clk.mark("row tiles: codes");
  // boundary pass lists: positions are edge ids
  const i64 nb = c->n_bedge;
  DM_CK(c, c->bedge_p.ensure(nb > 0 ? nb : 1));
  c->n_bseg = 0;
  if (nb > 0) {
    DM_CK(c, cudaMemcpyAsync(c->bedge_p.p, c->bedge.p, nb * sizeof(u64), cudaMemcpyDeviceToDevice,
                             c->stream));
    ScratchBuf<u32> idx(c->arena, rt_block(c));
    DM_CK(c, idx.ensure(nb + 1));
    DM_LAUNCH(c, k_rt_bflag, grid_for(nb, 256), 256, 0, c->bedge_p.p, nb, idx.p);
    int st = scan_exclusive(c, idx.p, idx.p, nb);
    if (st) return st;
    u32 ns = 0;
    DM_CK(c, cudaMemcpyAsync(&ns, idx.p + nb, sizeof(u32), cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    DM_CK(c, c->bseg.ensure(ns));
    DM_CK(c, c->bseg_start.ensure(ns + 1));
    DM_LAUNCH(c, k_rt_bseg_fill, grid_for(nb, 256), 256, 0, c->bedge_p.p, nb, idx.p, c->edges.p,
              c->bseg.p, c->bseg_start.p);
    c->n_bseg = ns;
  }
  clk.mark("row tiles: meta + boundary lists");
  if (const char* ck = std::getenv("DUALMESH_PLAN_CHECK")) {  // debugging aid: host audit
    if (std::atoi(ck) == 1) {
      std::vector<int4> hm(static_cast<size_t>(nt));
      std::vector<int2> hr((static_cast<size_t>(n0) + extra.size()) * kRowRuns);
      DM_CK(c, cudaMemcpy(hm.data(), c->rt_meta.p, nt * sizeof(int4), cudaMemcpyDeviceToHost));
      DM_CK(c, cudaMemcpy(hr.data(), c->rt_runs.p, hr.size() * sizeof(int2),
                          cudaMemcpyDeviceToHost));
      std::vector<uint8_t> blk(kRowCodeCap);
      i64 next_e = 0;
      for (i64 f = 0; f < nt; ++f) {
        const int4 m = hm[static_cast<size_t>(f)];
        DM_CK(c, cudaMemcpy(blk.data(), c->rcodes.p + 32 * static_cast<i64>(m.x), kRowCodeCap,
                            cudaMemcpyDeviceToHost));
        const int* h = reinterpret_cast<const int*>(blk.data());
        const uint16_t* wo = reinterpret_cast<const uint16_t*>(h + 2);
        int slots = 0;
        bool ok = m.y > 0 && m.y <= kRowCodeCap && m.z > 0 && m.z <= kRowRuns && h[0] == next_e &&
                  h[1] > 0 && h[1] <= kRowTile && wo[7] == m.y;
        for (int r = 0; r < m.z && ok; ++r) {
          const int2 x = hr[static_cast<size_t>(m.w) * kRowRuns + r];
          ok = (x.x & 1) == 0 && (x.y & 0xffff) > 0 && (x.y >> 16) == slots;
          slots += x.y & 0xffff;
        }
        ok = ok && slots <= kRowSlots;
        if (!ok) {
          std::fprintf(stderr, "[plan check] tile %lld: meta {%d %d %d %d} header e0 %d cnt %d "
                       "(expected e0 %lld) slots %d\n", static_cast<long long>(f), m.x, m.y,
                       m.z, m.w, h[0], h[1], static_cast<long long>(next_e), slots);
          return fail(c, DM_ERR_CUDA, "row plan audit failed");
        }
        next_e = h[0] + h[1];
      }
      if (next_e != ne) return fail(c, DM_ERR_CUDA, "row plan audit: edges not covered");
      std::fprintf(stderr, "[plan check] %lld row tiles ok\n", static_cast<long long>(nt));
    }
  }
  c->rt_ntiles = nt;
  c->row_plan = true;
  return DM_OK;
}

}  // namespace dm
