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
//   * the lanes of the tile take its edges in direction-major order (sorted
//     by the edge's index inside its origin row, then by origin): for a
//     structured grid the 32 lanes of a warp hold the same edge direction of
//     32 consecutive origins, so a ring step reads 32 consecutive table slots
//     (no bank conflicts, uniform ring length in the warp);
//   * the rows are staged in shared memory and leave as two TMA bulk stores
//     per tile (navs rows, s terms) -- contiguous, no per-lane stores.
// The plan is used when the tiles split little (<= 25 % more tiles than
// ne / kRowTile); otherwise the Morton plan of rings.cu.
//
// Code block of a tile (32-byte units, contiguous):
//   [tile header 32 B: e0 (i32), cnt (i32), eight u16 byte offsets of the
//    warp blocks from the tile's code start]
//   per warp w: [32 B: n | sign << 5 | closed << 7 per lane]
//               [32 B: edge offset e - e0 per lane]
//               [S_w steps x 32 B: slot(j), slot(k), slot(m_0), slot(m_1) ..]
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "dm_internal.cuh"
#include "ring_encode.cuh"

namespace dm {
namespace {

constexpr int kRTThreads = 256;   // plan kernels: one CTA per tile
constexpr int kRTHash = 4096;
constexpr int kRTUniqCap = 512;

// infeasibility bits of a candidate tile
constexpr int kRTTooManyNodes = 1;
constexpr int kRTTooManyRuns = 2;
constexpr int kRTTooManyCodes = 4;
constexpr int kRTRingTooLong = 8;

struct RTShared {
  int hs[kRTHash];
  int uq[kRTUniqCap];
  unsigned key[kRTThreads];
  int n_uniq;
  int nruns, nslots;
  int2 runs[kRowRuns];
  int wmax[8];
};

__device__ __forceinline__ void bitonic_sort_int(int* a, int P, int t) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = t; i < P; i += kRTThreads) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int x = a[i], y = a[ixj];
          if ((x > y) == ((i & k) == 0)) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
}

__device__ __forceinline__ void bitonic_sort_u32(unsigned* a, int t) {
  for (int k = 2; k <= kRTThreads; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      const int i = t, ixj = i ^ j;
      if (ixj > i) {
        const unsigned x = a[i], y = a[ixj];
        if ((x > y) == ((i & k) == 0)) {
          a[i] = y;
          a[ixj] = x;
        }
      }
      __syncthreads();
    }
}

// One CTA per candidate tile {e0, cnt}: the node set, its runs, the
// direction-major lane order and the code size.  BUILD: also writes the runs,
// each edge's tile and lane position and the block sizes.
template <bool BUILD>
__global__ void __launch_bounds__(kRTThreads)
    k_rt_tile(const int2* __restrict__ cand, const int2* __restrict__ edges,
              const u32* __restrict__ os, const int32_t* __restrict__ inc_ptr,
              const int32_t* __restrict__ inc, const int32_t* __restrict__ el,
              uint8_t* __restrict__ bad, int2* __restrict__ runs_out, int32_t* __restrict__ tile_of,
              uint8_t* __restrict__ pos, u32* __restrict__ wsz, int* __restrict__ nruns_out) {
  __shared__ RTShared S;
  const int t = threadIdx.x, f = blockIdx.x;
  const int2 cd = cand[f];
  const int e0 = cd.x, cnt = cd.y;
  for (int i = t; i < kRTHash; i += kRTThreads) S.hs[i] = -1;
  if (t == 0) S.n_uniq = 0;
  if (t < 8) S.wmax[t] = 0;
  __syncthreads();
  auto insert = [&](int v) {
    unsigned h = (static_cast<unsigned>(v) * 2654435761u) >> 20;  // 12 bits
    for (int probe = 0; probe < kRTHash; ++probe, h = (h + 1) & (kRTHash - 1)) {
      const int old = atomicCAS(&S.hs[h], -1, v);
      if (old == -1) {
        const int p = atomicAdd(&S.n_uniq, 1);
        if (p < kRTUniqCap) S.uq[p] = v;
        return;
      }
      if (old == v) return;
    }
  };
  int n_inc = 0;
  unsigned key = 0xffffffffu;
  if (t < cnt) {
    const int e = e0 + t;
    const int2 jk = edges[e];
    insert(jk.x);
    insert(jk.y);
    const int pb = inc_ptr[e];
    n_inc = inc_ptr[e + 1] - pb;
    for (int q = 0; q < n_inc; ++q) {
      const int4 v = reinterpret_cast<const int4*>(el)[inc[pb + q]];
      insert(v.x);
      insert(v.y);
      insert(v.z);
      insert(v.w);
    }
    // direction-major: index of the edge inside its origin row, then origin
    key = (static_cast<unsigned>(e - static_cast<int>(os[jk.x])) << 8) | static_cast<unsigned>(t);
  }
  S.key[t] = key;
  __syncthreads();
  const int nu = S.n_uniq;
  int badbits = 0;
  if (nu > kRTUniqCap) badbits |= kRTTooManyNodes;
  if (__syncthreads_or(t < cnt && n_inc > kRingMax)) badbits |= kRTRingTooLong;
  if (badbits) {
    if (t == 0) bad[f] = static_cast<uint8_t>(badbits);
    return;
  }
  int P = 2;
  while (P < nu) P <<= 1;
  for (int i = nu + t; i < P; i += kRTThreads) S.uq[i] = 0x7fffffff;
  __syncthreads();
  bitonic_sort_int(S.uq, P, t);
  // runs of the sorted node ids, each copied as an even-aligned range
  // [2*floor(a/2), 2*ceil((b+1)/2)); a node within one past the current range
  // extends it (at most one padding record) instead of opening a run
  if (t == 0) {
    int nr = 0, slots = 0, cs = 0, ce = 0;
    bool ok = true;
    for (int i = 0; i < nu; ++i) {
      const int v = S.uq[i];
      if (i > 0 && v <= ce + 1) {
        ce = max(ce, (v + 2) & ~1);
        continue;
      }
      if (i > 0) {
        if (nr < kRowRuns) S.runs[nr] = make_int2(cs, (ce - cs) | slots << 16);
        ++nr;
        slots += ce - cs;
      }
      cs = v & ~1;
      ce = (v + 2) & ~1;
    }
    if (nu > 0) {
      if (nr < kRowRuns) S.runs[nr] = make_int2(cs, (ce - cs) | slots << 16);
      ++nr;
      slots += ce - cs;
    }
    ok = nr <= kRowRuns && slots <= kRowSlots;
    S.nruns = nr;
    S.nslots = ok ? slots : -1;
  }
  // lane order
  bitonic_sort_u32(S.key, t);
  const unsigned kq = S.key[t];
  int ring = 0;
  if (t < cnt) {
    const int q = static_cast<int>(kq & 0xffu);
    const int e = e0 + q;
    ring = inc_ptr[e + 1] - inc_ptr[e];
    atomicMax(&S.wmax[t >> 5], ring + 3);
    if (BUILD) {
      tile_of[e] = f;
      pos[e] = static_cast<uint8_t>(t);
    }
  }
  __syncthreads();
  if (S.nruns > kRowRuns) badbits |= kRTTooManyRuns;
  if (S.nslots < 0 && S.nruns <= kRowRuns) badbits |= kRTTooManyNodes;
  int units = 1;  // tile header
  for (int w = 0; w < kRowTile / 32; ++w)
    if (w * 32 < cnt) units += 2 + S.wmax[w];
  if (32 * units > kRowCodeCap) badbits |= kRTTooManyCodes;
  if (t == 0) bad[f] = static_cast<uint8_t>(badbits);
  if (!BUILD) return;
  if (t < kRowRuns) runs_out[static_cast<i64>(f) * kRowRuns + t] = t < S.nruns ? S.runs[t] : make_int2(0, 0);
  if (t < 8) wsz[8 * static_cast<i64>(f) + t] = t == 0 ? 1u : (32 * (t - 1) < cnt ? 2u + S.wmax[t - 1] : 0u);
  if (t == 0) nruns_out[f] = S.nruns;
}

// Ring codes of every edge (one thread per edge).
__global__ void k_rt_codes(const int2* __restrict__ tiles, const int2* __restrict__ edges,
                           const int32_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc,
                           const int32_t* __restrict__ el, const int32_t* __restrict__ tile_of,
                           const uint8_t* __restrict__ pos, const int2* __restrict__ runs,
                           const int* __restrict__ nruns, const u32* __restrict__ woff, i64 ne,
                           uint8_t* __restrict__ codes, int* __restrict__ flag) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int f = tile_of[e];
  const int p = pos[e];
  const int lane = p & 31, w = p >> 5;
  const int2* R = runs + static_cast<i64>(f) * kRowRuns;
  const int nr = nruns[f];
  auto slot = [&](int v) -> int {
    for (int r = 0; r < nr; ++r) {
      const int2 x = R[r];
      if (v >= x.x && v < x.x + (x.y & 0xffff)) return (x.y >> 16) + (v - x.x);
    }
    return -1;
  };
  const i64 tbase = 32 * static_cast<i64>(woff[8 * static_cast<i64>(f)]);
  uint8_t* blk = codes + 32 * static_cast<i64>(woff[8 * static_cast<i64>(f) + 1 + w]);
  const int2 jk = edges[e];
  const int pb = inc_ptr[e], n = inc_ptr[e + 1] - pb;
  int miss = 0;
  const RingWalk r = ring_walk_encode(jk.x, jk.y, pb, n, inc, el, [&](int step, int v) {
    const int s = slot(v);
    miss |= s < 0;
    blk[64 + (2 + step) * 32 + lane] = static_cast<uint8_t>(s);
  });
  if (r.fail || miss) {
    atomicOr(flag, r.fail | (miss ? 1 : 0));
    return;
  }
  const int sj = slot(jk.x), sk = slot(jk.y);
  blk[64 + lane] = static_cast<uint8_t>(sj);
  blk[64 + 32 + lane] = static_cast<uint8_t>(sk);
  blk[lane] = static_cast<uint8_t>(n | (r.sign < 0 ? 32 : 0) | (r.closed ? 128 : 0));
  blk[32 + lane] = static_cast<uint8_t>(e - tiles[f].x);
  if (p == 0) {  // tile header
    int* h = reinterpret_cast<int*>(codes + tbase);
    h[0] = tiles[f].x;
    h[1] = tiles[f].y;
    uint16_t* wo = reinterpret_cast<uint16_t*>(h + 2);
    for (int q = 0; q < 8; ++q)
      wo[q] = static_cast<uint16_t>(32 * (woff[8 * static_cast<i64>(f) + 1 + q] -
                                          woff[8 * static_cast<i64>(f)]));
  }
}

__global__ void k_rt_meta(const u32* __restrict__ woff, const int* __restrict__ nruns, i64 ntiles,
                          int4* __restrict__ meta) {
  const i64 f = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= ntiles) return;
  const u32 a = woff[8 * f], b = woff[8 * f + 8];
  meta[f] = make_int4(static_cast<int>(a), static_cast<int>(32 * (b - a)), nruns[f], 0);
}

__global__ void k_rt_cand(i64 ne, i64 n, int2* __restrict__ cand) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const i64 e0 = i * kRowTile;
  cand[i] = make_int2(static_cast<int>(e0), static_cast<int>(ne - e0 < kRowTile ? ne - e0 : kRowTile));
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
  if (const char* e = std::getenv("DUALMESH_ROW_PLAN"))
    if (std::atoi(e) == 0) return DM_OK;
  ArenaScope scratch(c->arena);
  const i64 ne = c->ne;
  const i64 n0 = (ne + kRowTile - 1) / kRowTile;
  ScratchBuf<int2> cand(c->arena, rt_block(c));
  ScratchBuf<uint8_t> bad(c->arena, rt_block(c));
  DM_CK(c, cand.ensure(n0));
  DM_CK(c, bad.ensure(n0));
  DM_LAUNCH(c, k_rt_cand, grid_for(n0, 256), 256, 0, ne, n0, cand.p);
  // level 0: fixed kRowTile ranges; infeasible tiles are split in halves
  std::vector<int2> fin, pend(static_cast<size_t>(n0));
  DM_CK(c, cudaMemcpyAsync(pend.data(), cand.p, n0 * sizeof(int2), cudaMemcpyDeviceToHost,
                           c->stream));
  std::vector<uint8_t> hb;
  bool first = true;
  while (!pend.empty()) {
    const i64 np = static_cast<i64>(pend.size());
    DM_CK(c, cand.ensure(np));
    DM_CK(c, bad.ensure(np));
    if (!first)
      DM_CK(c, cudaMemcpyAsync(cand.p, pend.data(), np * sizeof(int2), cudaMemcpyHostToDevice,
                               c->stream));
    DM_LAUNCH(c, k_rt_tile<false>, static_cast<unsigned>(np), kRTThreads, 0, cand.p, c->edges.p,
              c->os.p, c->inc_ptr.p, c->inc.p, c->elems.p, bad.p, nullptr, nullptr, nullptr,
              nullptr, nullptr);
    hb.resize(static_cast<size_t>(np));
    DM_CK(c, cudaMemcpyAsync(hb.data(), bad.p, np, cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    std::vector<int2> next;
    i64 nbad = 0;
    for (i64 i = 0; i < np; ++i) {
      const int2 t = pend[static_cast<size_t>(i)];
      if (!hb[static_cast<size_t>(i)]) {
        fin.push_back(t);
        continue;
      }
      ++nbad;
      if ((hb[static_cast<size_t>(i)] & kRTRingTooLong) || t.y < 2) return DM_OK;  // Morton plan
      const int h = t.y >= 4 ? (t.y / 2 + 1) & ~1 : 1;  // even splits keep e0 even
      next.push_back(make_int2(t.x, h));
      next.push_back(make_int2(t.x + h, t.y - h));
    }
    if (first && nbad * 4 > n0) return DM_OK;  // tables too large: Morton plan
    first = false;
    pend.swap(next);
  }
  const i64 nt = static_cast<i64>(fin.size());
  if (nt * 4 > n0 * 5) return DM_OK;
  std::sort(fin.begin(), fin.end(), [](const int2& a, const int2& b) { return a.x < b.x; });
  ScratchBuf<int2> tiles(c->arena, rt_block(c));
  ScratchBuf<int32_t> tile_of(c->arena, rt_block(c));
  ScratchBuf<uint8_t> pos(c->arena, rt_block(c));
  ScratchBuf<u32> woff(c->arena, rt_block(c));
  ScratchBuf<int> nruns(c->arena, rt_block(c));
  DM_CK(c, tiles.ensure(nt));
  DM_CK(c, tile_of.ensure(ne));
  DM_CK(c, pos.ensure(ne));
  DM_CK(c, woff.ensure(8 * nt + 1));
  DM_CK(c, nruns.ensure(nt));
  DM_CK(c, bad.ensure(nt));
  DM_CK(c, c->rt_runs.ensure(static_cast<size_t>(nt * kRowRuns)));
  DM_CK(c, c->rt_meta.ensure(static_cast<size_t>(nt)));
  DM_CK(c, cudaMemcpyAsync(tiles.p, fin.data(), nt * sizeof(int2), cudaMemcpyHostToDevice,
                           c->stream));
  DM_LAUNCH(c, k_rt_tile<true>, static_cast<unsigned>(nt), kRTThreads, 0, tiles.p, c->edges.p,
            c->os.p, c->inc_ptr.p, c->inc.p, c->elems.p, bad.p, c->rt_runs.p, tile_of.p, pos.p,
            woff.p, nruns.p);
  int st = scan_exclusive(c, woff.p, woff.p, 8 * nt);
  if (st) return st;
  u32 units = 0;
  DM_CK(c, cudaMemcpyAsync(&units, woff.p + 8 * nt, sizeof(u32), cudaMemcpyDeviceToHost,
                           c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  const size_t nbytes = 32 * static_cast<size_t>(units);
  DM_CK(c, c->rcodes.ensure(nbytes + 16));
  DM_CK(c, cudaMemsetAsync(c->rcodes.p, 0, nbytes + 16, c->stream));
  DM_CK(c, c->flag.ensure(4));
  DM_CK(c, cudaMemsetAsync(c->flag.p, 0, sizeof(int), c->stream));
  DM_LAUNCH(c, k_rt_codes, grid_for(ne, 128), 128, 0, tiles.p, c->edges.p, c->inc_ptr.p, c->inc.p,
            c->elems.p, tile_of.p, pos.p, c->rt_runs.p, nruns.p, woff.p, ne, c->rcodes.p,
            c->flag.p);
  DM_LAUNCH(c, k_rt_meta, grid_for(nt, 256), 256, 0, woff.p, nruns.p, nt, c->rt_meta.p);
  int fl = 0;
  DM_CK(c, cudaMemcpyAsync(&fl, c->flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  if (fl) {  // a fan the walk cannot encode: the Morton plan reports it
    c->ring_fail = fl;
    return DM_OK;
  }
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
    st = scan_exclusive(c, idx.p, idx.p, nb);
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
  c->rt_ntiles = nt;
  c->row_plan = true;
  return DM_OK;
}

}  // namespace dm
