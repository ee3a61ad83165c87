// rings.cu -- connectivity-only structures of the fast GATHER path (3D).
//
// For an interior edge (j,k) the incident tetrahedra form a closed ring
// around it: element i has nodes {j, k, m_i, m_(i+1)}.  For a boundary edge
// the ring is an open chain.  The dual-free term of element i is
//   2 n_j^E = +-cross(m_i - x_k, m_(i+1) - x_k)
// (the face opposite j is {k, m_i, m_(i+1)}; the sign is the parity of
// (k, m_i, m_(i+1)) against the outward vertex order of the reference,
// mesh.cpp:15,103-110), so walking the ring needs ONE new coordinate per
// incidence instead of three.
//
//   edge order : tiles are 256 consecutive positions p of a permutation
//                eperm[p] = e of the edges.  Origins are visited in Morton
//                (Z-curve) order of their coordinates and each origin's
//                edge range [os[j], os[j+1]) is appended whole, so a tile
//                covers a compact 3D block of origins whatever the node
//                numbering: its node table (origins plus a one-node halo)
//                is ~4x the origin count instead of ~13x for a strip of
//                consecutive origins, and randomly numbered meshes keep
//                the same locality.  navs go to navs[e].  For node
//                numberings without spatial locality the edge-volume terms
//                stay in position order, svals[p], and the volume kernel
//                walks nodes in Morton rank order with each rank's incoming
//                (rin_ptr/rin_list) and outgoing (rpstart) edges as
//                positions -- the same per-node fold order as the edge-id
//                kernel, so the same bits.
//   coordinates: a copy of the coordinates in Morton rank order (mxy 16 B,
//                mz 8 B per node), refreshed with every coordinate update,
//                so a tile's table is a few contiguous rank ranges.
//   tile nodes : per tile, the sorted unique Morton ranks of every node the
//                tile touches (j, k, ring nodes), at a fixed stride of
//                kTileNodeCap, count in tnode_cnt[tile].
//   ring codes : per edge, n+3 16-bit words
//                  [slot(j) | s<<15, slot(k) | n<<11, slot(m_0) | b<<15,
//                   slot(m_1), ..., slot(m_n)]  (slots into the tile list;
//                                                b: edge has boundary facets)
//                or, when every tile table holds <= 256 nodes, n+3 bytes of
//                slots plus a per-lane header byte n | s<<5 | b<<6 at the
//                start of the warp block (half the code bytes to stream)
//                stored lane-transposed per warp of 32 consecutive positions:
//                the warp block holds S_w = max(n+3) steps x 32 lanes, entry
//                (step, lane) at wstart[w] + step*32 + lane, so the 32 lanes
//                of a ring step read 64 contiguous bytes (one wavefront).
//                s is the common orientation of all terms of the edge:
//                around a consistently oriented ring every term has the same
//                parity, so the sign is applied once to the sum
//                (sum(-c_i) == -sum(c_i) exactly in IEEE arithmetic).
//   boundary   : the (edge, facet) list re-keyed by position, (p << 32 |
//                facet), sorted, with per-tile slices.
// Built once per topology (the Morton order uses the coordinates present at
// build time; later coordinates only change locality, never results).  Any
// tile with more than kTileNodeCap nodes, an edge with more than kRingMax
// incidences or a non-manifold fan (the walk does not consume every incident
// element) sets ring_ok = false and the GATHER path falls back to the
// bit-exact row-table kernel.

#include <cmath>
#include <cstdlib>
#include <vector>

#include "dm_internal.cuh"
#include "ring_encode.cuh"

#include <chrono>
#include <cstdio>

namespace dm {
namespace {

constexpr int kHash = 4096;  // open-addressing set of the tile's node ranks
static_assert(kTileNodeCap <= kHash / 2, "hash set at most half full");

// Per tile: the sorted unique Morton ranks of every node its edges touch (j,
// k and the ring nodes).  Candidates go through a shared-memory hash set
// (linear probing, atomicCAS), the unique ones are bitonic-sorted.  Tiles
// with more than kTileNodeCap nodes set flag bit 2 and keep count 0.
__global__ void __launch_bounds__(kTileEdges)
    k_tile_nodes(const int2* __restrict__ edges, const int32_t* __restrict__ eperm,
                 const int32_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc,
                 const int32_t* __restrict__ el, const int32_t* __restrict__ rank, i64 ne,
                 int32_t* __restrict__ tnodes, u32* __restrict__ tcnt, int* __restrict__ flag) {
  __shared__ int hs[kHash];
  __shared__ int uq[2 * kTileNodeCap];
  __shared__ int s_n;
  const int t = threadIdx.x;
  for (int i = t; i < kHash; i += kTileEdges) hs[i] = -1;
  if (t == 0) s_n = 0;
  __syncthreads();
  auto insert = [&](int v) {
    unsigned h = (static_cast<unsigned>(v) * 2654435761u) >> 20;  // 12 bits
    for (int probe = 0; probe < kHash; ++probe, h = (h + 1) & (kHash - 1)) {
      const int old = atomicCAS(&hs[h], -1, v);
      if (old == -1) {
        const int pos = atomicAdd(&s_n, 1);
        if (pos < 2 * kTileNodeCap) uq[pos] = v;
        return;
      }
      if (old == v) return;
    }
  };
  const i64 p = static_cast<i64>(blockIdx.x) * kTileEdges + t;
  if (p < ne) {
    const int e = eperm[p];
    const int2 jk = edges[e];
    insert(rank[jk.x]);
    insert(rank[jk.y]);
    const int nq = inc_ptr[e + 1] - inc_ptr[e];  // side-list edges need only j, k
    for (int q = inc_ptr[e]; q < (nq > kRingMax ? inc_ptr[e] : inc_ptr[e + 1]); ++q) {
      const int4 v = reinterpret_cast<const int4*>(el)[inc[q]];
      const int vs[4] = {v.x, v.y, v.z, v.w};
      for (int a = 0; a < 4; ++a)
        if (vs[a] != jk.x && vs[a] != jk.y) insert(rank[vs[a]]);
    }
  }
  __syncthreads();
  const int n = s_n;
  if (t == 0) atomicMax(flag + 1, n);
  if (t == 0 && n > 256) atomicAdd(flag + 3, 1);  // tiles beyond an 8-bit table
  if (n > kTileNodeCap) {
    if (t == 0) atomicOr(flag, 2);
    return;
  }
  int P = 2;
  while (P < n) P <<= 1;
  for (int i = n + t; i < P; i += kTileEdges) uq[i] = 0x7fffffff;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = t; i < P; i += kTileEdges) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const int a = uq[i], b = uq[ixj];
          if ((a > b) == ((i & k) == 0)) {
            uq[i] = b;
            uq[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
  int32_t* out = tnodes + static_cast<i64>(blockIdx.x) * kTileNodeCap;
  for (int i = t; i < n; i += kTileEdges) out[i] = uq[i];
  if (t == 0) tcnt[blockIdx.x] = static_cast<u32>(n);
}

__device__ __forceinline__ int tslot(const int32_t* list, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (list[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <int W>
__global__ void k_ring_codes(const int2* __restrict__ edges, const int32_t* __restrict__ eperm,
                             const int32_t* __restrict__ inc_ptr,
                             const int32_t* __restrict__ inc, const int32_t* __restrict__ el,
                             const int32_t* __restrict__ rank, const uint8_t* __restrict__ bmark,
                             const int32_t* __restrict__ tnodes, const u32* __restrict__ tcnt,
                             const u32* __restrict__ wstart, i64 ne,
                             uint8_t* __restrict__ rcodes, int* __restrict__ flag,
                             int2* __restrict__ side) {
  const i64 p = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= ne) return;
  const int e = eperm[p];
  const i64 tile = p / kTileEdges;
  const int32_t* list = tnodes + tile * kTileNodeCap;
  const int nl = static_cast<int>(tcnt[tile]);
  const int2 jk = edges[e];
  const int j = jk.x, k = jk.y;
  const int pb = inc_ptr[e], n = inc_ptr[e + 1] - pb;
  // step s of this edge lives at out[s * 32]; W == 1: one byte per step
  // after a 32-byte header (n | sign << 5 | boundary << 6 | closed << 7 per lane)
  uint8_t* blk = rcodes + static_cast<i64>(wstart[p >> 5]) * 32;
  uint16_t* out = reinterpret_cast<uint16_t*>(blk) + (p & 31);
  uint8_t* out8 = blk + 32 + (p & 31);
  auto put = [&](int step, unsigned v) {
    if constexpr (W == 2) out[step * 32] = static_cast<uint16_t>(v);
    else out8[step * 32] = static_cast<uint8_t>(v);
  };
  int wide = 0;  // W == 1: a slot beyond the 8-bit table (a tile of more than 256 nodes)
  RingWalk r = ring_walk_encode(j, k, pb, n, inc, el, [&](int step, int v) {
    const int sl = tslot(list, nl, rank[v]);
    if (W == 1 && sl > 255) wide = kRingWideTile;
    put(2 + step, (W == 2 && step == 0) ? (sl | (bmark[e] ? 0x8000u : 0u)) : sl);
  });
  // closed: the last ring slot repeats slot(m_0) (word-0 bit 14 / header bit 7)
  int sj = tslot(list, nl, rank[j]), sk = tslot(list, nl, rank[k]);
  if (W == 1 && (sj > 255 || sk > 255)) {
    wide = kRingWideTile;
    sj = sk = 0;  // any table node: the side list recomputes the edge
  }
  r.fail |= wide;
  if (r.fail) {  // side list: an empty ring (m_0 := k), k_navs_side recomputes the edge
    if constexpr (W == 2) {
      put(0, sj);
      put(1, sk);
      put(2, sk | (bmark[e] ? 0x8000u : 0u));
    } else {
      put(0, sj);
      put(1, sk);
      put(2, sk);
      blk[p & 31] = static_cast<uint8_t>(bmark[e] ? 64 : 0);
    }
    atomicOr(flag, r.fail);
    const int q = atomicAdd(flag + 2, 1);
    if (q < kSideCap) side[q] = make_int2(e, static_cast<int>(p));
    return;
  }
  if constexpr (W == 2) {
    put(0, sj | (r.sign < 0 ? 0x8000u : 0u) | (r.closed ? 0x4000u : 0u));
    put(1, sk | n << 11);
  } else {
    put(0, sj);
    put(1, sk);
    blk[p & 31] = static_cast<uint8_t>(n | (r.sign < 0 ? 32 : 0) | (bmark[e] ? 64 : 0) |
                                       (r.closed ? 128 : 0));
  }
}

// Size of a warp block in 32-byte units, S_w = max over the warp's edges of
// n+3 steps: W == 2: S_w * 32 u16 codes; W == 1: a 32-byte header + S_w * 32
// bytes.
__global__ void k_ring_warpsize(const int32_t* __restrict__ eperm,
                                const int32_t* __restrict__ inc_ptr, i64 ne, i64 nwarps, int W,
                                u32* __restrict__ wsize) {
  const i64 w = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (w >= nwarps) return;
  int S = 3;
  for (i64 p = w * 32; p < w * 32 + 32 && p < ne; ++p) {
    const int e = eperm[p];
    const int n = inc_ptr[e + 1] - inc_ptr[e];
    S = max(S, (n > kRingMax ? 0 : n) + 3);  // side-list edges: 3 steps
  }
  wsize[w] = static_cast<u32>(W == 2 ? 2 * S : S + 1);  // 32-byte units
}

// meta[2t]   = {C0, NC, NU | nbnd << 16, bptr}  (C0 in 32-byte units, NC in bytes)
// meta[2t+1] = eight u16 warp-block byte offsets relative to C0
__global__ void k_ring_meta(const u32* __restrict__ wstart, const u32* __restrict__ tcnt,
                            const u32* __restrict__ tile_bptr, i64 nwarps, i64 ntiles,
                            int4* __restrict__ meta) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const i64 w0 = t * (kTileEdges / 32);
  const i64 w1 = (w0 + kTileEdges / 32 < nwarps) ? w0 + kTileEdges / 32 : nwarps;
  const u32 C0 = wstart[w0], C1 = wstart[w1];  // 32-byte units
  const int nb = static_cast<int>(tile_bptr[t + 1] - tile_bptr[t]);  // <= 3 * 256
  meta[2 * t] = make_int4(static_cast<int>(C0), static_cast<int>(32 * (C1 - C0)),
                          static_cast<int>(tcnt[t]) | nb << 16, static_cast<int>(tile_bptr[t]));
  unsigned o[4] = {0u, 0u, 0u, 0u};
  for (i64 w = w0; w < w1; ++w) {
    const u32 off = min(32 * (wstart[w] - C0), 0xffffu);
    const int q = static_cast<int>(w - w0);
    o[q >> 1] |= off << (16 * (q & 1));
  }
  meta[2 * t + 1] = make_int4(static_cast<int>(o[0]), static_cast<int>(o[1]),
                              static_cast<int>(o[2]), static_cast<int>(o[3]));
}


// ---- bank-conflict-aware slot colouring (8-bit plans)
//
// In the ring kernel the 8 lanes of a quarter warp read table entries in the
// same step: 16-byte (x,y) reads conflict when two distinct slots agree mod 8,
// 8-byte z reads when they agree mod 16 within the half warp.  Sorted-rank
// slots leave ~1.8x the ideal shared-memory wavefronts.  This pass recolours
// each tile's nodes (colour = slot mod 16, 16 slots per colour) by parallel
// min-conflict rounds: every node computes the colour that minimises its
// same-bank partners over the (warp, step, half) groups it is read in; it
// moves if that helps and no partner that wants a colour in the same mod-8
// class has a higher priority (a fixed hash), capacity permitting.  Slots are
// only a relabelling of the table, so results do not depend on it
// (tools/bank_sim.py models 1.8-1.9x -> ~1.45x ideal wavefronts; measured on
// C5: shared-load conflict wavefronts 177 M -> 97 M, element loop 2.36 -> 2.25
// ms, plan +0.1 s).
int color_rounds() {
  const char* r = std::getenv("DUALMESH_COLOR_ROUNDS");
  return r ? std::max(1, std::atoi(r)) : 8;
}

__device__ __forceinline__ unsigned color_prio(unsigned tile, unsigned v) {
  unsigned h = tile * 0x9E3779B1u ^ (v + 0x7F4A7C15u) * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0xC2B2AE3Du;
  return h ^ (h >> 13);
}

// Warp-cooperative: each warp walks its own code block step by step; the 32
// lanes of a step hold the nodes read together, so the colour histograms of a
// half / quarter warp come from 16 ballots, duplicates of a lane's own node
// are removed with __match_any_sync, and each lane adds its partner counts to
// its node's cost row in shared memory.  A node that wants to move is blocked
// by a higher-priority partner (same half warp) wanting the same mod-8 class
// (__match_any_sync + __reduce_max_sync); capacity 16 slots per colour.
__global__ void __launch_bounds__(kTileEdges)
    k_tile_color_warp(uint8_t* __restrict__ rcodes, int4* __restrict__ meta,
                      int32_t* __restrict__ tnodes, int ntiles, i64 ne, int rounds) {
  __shared__ __align__(16) uint8_t cb[2 * 4096];
  __shared__ uint16_t cost[256][24];  // per node: 16 half-warp (mod 16) + 8 quarter (mod 8)
  __shared__ uint8_t col[256], want[256], blocked[256], slot_new[256];
  __shared__ int ccount[16];
  __shared__ int wofs[kTileEdges / 32 + 1];
  __shared__ int32_t ids[256];
  const int tile = blockIdx.x;
  if (tile >= ntiles) return;
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  const int4 m = meta[2 * tile];
  const int nu = m.z & 0xffff, nbytes = m.y;
  if (nu > 256) return;
  int32_t* tn = tnodes + static_cast<i64>(tile) * kTileNodeCap;
  if (nbytes > static_cast<int>(sizeof(cb))) {  // not recoloured: identity fill list
    tn[kTileFillRanks + t] = t < nu ? tn[t] : -1;
    reinterpret_cast<uint8_t*>(tn + kTileFillSlots)[t] = static_cast<uint8_t>(t);
    return;
  }
  for (int i = t; i < nbytes / 16; i += kTileEdges)
    reinterpret_cast<uint4*>(cb)[i] = reinterpret_cast<const uint4*>(rcodes + 32 * static_cast<i64>(m.x))[i];
  const i64 left = ne - static_cast<i64>(tile) * kTileEdges;
  const int nw = static_cast<int>(left >= kTileEdges ? kTileEdges / 32 : (left + 31) / 32);
  if (t <= kTileEdges / 32) {
    const int4 wo = meta[2 * tile + 1];
    const unsigned o[4] = {static_cast<unsigned>(wo.x), static_cast<unsigned>(wo.y),
                           static_cast<unsigned>(wo.z), static_cast<unsigned>(wo.w)};
    wofs[t] = t < nw ? static_cast<int>((o[t >> 1] >> (16 * (t & 1))) & 0xffffu) : nbytes;
  }
  if (t < 16) ccount[t] = 0;
  __syncthreads();
  const bool has_block = w < nw;
  const int S = has_block ? (wofs[w + 1] - wofs[w]) / 32 - 1 : 0;  // steps in this warp block
  const int nl = has_block ? (cb[wofs[w] + l] & 31) : -3;
  const uint8_t* blk = cb + wofs[w] + 32;
  if (t < nu) {
    col[t] = static_cast<uint8_t>(t & 15);
    atomicAdd(&ccount[t & 15], 1);
  }
  __syncthreads();
  const unsigned half = (l & 16) ? 0xffff0000u : 0x0000ffffu;
  const unsigned quart = 0xffu << (l & 24);
  for (int round = 0; round < rounds; ++round) {
    for (int i = t; i < 256 * 24 / 2; i += kTileEdges) reinterpret_cast<uint32_t*>(cost)[i] = 0u;
    __syncthreads();
    // ---- partner histograms, step by step (warp-uniform loop)
    for (int st = 0; st < S; ++st) {
      const bool act = st < nl + 3;
      const int x = act ? blk[st * 32 + l] : 256 + l;  // inactive lanes: unique dummies
      const int cx = act ? col[x] : 31;
      const unsigned same = __match_any_sync(0xffffffffu, x);
      const unsigned others = ~same;
      unsigned h16[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) h16[c] = __ballot_sync(0xffffffffu, cx == c);
      // one lane per (node, half) adds the half-warp counts, one per
      // (node, quarter) the quarter counts: a node read by several lanes of a
      // phase is one address (a broadcast), so it counts once
      const unsigned me = 1u << l;
      const bool lead16 = act && ((same & half) & (me - 1)) == 0;
      const bool lead8 = act && ((same & quart) & (me - 1)) == 0;
      if (lead16) {
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          const unsigned n0 = __popc(h16[c] & half & others), n1 = __popc(h16[c + 1] & half & others);
          atomicAdd(reinterpret_cast<unsigned*>(&cost[x][c]), n0 | n1 << 16);  // no branch: mostly != 0
        }
      }
      if (lead8) {
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
          const unsigned n0 = __popc((h16[c] | h16[c + 8]) & quart & others);
          const unsigned n1 = __popc((h16[c + 1] | h16[c + 9]) & quart & others);
          atomicAdd(reinterpret_cast<unsigned*>(&cost[x][16 + c]), n0 | n1 << 16);
        }
      }
    }
    __syncthreads();
    if (t < nu) {
      const int cur = col[t];
      int best = cur, bc = cost[t][cur] + cost[t][16 + (cur & 7)];
      for (int c = 0; c < 16; ++c) {
        const int cc = cost[t][c] + cost[t][16 + (c & 7)];
        if (cc < bc) {
          bc = cc;
          best = c;
        }
      }
      want[t] = static_cast<uint8_t>(best != cur ? best : 0xff);
      blocked[t] = 0;
    }
    const int any = __syncthreads_or(t < nu && want[t] != 0xff);
    if (!any) break;
    // ---- a mover is blocked by a higher-priority partner wanting the same mod-8 class
    for (int st = 0; st < S; ++st) {
      const bool act = st < nl + 3;
      const int x = act ? blk[st * 32 + l] : 0;
      const int wx = act ? want[x] : 0xff;
      const bool mv = act && wx != 0xff;
      if (!__any_sync(0xffffffffu, mv)) continue;
      const unsigned pr = mv ? ((color_prio(tile, x) & ~0xffu) | static_cast<unsigned>(x)) : 0u;
      // per (mod-8 class, half warp): the largest (priority, id) among the
      // movers wins (uniform-mask reductions, classes without movers skipped)
      unsigned best = 0u;
      const int mk = mv ? (wx & 7) : -1;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const unsigned who = __ballot_sync(0xffffffffu, mk == k);
        if (who & 0x0000ffffu) {
          const unsigned b = __reduce_max_sync(0xffffffffu, (mk == k && l < 16) ? pr : 0u);
          if (mk == k && l < 16) best = b;
        }
        if (who & 0xffff0000u) {
          const unsigned b = __reduce_max_sync(0xffffffffu, (mk == k && l >= 16) ? pr : 0u);
          if (mk == k && l >= 16) best = b;
        }
      }
      if (mv && best != pr) blocked[x] = 1;
    }
    __syncthreads();
    if (t < nu) {
      slot_new[t] = col[t];
      if (want[t] != 0xff && !blocked[t]) {
        const int b = want[t];
        if (atomicAdd(&ccount[b], 1) < 16) {
          atomicSub(&ccount[col[t]], 1);
          slot_new[t] = static_cast<uint8_t>(b);
        } else {
          atomicSub(&ccount[b], 1);
        }
      }
    }
    __syncthreads();
    if (t < nu) col[t] = slot_new[t];
    __syncthreads();
  }
  // slot = colour + 16 * (rank among the nodes of that colour, in old order):
  // per-warp colour counts from __match_any_sync, then a prefix over warps
  __shared__ int wcnt[kTileEdges / 32][17];
  {
    const int cv = t < nu ? col[t] : 16;
    const unsigned same = __match_any_sync(0xffffffffu, cv);
    if (t < 17 * (kTileEdges / 32)) wcnt[t / 17][t % 17] = 0;
    __syncthreads();
    if ((same & ((1u << l) - 1)) == 0) wcnt[w][cv] = __popc(same);
    __syncthreads();
    if (t < nu) {
      int k = __popc(same & ((1u << l) - 1));
      for (int ww = 0; ww < w; ++ww) k += wcnt[ww][cv];
      slot_new[t] = static_cast<uint8_t>(cv + 16 * k);
    }
  }
  ids[t] = -1;
  __syncthreads();
  const int32_t rank_t = t < nu ? tn[t] : -1;  // old slot t = t-th smallest rank
  if (t < nu) ids[slot_new[t]] = rank_t;
  __syncthreads();
  tn[t] = ids[t];
  tn[kTileFillRanks + t] = rank_t;
  reinterpret_cast<uint8_t*>(tn + kTileFillSlots)[t] = t < nu ? slot_new[t] : 0;
  for (int st = 0; st < nl + 3; ++st) {
    uint8_t* p = cb + wofs[w] + 32 + st * 32 + l;
    *p = slot_new[*p];
  }
  __syncthreads();
  for (int i = t; i < nbytes / 16; i += kTileEdges)
    reinterpret_cast<uint4*>(rcodes + 32 * static_cast<i64>(m.x))[i] = reinterpret_cast<const uint4*>(cb)[i];
  if (t == 0) {
    int tp = 0;
    for (int u = 0; u < 256; ++u)
      if (ids[u] >= 0) tp = u + 1;
    meta[2 * tile].z = (m.z & ~0xffff) | tp;
  }
}

__global__ void k_sum_u32(const u32* __restrict__ x, i64 n, unsigned long long* __restrict__ out) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned long long v = i < n ? x[i] : 0ull;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(out, v);
}

// ---- Morton origin order and the edge permutation

static_assert(kTileFillSlots + 256 / 4 <= kTileNodeCap && kTileFillRanks + 256 <= kTileFillSlots,
              "fill lists fit behind the 256-slot table");
static_assert(kTileNodeCap <= 2048 && kRingMax < 32, "code word 1 packs slot(k) | n << 11");
static_assert(kRingMax + 4 <= 64 && kTileEdges / 32 * 64 * (kRingMax + 4) < 65536,
              "u16 warp-block byte offsets");

// per-block partial bounding box of the coordinates: part[6 * block + {lo, hi}]
__global__ void __launch_bounds__(256) k_bbox(const d4* __restrict__ x4, i64 nv,
                                              double* __restrict__ part) {
  __shared__ double sh[6][256];
  const int t = threadIdx.x;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (i64 v = static_cast<i64>(blockIdx.x) * 256 + t; v < nv;
       v += static_cast<i64>(gridDim.x) * 256) {
    const d4 r = x4[v];
    lo[0] = fmin(lo[0], r.x);
    lo[1] = fmin(lo[1], r.y);
    lo[2] = fmin(lo[2], r.z);
    hi[0] = fmax(hi[0], r.x);
    hi[1] = fmax(hi[1], r.y);
    hi[2] = fmax(hi[2], r.z);
  }
  for (int d = 0; d < 3; ++d) {
    sh[d][t] = lo[d];
    sh[3 + d][t] = hi[d];
  }
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (t < h)
      for (int d = 0; d < 3; ++d) {
        sh[d][t] = fmin(sh[d][t], sh[d][t + h]);
        sh[3 + d][t] = fmax(sh[3 + d][t], sh[3 + d][t + h]);
      }
    __syncthreads();
  }
  if (t < 6) part[6 * blockIdx.x + t] = sh[t][0];
}

__device__ __forceinline__ u64 spread21(u64 v) {  // bit i -> bit 3i
  v &= 0x1fffffull;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}

// Origin order key.  cells == 0: the Morton key of the node's 21-bit
// quantised position.  cells > 0: the Morton key of its coarse cell (the
// bounding cube split into cells^3, any cell count) above the node id, i.e.
// cells in Z-order and the
// nodes of a cell in id order -- for a numbering with runs of consecutive ids
// along a row, a cell's rows become runs of consecutive origins, whose edge
// ranges are adjacent in the edge list (coalesced output stores).
__global__ void k_morton(const d4* __restrict__ x4, i64 nv, double lx, double ly, double lz,
                         double sc, int cells, u64* __restrict__ key,
                         int32_t* __restrict__ id) {
  const i64 v = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const d4 r = x4[v];
  auto q = [&](double x) -> u64 {
    const double f = x * sc;
    const u64 q21 = f <= 0.0 ? 0ull : (f >= 2097151.0 ? 2097151ull : static_cast<u64>(f));
    return cells ? (q21 * static_cast<u64>(cells)) >> 21 : q21;
  };
  const u64 m = spread21(q(r.x - lx)) | spread21(q(r.y - ly)) << 1 | spread21(q(r.z - lz)) << 2;
  key[v] = cells ? (m << 32 | static_cast<u64>(v)) : m;
  id[v] = static_cast<int32_t>(v);
}

// Per-axis quantile cells: the cell index of a node along an axis is its rank
// in that coordinate (sorted) scaled to `cells` -- equal node counts per slab,
// so graded / stretched grids (boundary layers) get cells of ~cell_nodes
// nodes like uniform ones.
// Axis order key: the coordinate quantised to 32 bits over the bounding box
// (uniform buckets for the bucketed sort), then the node id.  The cells only
// shape the plan's layout (performance), never the results.
__global__ void k_axis_key(const d4* __restrict__ x4, i64 nv, int axis, double lo, double sc,
                           u64* __restrict__ key, int32_t* __restrict__ id) {
  const i64 v = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const d4 r = x4[v];
  const double f = ((axis == 0 ? r.x : (axis == 1 ? r.y : r.z)) - lo) * sc;
  const u64 q = f <= 0.0 ? 0ull : (f >= 4294967295.0 ? 4294967295ull : static_cast<u64>(f));
  key[v] = q << 32 | static_cast<u64>(v);
  id[v] = static_cast<int32_t>(v);
}

__global__ void k_axis_cell(const int32_t* __restrict__ sorted, i64 nv, int axis, int cells,
                            u32* __restrict__ cellpack) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nv) return;
  const u32 ci = static_cast<u32>((static_cast<u64>(r) * static_cast<u64>(cells)) /
                                  static_cast<u64>(nv));
  const int v = sorted[r];
  if (axis == 0) cellpack[v] = ci;
  else cellpack[v] |= ci << (10 * axis);
}

__global__ void k_cell_key(const u32* __restrict__ cellpack, i64 nv, u64* __restrict__ key,
                           int32_t* __restrict__ id) {
  const i64 v = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const u32 c = cellpack[v];
  const u64 m = spread21(c & 1023u) | spread21((c >> 10) & 1023u) << 1 |
                spread21((c >> 20) & 1023u) << 2;
  key[v] = m << 32 | static_cast<u64>(v);
  id[v] = static_cast<int32_t>(v);
}

__global__ void k_origin_count(const int32_t* __restrict__ ord, const u32* __restrict__ os, i64 nv,
                               u32* __restrict__ cnt) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const int o = ord[i];
  cnt[i] = os[o + 1] - os[o];
}

__global__ void k_eperm(const int32_t* __restrict__ ord, const u32* __restrict__ os,
                        const u32* __restrict__ pstart, i64 nv, int32_t* __restrict__ eperm,
                        int32_t* __restrict__ pinv) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const u32 base = os[ord[i]], p0 = pstart[i], n = pstart[i + 1] - p0;
  for (u32 q = 0; q < n; ++q) {
    eperm[p0 + q] = static_cast<int32_t>(base + q);
    pinv[base + q] = static_cast<int32_t>(p0 + q);
  }
}

// rank-ordered incoming lists as positions: rin_list[rin_ptr[r] + q] =
// pinv[in_list[in_ptr[morder[r]] + q]]
__global__ void k_rin_count(const int32_t* __restrict__ ord, const u32* __restrict__ in_ptr, i64 nv,
                            u32* __restrict__ cnt) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nv) return;
  const int n = ord[r];
  cnt[r] = in_ptr[n + 1] - in_ptr[n];
}

__global__ void k_rin_fill(const int32_t* __restrict__ ord, const u32* __restrict__ in_ptr,
                           const int32_t* __restrict__ in_list, const int32_t* __restrict__ pinv,
                           const u32* __restrict__ rptr, i64 nv, int32_t* __restrict__ out) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nv) return;
  const int n = ord[r];
  const u32 b = in_ptr[n], m = in_ptr[n + 1] - b, o = rptr[r];
  for (u32 q = 0; q < m; ++q) out[o + q] = pinv[in_list[b + q]];
}

// number of nodes n whose successor n+1 is within 8 Morton ranks
__global__ void k_locality(const int32_t* __restrict__ rank, i64 nv, u32* __restrict__ cnt) {
  const i64 n = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool near = n + 1 < nv && abs(rank[n + 1] - rank[n]) <= 8;
  const unsigned b = __ballot_sync(0xffffffffu, near);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(cnt, static_cast<u32>(__popc(b)));
}

// boundary-edge segments of the sorted position-keyed facet list
__global__ void k_bseg_flag(const u64* __restrict__ b, i64 n, u32* __restrict__ flag) {
  const i64 q = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < n) flag[q] = (q == 0 || (b[q] >> 32) != (b[q - 1] >> 32)) ? 1u : 0u;
}

__global__ void k_bseg_fill(const u64* __restrict__ b, i64 n, const u32* __restrict__ idx,
                            const int32_t* __restrict__ eperm, const int2* __restrict__ edges,
                            int4* __restrict__ seg, u32* __restrict__ start) {
  const i64 q = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  if (q == n - 1) start[idx[n]] = static_cast<u32>(n);
  if (idx[q + 1] == idx[q]) return;  // not a segment start
  const int p = static_cast<int>(b[q] >> 32);
  const int e = eperm[p];
  const int2 jk = edges[e];
  seg[idx[q]] = make_int4(e, jk.x, jk.y, p);
  start[idx[q]] = static_cast<u32>(q);
}

__global__ void k_bkey(const u64* __restrict__ bedge, i64 n, const int32_t* __restrict__ pinv,
                       u64* __restrict__ out) {
  const i64 q = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const u64 it = bedge[q];
  out[q] = static_cast<u64>(pinv[it >> 32]) << 32 | (it & 0xffffffffull);
}

__global__ void k_rank(const int32_t* __restrict__ order, i64 nv, int32_t* __restrict__ rank) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < nv) rank[order[r]] = static_cast<int32_t>(r);
}

__global__ void k_bmark(const u64* __restrict__ bedge, i64 n, uint8_t* __restrict__ mark) {
  const i64 q = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q < n) mark[bedge[q] >> 32] = 1;
}

// Morton-order copy of the raw coordinates (x, y | z per rank r, node order[r])
__global__ void k_morton_coords(const double* __restrict__ xc, const int32_t* __restrict__ order,
                                i64 nv, double2* __restrict__ xy, double* __restrict__ z) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nv) return;
  const double* p = xc + 3 * static_cast<i64>(__ldg(order + r));
  xy[r] = make_double2(__ldg(p), __ldg(p + 1));
  z[r] = __ldg(p + 2);
}

// First arena block: the plan's peak of temporaries in one allocation
// (k0, k1, i0, rank-sort scratch, rk, cellpack ~ 40 B/node; pinv, bmark,
// warp sizes ~ 6 B/edge).
size_t arena_block(const dm_ctx* c) {
  return static_cast<size_t>(48 * c->nv + 8 * c->ne + 12 * c->n_bedge) + (64u << 20);
}

int bits_for(u64 v) {
  int b = 1;
  while (b < 64 && (v >> b)) ++b;
  return b;
}

// eperm (Morton origin order), bedge_p and its per-tile slices.
int build_edge_order(dm_ctx* c) {
  PlanClock clk(c);
  const i64 nv = c->nv, ne = c->ne, nb = c->n_bedge;
  const i64 ntiles = (ne + kTileEdges - 1) / kTileEdges;
  // bounding box
  const int nblk = static_cast<int>(std::max<i64>(1, std::min<i64>(1024, (nv + 255) / 256)));
  ScratchBuf<double> part(c->arena, arena_block(c));
  DM_CK(c, part.ensure(6 * nblk));
  DM_LAUNCH(c, k_bbox, nblk, 256, 0, c->x4.p, nv, part.p);
  std::vector<double> hp(6 * nblk);
  DM_CK(c, cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int b = 0; b < nblk; ++b)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], hp[6 * b + d]);
      hi[d] = std::max(hi[d], hp[6 * b + 3 + d]);
    }
  double ext = std::max(hi[0] - lo[0], std::max(hi[1] - lo[1], hi[2] - lo[2]));
  if (!(ext > 0.0) || !std::isfinite(ext)) ext = 1.0;
  const double sc = 2097151.0 / ext;
  clk.mark("bbox");
  // Origin order.  First the plain Morton order of the nodes; if the node
  // numbering turns out to be spatially coherent (many id-consecutive nodes
  // within 8 Morton ranks), re-sort by (Morton key of a ~64-node cell, node
  // id): a cell's rows then become runs of consecutive origins, so a warp's
  // output rows are mostly contiguous (C5: 2.51 -> 2.42 ms).  Without
  // coherence (randomly numbered grids) the plain order keeps the tables
  // small and s stays in position order for the volume pass (vol_by_rank).
  ScratchBuf<u64> k0(c->arena, arena_block(c)), k1(c->arena, arena_block(c));
  ScratchBuf<int32_t> i0(c->arena, arena_block(c));
  DM_CK(c, k0.ensure(nv));
  DM_CK(c, k1.ensure(nv));
  DM_CK(c, i0.ensure(nv));
  DM_CK(c, c->morder.ensure(nv));
  int32_t* i1p = c->morder.p;
  auto radix = [&]() -> int {  // (k0, i0) -> ids in key order (ties: ascending id) in i1p
    return sort_u64(c, k0.p, reinterpret_cast<const u32*>(i0.p), nv, k1.p,
                    reinterpret_cast<u32*>(i1p));
  };
  auto sort_nodes = [&](int cells) -> int {
    DM_LAUNCH(c, k_morton, grid_for(nv, 256), 256, 0, c->x4.p, nv, lo[0], lo[1], lo[2], sc,
              cells, k0.p, i0.p);
    return radix();
  };
  int st = sort_nodes(0);
  if (st) return st;
  clk.mark("morton sort");
  {
    ScratchBuf<int32_t> rk(c->arena, arena_block(c));
    ScratchBuf<u32> cnt(c->arena, arena_block(c));
    DM_CK(c, rk.ensure(nv));
    DM_CK(c, cnt.ensure(1));
    DM_CK(c, cudaMemsetAsync(cnt.p, 0, sizeof(u32), c->stream));
    DM_LAUNCH(c, k_rank, grid_for(nv, 256), 256, 0, i1p, nv, rk.p);
    DM_LAUNCH(c, k_locality, static_cast<unsigned>((nv + 255) / 256), 256, 0, rk.p, nv, cnt.p);
    u32 near = 0;
    DM_CK(c, cudaMemcpyAsync(&near, cnt.p, sizeof(u32), cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    c->vol_by_rank = static_cast<double>(near) < 0.25 * static_cast<double>(nv);
  }
  clk.mark("locality");
  // cells of ~cell_nodes nodes (env DUALMESH_CELL_NODES, 0 = plain Morton always)
  double cell_nodes = 64.0;
  if (const char* cn = std::getenv("DUALMESH_CELL_NODES")) cell_nodes = std::atof(cn);
  if (!c->vol_by_rank && cell_nodes > 0.0 && nv > 0) {
    // cells^3 cells of ~cell_nodes nodes on a cubic grid (at most 1024 per
    // axis so the key, 3*10 + 32 bits, fits)
    const int cells = static_cast<int>(std::max<long>(
        1, std::min<long>(1024, std::lround(std::cbrt(static_cast<double>(nv) / cell_nodes)))));
    ScratchBuf<u32> cellpack(c->arena, arena_block(c));
    DM_CK(c, cellpack.ensure(nv));
    for (int axis = 0; axis < 3; ++axis) {
      const double ax_ext = hi[axis] - lo[axis];
      const double ax_sc = ax_ext > 0.0 && std::isfinite(ax_ext) ? 4294967295.0 / ax_ext : 0.0;
      DM_LAUNCH(c, k_axis_key, grid_for(nv, 256), 256, 0, c->x4.p, nv, axis, lo[axis], ax_sc,
                k0.p, i0.p);
      st = radix();
      if (st) return st;
      DM_LAUNCH(c, k_axis_cell, grid_for(nv, 256), 256, 0, i1p, nv, axis, cells, cellpack.p);
    }
    DM_LAUNCH(c, k_cell_key, grid_for(nv, 256), 256, 0, cellpack.p, nv, k0.p, i0.p);
    st = radix();
    if (st) return st;
  }
  clk.mark("quantile cells");
  // edge permutation: each origin's edge range appended whole, in that order
  u32* pstart = nullptr;
  ScratchBuf<int32_t> pinv(c->arena, arena_block(c));
  DM_CK(c, c->rpstart.ensure(nv + 1));
  pstart = c->rpstart.p;
  DM_CK(c, pinv.ensure(ne > 0 ? ne : 1));
  DM_CK(c, c->eperm.ensure(ne > 0 ? ne : 1));
  DM_LAUNCH(c, k_origin_count, grid_for(nv, 256), 256, 0, i1p, c->os.p, nv, pstart);
  st = scan_exclusive(c, pstart, pstart, nv);
  if (st) return st;
  DM_LAUNCH(c, k_eperm, grid_for(nv, 256), 256, 0, i1p, c->os.p, pstart, nv, c->eperm.p,
            pinv.p);
  // (lanes ordered by ring length inside each tile, to even out the warps'
  // ring lengths on irregular meshes, measured 29 % slower on a flipped grid
  // and 32 % on C5: the origin order's store and table locality matter more)
  clk.mark("eperm");
  // Edge-volume terms (vol_by_rank decided above): for a spatially coherent
  // numbering the edge-id order is already local, so s goes to svals[e] and
  // the id-order volume pass reads it coalesced; otherwise s stays in position
  // order and the volume pass walks Morton ranks.
  if (c->vol_by_rank) {  // incoming edges per rank, as positions (volumes.cu)
    st = ensure_incoming(c);
    if (st) return st;
    DM_CK(c, c->rin_ptr.ensure(nv + 1));
    DM_CK(c, c->rin_list.ensure(ne));
    DM_LAUNCH(c, k_rin_count, grid_for(nv, 256), 256, 0, i1p, c->in_ptr.p, nv, c->rin_ptr.p);
    st = scan_exclusive(c, c->rin_ptr.p, c->rin_ptr.p, nv);
    if (st) return st;
    DM_LAUNCH(c, k_rin_fill, grid_for(nv, 256), 256, 0, i1p, c->in_ptr.p, c->in_list.p, pinv.p,
              c->rin_ptr.p, nv, c->rin_list.p);
  }

  clk.mark("rank incoming");
  // boundary (edge, facet) list re-keyed by position
  DM_CK(c, c->bedge_p.ensure(nb > 0 ? nb : 1));
  DM_CK(c, c->tile_bptr_p.ensure(ntiles + 1));
  if (nb > 0) {
    ScratchBuf<u64> bk(c->arena, arena_block(c));
    DM_CK(c, bk.ensure(nb));
    DM_LAUNCH(c, k_bkey, grid_for(nb, 256), 256, 0, c->bedge.p, nb, pinv.p, bk.p);
    st = sort_u64(c, bk.p, nullptr, nb, c->bedge_p.p, nullptr);  // (position, facet): unique
    if (st) return st;
  }
  DM_LAUNCH(c, k_tile_bptr, grid_for(ntiles + 1, 256), 256, 0, c->bedge_p.p,
            static_cast<u32>(nb), ne, ntiles, c->tile_bptr_p.p);
  c->n_bseg = 0;
  if (nb > 0) {
    ScratchBuf<u32> idx(c->arena, arena_block(c));
    DM_CK(c, idx.ensure(nb + 1));
    DM_LAUNCH(c, k_bseg_flag, grid_for(nb, 256), 256, 0, c->bedge_p.p, nb, idx.p);
    st = scan_exclusive(c, idx.p, idx.p, nb);
    if (st) return st;
    u32 ns = 0;
    DM_CK(c, cudaMemcpyAsync(&ns, idx.p + nb, sizeof(u32), cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    DM_CK(c, c->bseg.ensure(ns));
    DM_CK(c, c->bseg_start.ensure(ns + 1));
    DM_LAUNCH(c, k_bseg_fill, grid_for(nb, 256), 256, 0, c->bedge_p.p, nb, idx.p, c->eperm.p,
              c->edges.p, c->bseg.p, c->bseg_start.p);
    c->n_bseg = ns;
  }
  clk.mark("boundary lists");
  return DM_OK;
}

}  // namespace

int ensure_rings(dm_ctx* c) {
  if (c->have_rings) return DM_OK;
  ArenaScope scratch(c->arena);  // temporaries of this plan are released on return
  PlanClock clk(c);
  int st0 = ensure_bedge(c);  // tile_bptr feeds the ring metadata
  if (st0) return st0;
  clk.mark("boundary edges");
  if (c->dim != 3) {
    c->ring_ok = false;
    c->row_plan = false;
    c->plan_colored = false;
    c->ring_max_nodes = 0;
    c->ring_fail = 0;
    c->n_side = 0;
    c->have_rings = true;
    return DM_OK;
  }
  // row tiles first (rowplan.cu): contiguous edge ranges whose tables fit
  c->row_plan = false;
  c->n_side = 0;
  c->ring_fail = 0;
  if (int sr = try_row_plan(c)) return sr;
  clk.mark("row plan");
  if (c->row_plan) {
    c->ring_ok = true;
    c->code_width = 1;
    c->vol_by_rank = false;
    c->plan_colored = false;
    c->ring_max_nodes = kRowSlots;
    c->have_rings = true;
    return DM_OK;
  }
  const i64 ne = c->ne;
  const i64 ntiles = (ne + kTileEdges - 1) / kTileEdges;
  const i64 nwarps = (ne + 31) / 32;
  if (int sx = ensure_x4(c)) return sx;  // the plan's Morton keys read the padded copy
  if (ne == 0 || !c->x4.p) {
    c->ring_ok = false;
    c->have_rings = true;
    return DM_OK;
  }
  int st1 = build_edge_order(c);
  if (st1) return st1;
  clk.mark("edge order (total)");
  DM_CK(c, c->tnodes.ensure(static_cast<size_t>(ntiles * kTileNodeCap)));
  DM_CK(c, c->tnode_cnt.ensure(static_cast<size_t>(ntiles)));
  // tiles that overflow the caps keep count 0 (their codes are never used:
  // the overflow sets ring_ok = false)
  DM_CK(c, cudaMemsetAsync(c->tnode_cnt.p, 0, ntiles * sizeof(u32), c->stream));
  DM_CK(c, c->ring_meta.ensure(static_cast<size_t>(2 * ntiles)));
  DM_CK(c, c->flag.ensure(4));
  DM_CK(c, cudaMemsetAsync(c->flag.p, 0, 4 * sizeof(int), c->stream));
  DM_CK(c, c->side.ensure(kSideCap));
  c->n_side = 0;
  ScratchBuf<int32_t> rank(c->arena, arena_block(c));
  ScratchBuf<uint8_t> bmark(c->arena, arena_block(c));
  DM_CK(c, rank.ensure(c->nv));
  DM_CK(c, bmark.ensure(ne));
  DM_LAUNCH(c, k_rank, grid_for(c->nv, 256), 256, 0, c->morder.p, c->nv, rank.p);
  DM_CK(c, cudaMemsetAsync(bmark.p, 0, ne, c->stream));
  if (c->n_bedge > 0)
    DM_LAUNCH(c, k_bmark, grid_for(c->n_bedge, 256), 256, 0, c->bedge.p, c->n_bedge, bmark.p);
  DM_LAUNCH(c, k_tile_nodes, static_cast<unsigned>(ntiles), kTileEdges, 0, c->edges.p,
            c->eperm.p, c->inc_ptr.p, c->inc.p, c->elems.p, rank.p, ne, c->tnodes.p,
            c->tnode_cnt.p, c->flag.p);
  // 8-bit slot codes when every tile table fits 256 nodes, else 16-bit
  int fl0[4] = {0, 0, 0, 0};
  DM_CK(c, cudaMemcpyAsync(fl0, c->flag.p, sizeof(fl0), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  c->code_width = fl0[1] <= 256 ? 1 : 2;
  // A few tiles just over 256 nodes (where the Morton curve jumps) would put the
  // whole mesh on 16-bit codes and the two-buffer kernel (256^3 permuted:
  // one tile of 262 nodes, element loop 3.13 instead of ~2.5 ms).  The plan
  // keeps 8-bit codes then: an edge whose slots pass 255 goes to the side
  // list, its tile reads the table from global memory (the slot colouring
  // leaves such tiles alone).
  // env DUALMESH_WIDE_TILES_MAX: tiles over 256 nodes tolerated per 1000 (default 5).
  {
    int per_mille = 5;
    if (const char* wt = std::getenv("DUALMESH_WIDE_TILES_MAX")) per_mille = std::atoi(wt);
    if (c->code_width == 2 && !(fl0[0] & 2) &&
        static_cast<i64>(fl0[3]) * 1000 <= static_cast<i64>(per_mille) * ntiles)
      c->code_width = 1;
  }
  clk.mark("tile nodes");
  ScratchBuf<u32> wstart(c->arena, arena_block(c));
  DM_CK(c, wstart.ensure(static_cast<size_t>(nwarps + 1)));
  DM_LAUNCH(c, k_ring_warpsize, grid_for(nwarps, 256), 256, 0, c->eperm.p, c->inc_ptr.p, ne,
            nwarps, c->code_width, wstart.p);
  // code offsets are 32-bit: check the exact total before the u32 scan
  {
    ScratchBuf<unsigned long long> tot(c->arena, arena_block(c));
    DM_CK(c, tot.ensure(1));
    DM_CK(c, cudaMemsetAsync(tot.p, 0, sizeof(unsigned long long), c->stream));
    DM_LAUNCH(c, k_sum_u32, grid_for(nwarps, 256), 256, 0, wstart.p, nwarps, tot.p);
    unsigned long long h = 0;
    DM_CK(c, cudaMemcpyAsync(&h, tot.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    if (h + 1 >= (1ull << 31)) {  // 32-byte units in int4 metadata: bit-exact path beyond 64 GB
      c->ring_fail = 32;
      c->ring_ok = false;
      c->have_rings = true;
      return DM_OK;
    }
  }
  int st = scan_exclusive(c, wstart.p, wstart.p, nwarps);
  if (st) return st;
  u32 nunits = 0;
  DM_CK(c, cudaMemcpyAsync(&nunits, wstart.p + nwarps, sizeof(u32), cudaMemcpyDeviceToHost,
                           c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  const size_t nbytes = 32 * static_cast<size_t>(nunits);
  clk.mark("code offsets");
  DM_CK(c, c->rcodes.ensure(nbytes + 16));
  DM_CK(c, cudaMemsetAsync(c->rcodes.p, 0, nbytes + 16, c->stream));
  if (c->code_width == 1)
    DM_LAUNCH(c, k_ring_codes<1>, grid_for(ne, 128), 128, 0, c->edges.p, c->eperm.p,
              c->inc_ptr.p, c->inc.p, c->elems.p, rank.p, bmark.p, c->tnodes.p, c->tnode_cnt.p,
              wstart.p, ne, c->rcodes.p, c->flag.p, c->side.p);
  else
    DM_LAUNCH(c, k_ring_codes<2>, grid_for(ne, 128), 128, 0, c->edges.p, c->eperm.p,
              c->inc_ptr.p, c->inc.p, c->elems.p, rank.p, bmark.p, c->tnodes.p, c->tnode_cnt.p,
              wstart.p, ne, c->rcodes.p, c->flag.p, c->side.p);
  DM_LAUNCH(c, k_ring_meta, grid_for(ntiles, 256), 256, 0, wstart.p, c->tnode_cnt.p,
            c->tile_bptr_p.p, nwarps, ntiles, c->ring_meta.p);
  clk.mark("ring codes");
  // bank-conflict-aware slots for 8-bit plans: by default only for coherent
  // numberings (the 2-3-flipped grid: element loop 0.712 -> 0.694 ms); on a
  // randomly numbered grid it no longer pays (C3: 0.562 ms without, 0.568-
  // 0.573 ms with 1-8 rounds, plus ~20 ms of plan; tools/color_rounds_sweep.py).
  // env DUALMESH_PLAN_COLOR=0 / 1 forces it off / on.
  c->plan_colored = false;
  if (c->code_width == 1) {
    const char* pc = std::getenv("DUALMESH_PLAN_COLOR");
    if (pc ? std::atoi(pc) != 0 : !c->vol_by_rank) {
      DM_LAUNCH(c, k_tile_color_warp, static_cast<unsigned>(ntiles), kTileEdges, 0,
                c->rcodes.p, c->ring_meta.p, c->tnodes.p, static_cast<int>(ntiles), ne,
                color_rounds());
      c->plan_colored = true;
    }
  }
  int fl[3] = {0, 0, 0};
  DM_CK(c, cudaMemcpyAsync(fl, c->flag.p, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  c->ring_fail = fl[0];
  c->ring_max_nodes = fl[1];
  // edges the rings cannot describe ride the side list; only an oversized
  // tile table (bit 2) or an overfull side list disables the ring path
  c->n_side = fl[2];
  c->ring_ok = (fl[0] & 2) == 0 && fl[2] <= kSideCap;
  c->have_rings = true;
  clk.mark("colouring");
  return DM_OK;  // the Morton-order coordinates are staged by every navs call
}

int refresh_ring_coords(dm_ctx* c) {
  const i64 nv = c->nv;
  DM_CK(c, c->mxy.ensure(nv));
  DM_CK(c, c->mz.ensure(nv));
  DM_LAUNCH(c, k_morton_coords, grid_for(nv, 256), 256, 0, c->coords.p, c->morder.p, nv,
            c->mxy.p, c->mz.p);
  return DM_OK;
}

}  // namespace dm
