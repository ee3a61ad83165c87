// edge_extract.cu -- K1 on origin buckets of element entries: the edge list,
// origin CSR, edge->element incidence and element->local-edge map of
// north_star (a), bit-exact with the reference build_edges
// (proj/src/mesh.cpp:256-285: pairs (min, max), sorted lexicographically)
// with each edge's incident elements ascending (the element order of the
// per-edge sums).
//
// The reference hashes every (element, local edge) pair and sorts the
// unique pairs.  Here the unit of work is the origin bucket of node j: the
// elements in which j is not the largest node (an "entry" per such element,
// D per element), each contributing the pairs (j, k) for its nodes k > j.
//
//   k_ent_fill     per element: each entry node takes a slot in its fixed-
//                  capacity bucket row (runs of adjacent lanes with the same
//                  node -- a hex's tets share a corner -- take their slots
//                  with one atomic) and the element id goes there; flags
//                  repeated or out-of-range nodes and rows that overflow
//   k_edge_chunks  a warp per chunk of 32 consecutive buckets, a lane per
//                  bucket: the chunk's rows are staged coalesced, each lane
//                  sorts its entries by element id and its items by
//                  (k - j, entry rank) with register sorting networks
//                  (sortnet.cuh) and counts its edges and items; a
//                  decoupled look-back over CTA tiles (8 chunks) gives the
//                  first edge id and item position; the lanes emit e2l
//                  directly and stage inc, edges and inc_ptr in shared
//                  memory for coalesced stores.  A narrow variant holds
//                  rows of <= 21 entries in registers, a wide one <= 25
//                  (chosen by a k_ent_fill flag).
//
// Buckets with more entries than a row holds (Caps::kNe) take a side path
// before k_edge_chunks: their entries are collected into exact lists,
// expanded into (k << 32 | e*L + l) items and sorted by the generic
// segmented sort; their lanes emit from that list.  Meshes with a repeated
// node inside an element or an element spanning 2^25 node ids take the generic item-sort
// path (edges.cu).
#include <cstdlib>
#include <utility>

#include "dm_internal.cuh"
#include "sortnet.cuh"

#ifdef DM_K1_DEBUG
#define K1_CHECK(cond, what, v)                                                        \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("K1 check failed: %s (%lld) line %d\n", what, (long long)(v), __LINE__); \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define K1_CHECK(cond, what, v) \
  do {                          \
  } while (0)
#endif

namespace dm {
namespace {

constexpr unsigned F = 0xffffffffu;
constexpr u32 kInf = 0xffffffffu;
constexpr int kChunk = 32;  // buckets per warp chunk (a lane each)
constexpr int kWarps = 8;   // warp chunks per CTA tile of k_edge_chunks
constexpr int kCtasPerSm = 16 / kWarps;  // 16 warps per SM at ~128 registers
constexpr u64 kFlagA = 1ull << 62, kFlagP = 2ull << 62, kValMask = (1ull << 62) - 1;
// look-back values pack (edges << 31 | items): both stay below 2^31
constexpr u64 kItemMask = (1ull << 31) - 1;

// Bucket row capacity (entries on the register path; odd, so the staged
// rows are read without shared-memory bank conflicts) and the per-warp
// staging sizes.  A 3D Kuhn interior node has 18 entries, 36 items and 7
// edges; a 2D node ~4 entries.
template <int D>
struct Caps {
  static constexpr int kNe = D == 3 ? 25 : 23;      // row capacity (entries per bucket row)
  static constexpr int kNarrow = D == 3 ? 21 : 23;  // register path of the narrow chunk kernel
  static constexpr int kIncStage = D == 3 ? 1152 : 768;  // items per chunk (entries staged here first)
  static constexpr int kHeadStage = D == 3 ? 288 : 256;  // edges per chunk
};

// Local edge id of the local node pair (p, q), 4 bits at (4p + q), symmetric.
// tet_local_edges = {01,02,03,12,13,23} (mesh.cpp:17); 2D {01,12,20}
// (mesh.cpp:263-265).
constexpr u64 ledge_table(bool tet) {
  const int tp[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
  const int tr[3][2] = {{0, 1}, {1, 2}, {2, 0}};
  u64 t = 0;
  const int n = tet ? 6 : 3;
  for (int l = 0; l < n; ++l) {
    const int a = tet ? tp[l][0] : tr[l][0], b = tet ? tp[l][1] : tr[l][1];
    t |= static_cast<u64>(l) << (4 * (4 * a + b));
    t |= static_cast<u64>(l) << (4 * (4 * b + a));
  }
  return t;
}
constexpr u64 kTetLedge = ledge_table(true);
constexpr u64 kTriLedge = ledge_table(false);

template <int D>
__device__ __forceinline__ u32 ledge(int p, int q) {
  return static_cast<u32>(((D == 3 ? kTetLedge : kTriLedge) >> (4 * (4 * p + q))) & 0xF);
}

template <int D>
__device__ __forceinline__ void load_nodes(const int32_t* el, i64 e, int (&v)[4]) {
  if (D == 3) {
    const int4 t = ld_i4(reinterpret_cast<const int4*>(el) + e);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
    v[0] = __ldg(el + 3 * e); v[1] = __ldg(el + 3 * e + 1); v[2] = __ldg(el + 3 * e + 2);
    v[3] = 0;
  }
}

// ---------------------------------------------------------------- entry rows
// Node v[p] ranks above r other nodes of its element; with r < D it is the
// origin of D - r of the element's pairs.  Flags: 1 = node id out of range,
// 2 = repeated node (the generic path handles the reference's (a, a) pairs).
template <int D>
__device__ __forceinline__ int elem_ranks(const int (&v)[4], i64 nv, int (&rk)[4]) {
  int bad = 0;
#pragma unroll
  for (int p = 0; p <= D; ++p) {
    if (static_cast<unsigned>(v[p]) >= static_cast<u64>(nv)) bad |= 1;
    rk[p] = 0;
  }
#pragma unroll
  for (int p = 0; p <= D; ++p)
#pragma unroll
    for (int q = 0; q <= D; ++q)
      if (q != p) {
        rk[p] += v[q] < v[p];
        if (q > p && v[q] == v[p]) bad |= 2;
        // the item keys hold k - j in 25 bits (k_edge_chunks)
        if (!(bad & 1) && static_cast<i64>(v[q]) - v[p] >= (1ll << 25)) bad |= 16;
      }
  return bad;
}

// Flag 4: some bucket has more than Caps::kNe entries (side path); flag 8:
// some bucket has more than Caps::kNarrow (the wide chunk kernel); flag 16
// (elem_ranks): an element spans node ids 2^25 or more apart (generic path).
template <int D>
__global__ void k_ent_fill(const int32_t* __restrict__ el, i64 nE, i64 nv, u32* __restrict__ cnt,
                           u32* __restrict__ ent, int* flag) {
  constexpr int CAP = Caps<D>::kNe;
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int v[4] = {0, 0, 0, 0}, rk[4] = {D, D, D, D};
  int bad = 0;
  if (e < nE) {
    load_nodes<D>(el, e, v);
    bad = elem_ranks<D>(v, nv, rk);
    if (bad) atomicOr(flag, bad);
  }
  const bool live = e < nE && !bad;
  // per role r: the origin, its run of adjacent lanes with the same origin
  // (consecutive elements sharing a node, e.g. the tets of one hex) and
  // the run's first lane, which takes the run's slots with one atomic; the
  // D atomics are issued back to back (predicated, no branches between)
  int jr[D], lead[D];
  u32 base[D];
#pragma unroll
  for (int r = 0; r < D; ++r) {
    int j = -1;
#pragma unroll
    for (int p = 0; p <= D; ++p)
      if (rk[p] == r) j = v[p];
    if (!live) j = -1;
    const int up = __shfl_up_sync(F, j, 1);
    const unsigned heads = __ballot_sync(F, lane == 0 || up != j);
    const int leader = 31 - __clz(heads & (0xffffffffu >> (31 - lane)));
    const unsigned after = heads & ~(0xffffffffu >> (31 - lane));
    const u32 run = static_cast<u32>((after ? __ffs(after) - 1 : 32) - lane);
    const u32 go = lane == leader && j >= 0;
    u32* addr = cnt + (j >= 0 ? j : 0);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %3, 0;\n\t"
        "@p atom.global.add.u32 %0, [%1], %2;\n\t}"
        : "=r"(base[r])
        : "l"(addr), "r"(run), "r"(go)
        : "memory");
    jr[r] = j;
    lead[r] = leader;
  }
  int over = 0;
#pragma unroll
  for (int r = 0; r < D; ++r) {
    const u32 b = __shfl_sync(F, base[r], lead[r]);
    if (jr[r] >= 0) {
      const u32 slot = b + static_cast<u32>(lane - lead[r]);
      if (slot < static_cast<u32>(CAP))
        ent[static_cast<i64>(jr[r]) * CAP + slot] = static_cast<u32>(e);
      else over |= 4;
      if (slot >= static_cast<u32>(Caps<D>::kNarrow)) over |= 8;
    }
  }
  over = __reduce_or_sync(F, over);
  if (over && lane == 0) atomicOr(flag, over);
}

// ---------------------------------------------------------------- side path
// bflag[j] = 1 for a bucket beyond its row (scanned into the side index).
template <int D>
__global__ void k_big_mark(const u32* __restrict__ cnt, i64 nv, u32* __restrict__ f) {
  const i64 j = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < nv) f[j] = cnt[j] > static_cast<u32>(Caps<D>::kNe);
}

__global__ void k_big_list(const u32* __restrict__ cnt, const u32* __restrict__ bscan, i64 nv,
                           u32* __restrict__ blist, u32* __restrict__ bent_cnt) {
  const i64 j = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= nv) return;
  const u32 b = bscan[j];
  if (bscan[j + 1] == b) return;
  blist[b] = static_cast<u32>(j);
  bent_cnt[b] = cnt[j];
}

// Every entry of a side bucket into its exact list (order is irrelevant:
// the items are sorted).
template <int D>
__global__ void k_big_collect(const int32_t* __restrict__ el, i64 nE, const u32* __restrict__ cnt,
                              const u32* __restrict__ bscan, const u32* __restrict__ bent_seg,
                              u32* __restrict__ bfill, u32* __restrict__ bent) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nE) return;
  int v[4], rk[4];
  load_nodes<D>(el, e, v);
#pragma unroll
  for (int p = 0; p <= D; ++p) {
    rk[p] = 0;
#pragma unroll
    for (int q = 0; q <= D; ++q) rk[p] += q != p && v[q] < v[p];
  }
#pragma unroll
  for (int p = 0; p <= D; ++p)
    if (rk[p] < D && cnt[v[p]] > static_cast<u32>(Caps<D>::kNe)) {
      const u32 b = bscan[v[p]];
      bent[bent_seg[b] + atomicAdd(bfill + b, 1u)] = static_cast<u32>(e);
    }
}

// Warp per side bucket: items per bucket (count == nullptr: the items
// themselves, (k << 32 | e*L + l), into their segment).
template <int D>
__global__ void k_big_items(const int32_t* __restrict__ el, const u32* __restrict__ blist,
                            const u32* __restrict__ bent_seg, const u32* __restrict__ bent,
                            u32 nbig, u32* __restrict__ count, const u32* __restrict__ bseg,
                            u64* __restrict__ items) {
  constexpr int L = D == 3 ? 6 : 3;
  const int lane = threadIdx.x & 31;
  const u32 b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (b >= nbig) return;
  const int j = static_cast<int>(blist[b]);
  const u32 eb = bent_seg[b], n = bent_seg[b + 1] - eb;
  u32 out = count ? 0u : bseg[b];
  for (u32 i0 = 0; i0 < n; i0 += 32) {
    const u32 i = i0 + lane;
    int v[4] = {0, 0, 0, 0};
    u32 e = 0;
    int cntk = 0;
    if (i < n) {
      e = bent[eb + i];
      load_nodes<D>(el, e, v);
#pragma unroll
      for (int p = 0; p <= D; ++p) cntk += v[p] > j;
    }
    int incl = cntk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(F, incl, o);
      if (lane >= o) incl += t;
    }
    if (!count && i < n) {
      int pj = 0;
#pragma unroll
      for (int p = 0; p <= D; ++p)
        if (v[p] == j) pj = p;
      u32 w = out + static_cast<u32>(incl - cntk);
#pragma unroll
      for (int p = 0; p <= D; ++p)
        if (v[p] > j)
          items[w++] = (static_cast<u64>(static_cast<u32>(v[p])) << 32) |
                       static_cast<u64>(e * static_cast<u32>(L) + ledge<D>(pj, p));
    }
    out += static_cast<u32>(__shfl_sync(F, incl, 31));
  }
  if (count && lane == 0) count[b] = out;
}

// ---------------------------------------------------------------- chunks
// Decoupled look-back over CTA-tile totals (one warp): returns the exclusive
// prefix of tile t and publishes its inclusive prefix.  Tiles are taken in
// ticket order, so every predecessor is running or done; with one status
// word per CTA tile at most ~2 x #SMs tiles are in flight, which bounds the
// walk over predecessors that have only their aggregate published.
__device__ __forceinline__ u64 ld_relaxed_gpu(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ u64 tile_lookback(u64* status, u32 t, u64 total, int lane) {
  if (t == 0) {
    if (lane == 0) st_relaxed_gpu(status, kFlagP | total);
    return 0;
  }
  if (lane == 0) st_relaxed_gpu(status + t, kFlagA | total);
  u64 prefix = 0;
  i64 base = static_cast<i64>(t) - 1;
  for (;;) {
    const i64 idx = base - lane;
    const u64 v = idx >= 0 ? ld_relaxed_gpu(status + idx) : kFlagP;
    const unsigned notready = __ballot_sync(F, (v >> 62) == 0);
    const unsigned isp = __ballot_sync(F, (v >> 62) == 2);
    const unsigned need = isp ? (isp & (0u - isp)) * 2u - 1u : F;  // lanes up to the first P
    if (notready & need) {
      __nanosleep(64);
      continue;
    }
    u64 x = (need >> lane) & 1u ? (v & kValMask) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(F, x, o);
    prefix += x;
    if (isp) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed_gpu(status + t, kFlagP | (prefix + total));
  return prefix;
}

struct ChunkArgs {
  const int32_t* el;
  const u32* cnt;
  const u32* ent;
  i64 nv;
  u32 nchunks, ntiles;
  u32* ticket;
  u64* status;
  // side buckets (nullptr when none)
  const u32* bscan;
  const u32* bseg;
  const u32* bd;
  const u64* bitems;
  // outputs
  int2* edges;
  u32* os;
  int32_t* inc_ptr;
  int32_t* inc;
  int32_t* e2l;
  u32 cap_edges;
  int* overflow;
  u32 m_items, n_elems;  // bounds (debug checks)
};

struct Lane {
  i64 j;
  bool valid, big;
  u32 n_ent;
};

// Per-CTA tile scratch: the ticket and the warps' packed (edges, items)
// totals, then their first edge id / item position.
struct TileShared {
  u32 ticket;
  u64 wtot[kWarps];
};

// One warp chunk with at most NE entries in any register-path bucket; every
// warp of the CTA calls it once per tile (it holds the tile's barriers).
template <int D, int NE>
__device__ __forceinline__ void process_chunk(const ChunkArgs& A, u32 tile, u32 c,
                                              const Lane& Ln, const u32* s_ent,
                                              u64 (*s_info)[32], u32* s_inc, int2* s_hedge,
                                              u32* s_hptr, TileShared& ts, int warp, int lane,
                                              u32 inc_cap) {
  constexpr int L = D == 3 ? 6 : 3;
  constexpr int CAP = Caps<D>::kNe;
  constexpr int S = D * NE;  // item slots: D per entry (the element's other nodes)
  const bool reg = Ln.valid && !Ln.big;
  const int j = static_cast<int>(Ln.j);
  K1_CHECK(!reg || Ln.n_ent <= static_cast<u32>(NE), "n_ent", Ln.n_ent);

  // entries of this bucket, ascending element id
  u32 es[NE];
#pragma unroll
  for (int s = 0; s < NE; ++s)
    es[s] = reg && static_cast<u32>(s) < Ln.n_ent ? s_ent[lane * CAP + s] : kInf;
  oem_sort<NE>(es);
  __syncwarp();  // the staged rows are dead: the space becomes the inc stage

  // items: key = (k - j) << 7 | entry rank << 2 | t, t = the node's place
  // among the element's other nodes; kInf for nodes below j / empty slots
  u32 key[S];
  constexpr int GB = 6;  // element rows gathered per batch (loads in flight; 4-12 measured equal)
  static_for<0, (NE + GB - 1) / GB>([&](auto batch) {
    constexpr int s0 = decltype(batch)::value * GB;
    int4 row[GB];
#pragma unroll
    for (int u = 0; u < GB; ++u) {
      const int s = s0 + u;
      row[u] = make_int4(0, 0, 0, 0);
      if (s < NE && es[s] != kInf) {
        K1_CHECK(es[s] < A.n_elems, "entry", es[s]);
        if (D == 3) {
          row[u] = ld_i4(reinterpret_cast<const int4*>(A.el) + es[s]);
        } else {
          const int32_t* r = A.el + 3 * static_cast<i64>(es[s]);
          row[u] = make_int4(__ldg(r), __ldg(r + 1), __ldg(r + 2), 0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < GB; ++u) {
      const int s = s0 + u;
      if (s < NE) {
        const bool live = es[s] != kInf;
        const int v[4] = {row[u].x, row[u].y, row[u].z, row[u].w};
        const int pj = v[0] == j ? 0 : v[1] == j ? 1 : (D == 3 && v[2] == j) ? 2 : D;
        u32 ls = 0;
#pragma unroll
        for (int t = 0; t < D; ++t) {
          const int q = t + (t >= pj);  // the element's other local nodes, in order
          const int a = sel4(v[0], v[1], v[2], v[3], q);
          key[D * s + t] = live && a > j
                               ? (static_cast<u32>(a - j) << 7) | (static_cast<u32>(s) << 2) | t
                               : kInf;
          ls |= ledge<D>(pj, q) << (3 * t);
        }
        if (live) s_info[s][lane] = (static_cast<u64>(ls) << 32) | es[s];
      }
    }
  });
  oem_sort<S>(key);

  // edges and items of the bucket; slots past the warp's fullest bucket are
  // empty and skipped warp-uniformly
  u32 d = 0, nit = 0;
  if (reg) {
    u32 prev = kInf;
    if constexpr (S <= 64) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (key[s] == kInf) break;
        const u32 kd = key[s] >> 7;
        d += kd != prev;
        prev = kd;
        ++nit;
      }
    } else {  // the wide kernel: a compile-time loop keeps key[] in registers
      static_for<0, S>([&](auto si) {
        constexpr int s = decltype(si)::value;
        const u32 kd = key[s] >> 7;
        const bool v = key[s] != kInf;
        d += v && kd != prev;
        prev = kd;
        nit += v;
      });
    }
  } else if (Ln.big) {
    const u32 b = A.bscan[Ln.j];
    d = A.bd[b];
    nit = A.bseg[b + 1] - A.bseg[b];
  }
  const u32 nmax = __reduce_max_sync(F, reg ? nit : 0u);
  u64 x = (static_cast<u64>(d) << 31) | nit;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u64 t = __shfl_up_sync(F, x, o);
    if (lane >= o) x += t;
  }
  // tile prefix: warp totals -> warp 0 looks back -> every warp's first id
  if (lane == 31) ts.wtot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const u64 w = lane < kWarps ? ts.wtot[lane] : 0ull;
    u64 wi = w;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const u64 t = __shfl_up_sync(F, wi, o);
      if (lane >= o) wi += t;
    }
    const u64 ttot = __shfl_sync(F, wi, kWarps - 1);
    const u64 tfirst = tile_lookback(A.status, tile, ttot, lane);
    if (lane < kWarps) ts.wtot[lane] = tfirst + wi - w;  // exclusive, per warp
  }
  __syncthreads();
  const u64 wfirst = ts.wtot[warp];
  const u64 mine = wfirst + x - ((static_cast<u64>(d) << 31) | nit);
  const u32 osj = static_cast<u32>(mine >> 31), ib = static_cast<u32>(mine & kItemMask);
  const u64 wlast = __shfl_sync(F, x, 31);
  const u32 e0 = static_cast<u32>(wfirst >> 31), ib0 = static_cast<u32>(wfirst & kItemMask);
  const u32 ne_w = static_cast<u32>(wlast >> 31), ni_w = static_cast<u32>(wlast & kItemMask);
  if (Ln.valid) {
    A.os[Ln.j] = osj;
    if (Ln.j == A.nv - 1) A.os[A.nv] = osj + d;
  }
  if (e0 + ne_w > A.cap_edges && lane == 0) atomicOr(A.overflow, 1);

  // inc, edges and inc_ptr through shared memory when the chunk fits
  const bool anybig = __any_sync(F, Ln.big);
  const bool st_inc = !anybig && ni_w <= inc_cap;
  const bool st_head = !anybig && ne_w <= static_cast<u32>(Caps<D>::kHeadStage);
  if (reg) {
    u32 prev = kInf, g = 0;
    auto emit = [&](const int s) {
      if (key[s] != kInf) {
        const u32 kd = key[s] >> 7, se = (key[s] >> 2) & 31, t = key[s] & 3;
        const bool head = kd != prev;
        prev = kd;
        g += head;
        const u64 info = s_info[se][lane];
        const u32 e = static_cast<u32>(info);
        const u32 l = static_cast<u32>(info >> (32 + 3 * t)) & 7;
        const u32 id = osj + g - 1;
        K1_CHECK(e < A.n_elems && l < static_cast<u32>(L), "e2l", e);
        K1_CHECK(ib + s < A.m_items, "inc", ib + s);
        if (st_inc) s_inc[ib - ib0 + s] = e;
        else A.inc[ib + s] = static_cast<int32_t>(e);
        A.e2l[e * static_cast<u32>(L) + l] = static_cast<int32_t>(id);
        if (head) {
          if (st_head) {
            s_hedge[id - e0] = make_int2(j, j + static_cast<int>(kd));
            s_hptr[id - e0] = ib + s;
          } else if (id < A.cap_edges) {
            A.edges[id] = make_int2(j, j + static_cast<int>(kd));
            A.inc_ptr[id] = static_cast<int32_t>(ib + s);
          }
        }
      }
    };
    if constexpr (S <= 64) {
#pragma unroll
      for (int s = 0; s < S; ++s) {
        if (static_cast<u32>(s) >= nmax) break;
        emit(s);
      }
    } else {
      static_for<0, S>([&](auto si) {
        if (static_cast<u32>(decltype(si)::value) < nmax) emit(decltype(si)::value);
      });
    }
  }
  // side buckets: the warp emits each from its sorted item list
  unsigned bigm = __ballot_sync(F, Ln.big);
  while (bigm) {
    const int b = __ffs(bigm) - 1;
    bigm &= bigm - 1;
    const i64 jb = static_cast<i64>(c) * kChunk + b;
    const u32 bi = A.bscan[jb];
    const u32 s0 = A.bseg[bi], n = A.bseg[bi + 1] - s0;
    const u32 ibb = __shfl_sync(F, ib, b);
    u32 id_base = __shfl_sync(F, osj, b);
    u32 prev_hi = kInf;
    for (u32 i0 = 0; i0 < n; i0 += 32) {
      const u32 i = i0 + lane;
      const u64 it = i < n ? A.bitems[s0 + i] : ~0ull;
      const u32 hi = static_cast<u32>(it >> 32);
      u32 up = __shfl_up_sync(F, hi, 1);
      if (lane == 0) up = prev_hi;
      prev_hi = __shfl_sync(F, hi, 31);
      const bool head = i < n && hi != up;
      const unsigned hm = __ballot_sync(F, head);
      if (i < n) {
        const u32 id = id_base + __popc(hm & (F >> (31 - lane))) - 1;
        const u32 val = static_cast<u32>(it);
        if (head && id < A.cap_edges) {
          A.edges[id] = make_int2(static_cast<int>(jb), static_cast<int>(hi));
          A.inc_ptr[id] = static_cast<int32_t>(ibb + i);
        }
        A.inc[ibb + i] = static_cast<int32_t>(val / L);
        A.e2l[val] = static_cast<int32_t>(id);
      }
      id_base += __popc(hm);
    }
  }
  __syncwarp();
  if (st_inc)
    for (u32 i = lane; i < ni_w; i += 32) A.inc[ib0 + i] = static_cast<int32_t>(s_inc[i]);
  if (st_head)
    for (u32 i = lane; i < ne_w; i += 32)
      if (e0 + i < A.cap_edges) {
        A.edges[e0 + i] = s_hedge[i];
        A.inc_ptr[e0 + i] = static_cast<int32_t>(s_hptr[i]);
      }
  __syncwarp();
}

// Shared memory per warp of k_edge_chunks<D, NEMAX>: entry info [NEMAX][32]
// (element id | local edges << 32); the chunk's staged rows, then inc;
// staged edges and inc_ptr.  Sized for kCtasPerSm CTAs per SM.
template <int D, int NEMAX>
struct ChunkSmem {
  static constexpr int kInfo = NEMAX * 32 * 8;
  static constexpr int kInc = NEMAX > 21 ? 1024 : Caps<D>::kIncStage;
  static constexpr int kHead = Caps<D>::kHeadStage;
  static constexpr int kWarpBytes = kInfo + kInc * 4 + kHead * 12;
  static_assert(kInc >= Caps<D>::kNe * 32, "the chunk's rows are staged inside the inc stage");
  static_assert(kCtasPerSm * (kWarps * kWarpBytes + 1024 + 128) <= 228 * 1024, "CTAs per SM");
};

template <int D, int NEMAX>
__global__ void __launch_bounds__(kWarps * 32, kCtasPerSm) k_edge_chunks(ChunkArgs A) {
  constexpr int NE = Caps<D>::kNe;  // row stride
  using SM = ChunkSmem<D, NEMAX>;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ TileShared ts;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* wbase = smem + warp * SM::kWarpBytes;
  u64 (*s_info)[32] = reinterpret_cast<u64 (*)[32]>(wbase);
  u32* s_inc = reinterpret_cast<u32*>(wbase + SM::kInfo);
  int2* s_hedge = reinterpret_cast<int2*>(wbase + SM::kInfo + SM::kInc * 4);
  u32* s_hptr = reinterpret_cast<u32*>(wbase + SM::kInfo + SM::kInc * 4 + SM::kHead * 8);
  for (;;) {
    if (threadIdx.x == 0) ts.ticket = atomicAdd(A.ticket, 1u);
    __syncthreads();
    const u32 tile = ts.ticket;
    __syncthreads();  // ticket read by all before thread 0 takes the next one
    if (tile >= A.ntiles) break;
    const u32 c = tile * kWarps + warp;
    Lane Ln;
    Ln.j = static_cast<i64>(c) * kChunk + lane;
    Ln.valid = Ln.j < A.nv;
    Ln.n_ent = Ln.valid ? A.cnt[Ln.j] : 0u;
    Ln.big = Ln.n_ent > static_cast<u32>(NEMAX);
    // the chunk's rows, coalesced (rows past nv exist and are never read)
    if (c < A.nchunks) {
      const uint4* src = reinterpret_cast<const uint4*>(A.ent + static_cast<i64>(c) * kChunk * NE);
      uint4* dst = reinterpret_cast<uint4*>(s_inc);
      constexpr int N4 = NE * 32 / 4;
#pragma unroll
      for (int i = lane; i < N4; i += 32) dst[i] = __ldg(src + i);
    }
    __syncwarp();
    const u32 wmax = __reduce_max_sync(F, Ln.valid && !Ln.big ? Ln.n_ent : 0u);
    if (D == 3) {
      if (wmax <= 12)
        process_chunk<D, 12>(A, tile, c, Ln, s_inc, s_info, s_inc, s_hedge, s_hptr, ts, warp, lane, SM::kInc);
      else if (wmax <= 15)
        process_chunk<D, 15>(A, tile, c, Ln, s_inc, s_info, s_inc, s_hedge, s_hptr, ts, warp, lane, SM::kInc);
      else if (wmax <= 18)
        process_chunk<D, 18>(A, tile, c, Ln, s_inc, s_info, s_inc, s_hedge, s_hptr, ts, warp, lane, SM::kInc);
      else if (NEMAX <= 21 || wmax <= 21)
        process_chunk<D, 21>(A, tile, c, Ln, s_inc, s_info, s_inc, s_hedge, s_hptr, ts, warp, lane, SM::kInc);
      else
        process_chunk<D, (NEMAX > 21 ? NEMAX : 21)>(A, tile, c, Ln, s_inc, s_info, s_inc, s_hedge,
                                                    s_hptr, ts, warp, lane, SM::kInc);
    } else {
      if (wmax <= 8)
        process_chunk<D, 8>(A, tile, c, Ln, s_inc, s_info, s_inc, s_hedge, s_hptr, ts, warp, lane, SM::kInc);
      else if (wmax <= 16)
        process_chunk<D, 16>(A, tile, c, Ln, s_inc, s_info, s_inc, s_hedge, s_hptr, ts, warp, lane, SM::kInc);
      else
        process_chunk<D, NEMAX>(A, tile, c, Ln, s_inc, s_info, s_inc, s_hedge, s_hptr, ts, warp, lane, SM::kInc);
    }
  }
}

__global__ void k_set_i32_k1(int32_t* p, int32_t v) { *p = v; }

template <int D, int NEMAX>
int run_chunks(dm_ctx* c, ChunkArgs A, int* flags_host) {
  DM_CK(c, cudaMemsetAsync(c->k1_status.p, 0, sizeof(u64) * A.ntiles, c->stream));
  DM_CK(c, cudaMemsetAsync(c->flag.p, 0, 4 * sizeof(int), c->stream));
  A.ticket = reinterpret_cast<u32*>(c->flag.p + 1);
  A.overflow = c->flag.p + 2;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = static_cast<unsigned>(std::min<i64>(sms * kCtasPerSm, A.ntiles));
  constexpr size_t smem = kWarps * ChunkSmem<D, NEMAX>::kWarpBytes;
  DM_CK(c, cudaFuncSetAttribute(k_edge_chunks<D, NEMAX>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  DM_LAUNCH(c, (k_edge_chunks<D, NEMAX>), grid, kWarps * 32, smem, A);
  DM_CK(c, cudaMemcpyAsync(flags_host, c->flag.p, 4 * sizeof(int), cudaMemcpyDeviceToHost,
                           c->stream));
  return DM_OK;
}

}  // namespace

template <int D>
static int build_buckets(dm_ctx* c) {
  constexpr int L = D == 3 ? 6 : 3;
  constexpr int CAP = Caps<D>::kNe;
  const i64 nv = c->nv, nE = c->nE, M = static_cast<i64>(L) * nE;
  ChunkArgs A{};
  A.nv = nv;
  A.nchunks = static_cast<u32>((nv + kChunk - 1) / kChunk);
  A.ntiles = (A.nchunks + kWarps - 1) / kWarps;
  A.m_items = static_cast<u32>(M);
  A.n_elems = static_cast<u32>(nE);
  DM_CK(c, c->fill.ensure(static_cast<size_t>(nv + 1)));
  DM_CK(c, c->k1_ent.ensure(static_cast<size_t>(A.nchunks) * kChunk * CAP));
  DM_CK(c, c->flag.ensure(4));
  DM_CK(c, cudaMemsetAsync(c->fill.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_CK(c, cudaMemsetAsync(c->flag.p, 0, 4 * sizeof(int), c->stream));
  DM_LAUNCH(c, k_ent_fill<D>, grid_for(nE, 256), 256, 0, c->elems.p, nE, nv, c->fill.p,
            c->k1_ent.p, c->flag.p);
  int hflag = 0;
  DM_CK(c, cudaMemcpyAsync(&hflag, c->flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  if (hflag & 1)
    return fail(c, DM_ERR_INVALID_ARG, "an element references a node id outside [0, n_nodes)");
  if (hflag & (2 | 16)) return kK1Unsupported;
  A.el = c->elems.p;
  A.cnt = c->fill.p;
  A.ent = c->k1_ent.p;

  if (hflag & 4) {  // side buckets
    DM_CK(c, c->k1_bscan.ensure(static_cast<size_t>(nv + 1)));
    DM_LAUNCH(c, k_big_mark<D>, grid_for(nv, 256), 256, 0, c->fill.p, nv, c->k1_bscan.p);
    int st = scan_exclusive(c, c->k1_bscan.p, c->k1_bscan.p, nv);
    if (st) return st;
    u32 nbig = 0;
    DM_CK(c, cudaMemcpyAsync(&nbig, c->k1_bscan.p + nv, sizeof(u32), cudaMemcpyDeviceToHost,
                             c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    // per side bucket: entry list segment, item count, item segment
    DM_CK(c, c->k1_blist.ensure(nbig));
    DM_CK(c, c->k1_bseg.ensure(2 * (static_cast<size_t>(nbig) + 1)));  // entry segs | item segs
    DM_CK(c, c->k1_bd.ensure(2 * static_cast<size_t>(nbig) + 1));      // distinct | fill
    u32* bent_seg = c->k1_bseg.p;
    u32* bseg = c->k1_bseg.p + nbig + 1;
    u32* bfill = c->k1_bd.p + nbig;
    DM_LAUNCH(c, k_big_list, grid_for(nv, 256), 256, 0, c->fill.p, c->k1_bscan.p, nv,
              c->k1_blist.p, bent_seg);
    st = scan_exclusive(c, bent_seg, bent_seg, nbig);
    if (st) return st;
    u32 nbent = 0;
    DM_CK(c, cudaMemcpyAsync(&nbent, bent_seg + nbig, sizeof(u32), cudaMemcpyDeviceToHost,
                             c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    DevBuf<u32> bent;
    DM_CK(c, bent.ensure(std::max<u32>(nbent, 1)));
    DM_CK(c, cudaMemsetAsync(bfill, 0, sizeof(u32) * (nbig + 1), c->stream));
    DM_LAUNCH(c, k_big_collect<D>, grid_for(nE, 256), 256, 0, c->elems.p, nE, c->fill.p,
              c->k1_bscan.p, bent_seg, bfill, bent.p);
    const unsigned gb = grid_for(static_cast<i64>(nbig) * 32, 256);
    DM_LAUNCH(c, k_big_items<D>, gb, 256, 0, c->elems.p, c->k1_blist.p, bent_seg, bent.p, nbig,
              bseg, nullptr, nullptr);
    st = scan_exclusive(c, bseg, bseg, nbig);
    if (st) return st;
    u32 nbi = 0;
    DM_CK(c, cudaMemcpyAsync(&nbi, bseg + nbig, sizeof(u32), cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    DM_CK(c, c->k1_bitems.ensure(std::max<u32>(nbi, 1)));
    DM_LAUNCH(c, k_big_items<D>, gb, 256, 0, c->elems.p, c->k1_blist.p, bent_seg, bent.p, nbig,
              nullptr, bseg, c->k1_bitems.p);
    st = segment_sort_unique_u64(c, c->k1_bitems.p, bseg, nbig, c->k1_bd.p);
    // the entry lists (bent) are freed at the end of this block: the stream
    // must be past their readers on every path
    const cudaError_t sync = cudaStreamSynchronize(c->stream);
    if (st) return st;
    DM_CK(c, sync);
    A.bscan = c->k1_bscan.p;
    A.bseg = bseg;
    A.bd = c->k1_bd.p;
    A.bitems = c->k1_bitems.p;
  }
  // edge count estimate (V + T for a simplicial complex, plus slack); an
  // overflow re-runs k_edge_chunks with the exact count
  i64 est = std::min<i64>(M, (nv + nE) + (nv + nE) / 8 + 1024);
  if (const char* t = std::getenv("DUALMESH_K1_EDGE_EST")) est = std::max<i64>(1, std::atoll(t));
  if (c->edges.n < static_cast<size_t>(est)) {
    DM_CK(c, c->edges.ensure(static_cast<size_t>(est)));
    DM_CK(c, c->inc_ptr.ensure(static_cast<size_t>(est + 1)));
  }
  DM_CK(c, c->os.ensure(static_cast<size_t>(nv + 1)));
  DM_CK(c, c->inc.ensure(static_cast<size_t>(std::max<i64>(M, 1))));
  DM_CK(c, c->e2l.ensure(static_cast<size_t>(std::max<i64>(M, 1))));
  DM_CK(c, c->k1_status.ensure(std::max<u32>(A.ntiles, 1)));
  A.status = c->k1_status.p;
  A.os = c->os.p;
  A.inc = c->inc.p;
  A.e2l = c->e2l.p;
  for (int pass = 0; pass < 2; ++pass) {
    A.edges = c->edges.p;
    A.inc_ptr = c->inc_ptr.p;
    A.cap_edges = static_cast<u32>(std::min<size_t>(c->edges.n, 0xffffffffu));
    int hf[4] = {0, 0, 0, 0};
    int st = (hflag & 8) ? run_chunks<D, Caps<D>::kNe>(c, A, hf)
                         : run_chunks<D, Caps<D>::kNarrow>(c, A, hf);
    if (st) return st;
    u32 ne32 = 0;
    DM_CK(c, cudaMemcpyAsync(&ne32, c->os.p + nv, sizeof(u32), cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    c->ne = ne32;
    if (!hf[2]) break;
    if (pass == 1) return fail(c, DM_ERR_CUDA, "edge extraction: edge count overflow on re-run");
    DM_CK(c, c->edges.ensure(static_cast<size_t>(c->ne)));
    DM_CK(c, c->inc_ptr.ensure(static_cast<size_t>(c->ne + 1)));
  }
  DM_LAUNCH(c, k_set_i32_k1, 1, 1, 0, c->inc_ptr.p + c->ne, static_cast<int32_t>(M));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}

int build_edges_buckets(dm_ctx* c) {
  // (any node count the device layout takes: what the item keys limit is the
  // node-id span of an element, k - j < 2^25, flagged by k_ent_fill)
  if (c->nv < 1) return kK1Unsupported;
  return c->dim == 3 ? build_buckets<3>(c) : build_buckets<2>(c);
}

}  // namespace dm
