// navs.cu -- lumped directed-area vectors (navs) on the GPU.
//
//   K2  element loop     : dual-free or traditional
//                           contributions
//   K3  boundary pass    : n_jk += n_B / (D(D+1))
//   s   edge dot product : s_e = (x_k - x_j) . n_jk, the per-edge term of the
//                          edge-based dual volumes, fused here
//                          so K4 never re-reads navs.
//
// Variants (dm_navs(ctx, algo, variant)):
//   GATHER (default, 3D): the ring walk over the Morton-tile plan of rings.cu
//       (k_navs_ring_pipe): one new table node per incidence, persistent CTAs
//       with a double-buffered cp.async pipeline; dual-free (K3 in
//       k_ring_boundary) and traditional forms; <= 1e-12 of
//       the serial loop, deterministic.
//   GATHER_EXACT: row-table gather (k_navs_gather) summing in ascending
//       element id -- bitwise the serial oracle; traditional: face list.
//   GATHER_FACES: one thread per edge over the face-list incidence (ifl),
//       ascending element id, bitwise (also 2D and the fallbacks).
//   GATHER_ELEM: the same fold through the element-id CSR (inc) and a
//       dependent connectivity gather per incidence (kept for comparison).
//   SCATTER: one thread per element, fp64 atomics (REDG.E.ADD.F64) through
//       e2l into zeroed navs, aggregated per warp over lanes hitting the same
//       edge, then the same per-edge tail; summation order varies run to run
//       (<=1e-12 parity, not deterministic).
#include <algorithm>
#include <cstdlib>

#include "geometry.cuh"

namespace dm {
namespace {

constexpr int kEB = kTileEdges;  // edges per CTA (one per thread)
constexpr int kCH = 1536;        // GATHER_ELEM incidences per shared-memory chunk
constexpr int kNodeMask = (1 << 30) - 1;

template <int D>
using Pt = typename std::conditional<D == 3, d4, double2>::type;

template <int D, int ALGO>
__device__ __forceinline__ void contribution(const Coords<D>& X, const int32_t* __restrict__ el,
                                             int E, int j, int k, double* c) {
  if constexpr (D == 3) {
    const int4 t = ld_i4(reinterpret_cast<const int4*>(el) + E);
    const int ij = t.x == j ? 0 : (t.y == j ? 1 : (t.z == j ? 2 : 3));
    if constexpr (ALGO == kDualFree) {
      df3(X, t.x, t.y, t.z, t.w, ij, c[0], c[1], c[2]);
    } else {
      const int ik = t.x == k ? 0 : (t.y == k ? 1 : (t.z == k ? 2 : 3));
      tr3(X, t.x, t.y, t.z, t.w, ij, ik, c[0], c[1], c[2]);
    }
  } else {
    const int v0 = __ldg(el + 3 * E), v1 = __ldg(el + 3 * E + 1), v2 = __ldg(el + 3 * E + 2);
    const int ij = v0 == j ? 0 : (v1 == j ? 1 : 2);
    if constexpr (ALGO == kDualFree) {
      df2(X, v0, v1, v2, ij, c[0], c[1]);
    } else {
      const int ik = v0 == k ? 0 : (v1 == k ? 1 : 2);
      tr2(X, v0, v1, v2, ij, ik, c[0], c[1]);
    }
  }
}

// Contribution from a face-list entry f, with x_j / x_k of the edge.
template <int ALGO>
__device__ __forceinline__ void face_contrib3(int ij, int ik, const d4& xj, const d4& xk,
                                              const d4& xl, const d4& xr, double& c0, double& c1,
                                              double& c2) {
  const unsigned rest = 0xFu & ~((1u << ij) | (1u << ik));
  const int il = __ffs(rest) - 1;
  // value selects (no references: a runtime-chosen reference would force
  // the operands to the stack)
  auto pick = [&](int i) -> d4 {
    d4 r;
    r.x = i == ij ? xj.x : (i == ik ? xk.x : (i == il ? xl.x : xr.x));
    r.y = i == ij ? xj.y : (i == ik ? xk.y : (i == il ? xl.y : xr.y));
    r.z = i == ij ? xj.z : (i == ik ? xk.z : (i == il ? xl.z : xr.z));
    r.w = 0.0;
    return r;
  };
  if constexpr (ALGO == kDualFree) {
    const unsigned fc = (kOppPacked >> (6 * ij)) & 63u;  // ref mesh.cpp:15
    const d4 p0 = pick(fc & 3);
    const d4 p1 = pick((fc >> 2) & 3);
    const d4 p2 = pick((fc >> 4) & 3);
    cross3(p1.x - p0.x, p1.y - p0.y, p1.z - p0.z, p2.x - p0.x, p2.y - p0.y, p2.z - p0.z, c0, c1,
           c2);
  } else {
    tr3_core(pick(0), pick(1), pick(2), pick(3), xj, xk, xl, xr, c0, c1, c2);
  }
}

template <int ALGO>
__device__ __forceinline__ void face_contrib2(int ij, int ik, const double2& xj, const double2& xk,
                                              const double2& xm, double& c0, double& c1) {
  auto pick = [&](int i) -> double2 {
    return make_double2(i == ij ? xj.x : (i == ik ? xk.x : xm.x),
                        i == ij ? xj.y : (i == ik ? xk.y : xm.y));
  };
  if constexpr (ALGO == kDualFree) {
    const double2 p = pick(ij == 2 ? 0 : ij + 1);  // ref mesh.cpp:97-101
    const double2 q = pick(ij == 0 ? 2 : ij - 1);
    c0 = (1.0 / 3.0) * (q.y - p.y);
    c1 = (1.0 / 3.0) * (p.x - q.x);
  } else {
    tr2_core(pick(0), pick(1), pick(2), xj, xk, c0, c1);
  }
}

// Per-edge tail shared by all variants: scale pass, boundary pass and the
// edge-volume term s.  acc holds the element-loop sum for edge e; [rb, re)
// is the tile's slice of the sorted boundary (edge, facet) list.
template <int D, int ALGO>
__device__ __forceinline__ void edge_tail_values(const Coords<D>& X, i64 e, const double* acc,
                                                 const Pt<D>& xj, const Pt<D>& xk,
                                                 const u64* __restrict__ bedge, u32 rb, u32 re,
                                                 const int32_t* __restrict__ bnd, double* n,
                                                 double& s) {
  n[0] = acc[0];
  n[1] = acc[1];
  n[2] = D == 3 ? acc[2] : 0.0;
  if constexpr (D == 3) {
    const double f = ALGO == kDualFree ? (1.0 / 12.0) : 0.5;  // SPEC.md:162 / PAPER.md:170
    n[0] *= f;
    n[1] *= f;
    n[2] *= f;
  }
  if constexpr (ALGO == kDualFree) {
    if (rb < re) {
      u32 lo = rb, hi = re;  // lower bound of e in the tile slice
      while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if ((bedge[mid] >> 32) < static_cast<u64>(e)) lo = mid + 1;
        else hi = mid;
      }
      constexpr double fb = 1.0 / static_cast<double>(D * (D + 1));
      for (u32 q = lo; q < re; ++q) {
        const u64 it = bedge[q];
        if ((it >> 32) != static_cast<u64>(e)) break;
        const i64 b = static_cast<i64>(it & 0xffffffffu);
        if constexpr (D == 3) {
          double b0, b1, b2;
          bnormal3(X, bnd + 3 * b, b0, b1, b2);
          n[0] += fb * b0;
          n[1] += fb * b1;
          n[2] += fb * b2;
        } else {
          double b0, b1;
          bnormal2(X, bnd + 2 * b, b0, b1);
          n[0] += fb * b0;
          n[1] += fb * b1;
        }
      }
    }
  }
  s = (xk.x - xj.x) * n[0] + (xk.y - xj.y) * n[1];
  if constexpr (D == 3) s = s + (xk.z - xj.z) * n[2];
}

template <int D, int ALGO>
__device__ __forceinline__ void edge_tail(const Coords<D>& X, i64 e, const double* acc,
                                          const Pt<D>& xj, const Pt<D>& xk,
                                          const u64* __restrict__ bedge, u32 rb, u32 re,
                                          const int32_t* __restrict__ bnd,
                                          double* __restrict__ navs, double* __restrict__ svals) {
  double n[3], s;
  edge_tail_values<D, ALGO>(X, e, acc, xj, xk, bedge, rb, re, bnd, n, s);
#pragma unroll
  for (int d = 0; d < D; ++d) navs[D * e + d] = n[d];
  svals[e] = s;
}

// Coalesced store of a warp's block of 32 consecutive edges' navs: lane l
// stores doubles l, l+32, l+64 of the warp's contiguous 32*D-double block
// (shuffle transpose).  All 32 lanes must call it.
template <int D>
__device__ __forceinline__ void store_navs_warp(const double* n, i64 wbase, i64 ne,
                                                double* __restrict__ navs) {
  __syncwarp();
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int r = 0; r < D; ++r) {
    const int i = lane + 32 * r;  // double index inside the warp block
    const int src = i / D, comp = i - src * D;
    const double v0 = __shfl_sync(0xffffffffu, n[0], src);
    const double v1 = __shfl_sync(0xffffffffu, n[1], src);
    double v = comp == 0 ? v0 : v1;
    if constexpr (D == 3) {
      const double v2 = __shfl_sync(0xffffffffu, n[2], src);
      v = comp == 2 ? v2 : v;
    }
    if (wbase + src < ne) navs[D * wbase + i] = v;
  }
}

// Per-lane store of one 3D navs row (24 bytes at 24e): one 16-byte and one
// 8-byte store, ordered by the row's 16-byte alignment (e even: xy | z,
// e odd: x | yz).
__device__ __forceinline__ void store_nav_row(double* __restrict__ navs, i64 e, const double* n) {
  double* r = navs + 3 * e;
  if ((e & 1) == 0) {
    *reinterpret_cast<double2*>(r) = make_double2(n[0], n[1]);
    r[2] = n[2];
  } else {
    r[0] = n[0];
    *reinterpret_cast<double2*>(r + 1) = make_double2(n[1], n[2]);
  }
}

// ------------------------------------------------------------------ GATHER (row table)
// One CTA per 256-edge tile, one thread per edge.  The tile's edges belong
// to consecutive origin rows [j0, jl]; per-tile metadata (tables.cu) gives
// the tile's contiguous slices of the incidence codes, of the rows'
// adjacency and of the row pointers, so the CTA stages everything in two
// independent waves -- (1) codes, adjacency ids, row pointers, row-node
// coordinates (all coalesced), (2) one gather of the adjacency coordinates
// (about two random node loads per edge instead of two per incidence) --
// and then evaluates every incidence from shared memory only.  Tiles larger
// than the shared-memory caps read the same data from global memory (same
// arithmetic, same order).
constexpr int kTabCap = 1024;   // adjacency coordinates per tile
constexpr int kCodeCap = 2048;  // incidence codes per tile
constexpr int kRowCap = 320;    // origin rows per tile

// Dual-free term of one incidence from its code and a coordinate source.
template <int D, typename Tab>
__device__ __forceinline__ void df_code(unsigned cd, int rb, const Tab& tab, double* c) {
  if constexpr (D == 3) {
    const d4 p0 = tab(rb + static_cast<int>(cd & 31u));
    const d4 p1 = tab(rb + static_cast<int>((cd >> 5) & 31u));
    const d4 p2 = tab(rb + static_cast<int>((cd >> 10) & 31u));
    cross3(p1.x - p0.x, p1.y - p0.y, p1.z - p0.z, p2.x - p0.x, p2.y - p0.y, p2.z - p0.z, c[0],
           c[1], c[2]);
  } else {
    const double2 p = tab(rb + static_cast<int>(cd & 31u));
    const double2 q = tab(rb + static_cast<int>((cd >> 5) & 31u));
    c[0] = (1.0 / 3.0) * (q.y - p.y);
    c[1] = (1.0 / 3.0) * (p.x - q.x);
  }
}

template <int D, int U, int MINB>
__global__ void __launch_bounds__(kEB, MINB)
    k_navs_gather(const int2* __restrict__ edges, const int32_t* __restrict__ inc_ptr,
                  const uint16_t* __restrict__ codes, const u32* __restrict__ adj_ptr,
                  const int32_t* __restrict__ adj, const u32* __restrict__ os,
                  const int4* __restrict__ tile_meta, Coords<D> X, i64 ne,
                  const u64* __restrict__ bedge, const u32* __restrict__ tile_bptr,
                  const int32_t* __restrict__ bnd, double* __restrict__ navs,
                  double* __restrict__ svals) {
  __shared__ double s_t[D][kTabCap];     // adjacency coordinates (SoA)
  __shared__ double s_xr[D][kRowCap];    // row-node coordinates (SoA)
  __shared__ u32 s_rp[kRowCap + 1];      // adj_ptr of the rows (tile-relative)
  __shared__ u32 s_ro[kRowCap];          // adj_ptr[j+1] - os[j+1] (tile-relative)
  __shared__ uint16_t s_cd[kCodeCap];    // incidence codes
  const int t = threadIdx.x;
  const int lane = t & 31;
  const i64 e0 = static_cast<i64>(blockIdx.x) * kEB;
  const i64 e = e0 + t;
  const bool valid = e < ne;
  // tile_meta[2*tile] = {A0, A1, P0, P1}, [2*tile+1] = {j0, jl, 0, 0}
  const int4 m0 = __ldg(tile_meta + 2 * blockIdx.x);
  const int4 m1 = __ldg(tile_meta + 2 * blockIdx.x + 1);
  const u32 A0 = static_cast<u32>(m0.x);
  const int T = m0.y - m0.x, P0 = m0.z, NP = m0.w - m0.z;
  const int j0 = m1.x, NR = m1.y - m1.x + 1;
  const bool fast = T <= kTabCap && NP <= kCodeCap && NR <= kRowCap;  // CTA-uniform
  int2 jk = make_int2(j0, j0);  // idle lanes of a partial tile point at row j0
  int pb = 0, pe = 0;
  if (valid) {
    jk = edges[e];
    pb = inc_ptr[e];
    pe = inc_ptr[e + 1];
  }
  double acc[3] = {0.0, 0.0, 0.0};
  Pt<D> xj, xk;
  if (fast) {
    // wave 1: codes, row pointers, row-node coordinates (coalesced)
    for (int i = t; i < NP; i += kEB) s_cd[i] = __ldg(codes + P0 + i);
    for (int r = t; r <= NR; r += kEB) {
      const u32 ap = __ldg(adj_ptr + j0 + r);
      s_rp[r] = ap - A0;
      if (r > 0) s_ro[r - 1] = ap - __ldg(os + j0 + r) - A0;
    }
    for (int r = t; r < NR; r += kEB) {
      const Pt<D> p = X[j0 + r];
      s_xr[0][r] = p.x;
      s_xr[1][r] = p.y;
      if constexpr (D == 3) s_xr[2][r] = p.z;
    }
    // wave 2: adjacency coordinates (one gather per adjacency entry)
    for (int i = t; i < T; i += kEB) {
      const Pt<D> p = X[__ldg(adj + A0 + i)];
      s_t[0][i] = p.x;
      s_t[1][i] = p.y;
      if constexpr (D == 3) s_t[2][i] = p.z;
    }
    __syncthreads();
    auto tab = [&](int i) -> Pt<D> {
      Pt<D> p;
      p.x = s_t[0][i];
      p.y = s_t[1][i];
      if constexpr (D == 3) p.z = s_t[2][i];
      return p;
    };
    const int r = jk.x - j0;
    const int rb = static_cast<int>(s_rp[r]);
    xj.x = s_xr[0][r];
    xj.y = s_xr[1][r];
    if constexpr (D == 3) xj.z = s_xr[2][r];
    xk = tab(static_cast<int>(s_ro[r] + static_cast<u32>(e)));
    const uint16_t* cd = s_cd - P0;
    int q = pb;
    for (; q + U <= pe; q += U) {
      unsigned w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = cd[q + u];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        double c[3];
        df_code<D>(w[u], rb, tab, c);
#pragma unroll
        for (int d = 0; d < D; ++d) acc[d] += c[d];
      }
    }
    for (; q < pe; ++q) {
      double c[3];
      df_code<D>(cd[q], rb, tab, c);
#pragma unroll
      for (int d = 0; d < D; ++d) acc[d] += c[d];
    }
  } else {
    // oversized tile: identical arithmetic and order straight from global memory
    auto tab = [&](int i) -> Pt<D> { return X[__ldg(adj + A0 + i)]; };
    const int rb = static_cast<int>(__ldg(adj_ptr + jk.x) - A0);
    xj = X[jk.x];
    xk = tab(static_cast<int>(__ldg(adj_ptr + jk.x + 1) - __ldg(os + jk.x + 1) +
                              static_cast<u32>(e) - A0));
    for (int q = pb; q < pe; ++q) {
      double c[3];
      df_code<D>(__ldg(codes + q), rb, tab, c);
#pragma unroll
      for (int d = 0; d < D; ++d) acc[d] += c[d];
    }
  }
  double n[3] = {0.0, 0.0, 0.0};
  double s = 0.0;
  if (valid) {
    edge_tail_values<D, kDualFree>(X, e, acc, xj, xk, bedge, tile_bptr[blockIdx.x],
                                   tile_bptr[blockIdx.x + 1], bnd, n, s);
    svals[e] = s;
  }
  store_navs_warp<D>(n, e - lane, ne, navs);
}

// ------------------------------------------------------------------ GATHER (pipelined ring walk)
// The default 3D dual-free kernel.  Persistent CTAs walk the 256-edge tiles
// of the Morton edge order (rings.cu) blockIdx.x, blockIdx.x + gridDim.x,
// ...; one thread per edge walks the ring of its incident elements through a
// shared-memory table of the tile's nodes (one table read per incidence).
// While tile i is evaluated, the node table (16-byte xy + 8-byte z cp.async
// per node) and ring codes of tile i+1 stream into the other half of a
// double buffer with cp.async (LDGSTS, no register round trip), and the node
// ids, edge ids and metadata of tile i+2 are prefetched into registers -- so
// the per-tile gather latency hides behind the previous tile's arithmetic.
// The terms of an edge are summed unsigned and the edge's common orientation
// applied once.  Tiles with more than CAP nodes or kPipeCodeCap codes are
// evaluated straight from global memory (same arithmetic, same order).
constexpr int kPipeCodeCap = 4096;  // 16-bit codes per buffer
extern __shared__ __align__(128) unsigned char dm_smem[];

// NB buffers of CCAP 16-bit code units each.  With two buffers a tile ends
// with a barrier before its buffer is refilled; with three the refill of
// buffer (i+1) mod 3 at tile i only needs every thread past tile i-1's
// evaluation, which the one barrier of tile i already guarantees.
template <int CAP, int NB = 2, int CCAP = kPipeCodeCap>
struct PipeSmem {
  static_assert((CCAP / 2 + 4) % 4 == 0, "code rows stay 16-byte aligned");
  static constexpr int kCodeBytes = 2 * CCAP;
  // node table split into a 16-byte (x,y) array and an 8-byte z array: a
  // random 16-byte LDS spreads over 8 bank groups instead of the 4 a 32-byte
  // record allows, and z over 16 (fewer conflict wavefronts per read)
  double2 xy[NB][CAP];
  double z[NB][CAP];
  uint32_t cd[NB][CCAP / 2 + 4];  // rows stay 16-byte aligned for cp.async.16
  int4 wo[NB];                    // u16 warp-block code offsets of the tile
  uint64_t full[NB], empty[NB];   // mbarrier pipeline (OPT & 16)
};
static_assert(sizeof(double) * 2 * 512 % 16 == 0 && (kPipeCodeCap / 2 + 4) % 4 == 0 &&
                  (2048 / 2 + 4) % 4 == 0,
              "PipeSmem members must stay 16-byte aligned");

__device__ __forceinline__ int meta_nu(const int4& m) { return m.z & 0xffff; }

template <int CAP, bool FILL = true, int OPT = 0, typename SM>
__device__ __forceinline__ void pipe_issue(SM& S, int b, int tile, const int4& m,
                                           const int (&ids)[CAP / kEB],
                                           const int (&sl)[CAP / kEB],
                                           const double2* __restrict__ mxy,
                                           const double* __restrict__ mz,
                                           const uint8_t* __restrict__ rcodes,
                                           const int4* __restrict__ meta) {
  const int t = threadIdx.x;
  const int nu = meta_nu(m);
  if (FILL && nu <= CAP) {
#pragma unroll
    for (int u = 0; u < CAP / kEB; ++u) {
      // OPT & 32: thread i copies the i-th smallest rank into its slot
      // (coalesced sources); else slot i's rank (recoloured tables have holes)
      const int i = (OPT & 32) ? sl[u] : t + u * kEB;
      if (((OPT & 32) || i < nu) && ids[u] >= 0) {
        if (OPT & 1) cp_async16_cg(&S.xy[b][i], mxy + ids[u]);
        else cp_async16(&S.xy[b][i], mxy + ids[u]);
        cp_async8(&S.z[b][i], mz + ids[u]);
      }
    }
  }
  if (m.y <= SM::kCodeBytes) {
    // code blocks are multiples of 32 bytes: 16-byte pieces
    const uint4* src = reinterpret_cast<const uint4*>(rcodes + 32 * static_cast<i64>(m.x));
    for (int w = t; w < m.y / 16; w += kEB) {
      if (OPT & 1) cp_async16_cg(&S.cd[b][4 * w], src + w);
      else cp_async16(&S.cd[b][4 * w], src + w);
    }
  }
  if (t == 0) cp_async16(&S.wo[b], meta + 2 * tile + 1);
}

// node ids and this thread's edge id of `tile` into registers (always the
// full CAP window: the tile list has a fixed stride, so no dependency on the
// tile's metadata).
template <int NI, bool SF = false>
__device__ __forceinline__ void pipe_ids(int tile, int ntiles, const int32_t* __restrict__ tnodes,
                                         const int32_t* __restrict__ eperm, i64 ne,
                                         int (&ids)[NI], int (&sl)[NI], int& eid) {
  if (tile < ntiles) {
    const int32_t* tn = tnodes + static_cast<i64>(tile) * kTileNodeCap;
    if constexpr (SF) {  // sorted fill list of a coloured 256-node table (rings.cu)
      static_assert(NI == 1, "sorted fill lists hold 256 nodes");
      ids[0] = __ldg(tn + kTileFillRanks + threadIdx.x);
      sl[0] = __ldg(reinterpret_cast<const uint8_t*>(tn + kTileFillSlots) + threadIdx.x);
    } else {
#pragma unroll
      for (int u = 0; u < NI; ++u) ids[u] = __ldg(tn + threadIdx.x + u * kEB);
    }
    const i64 p = static_cast<i64>(tile) * kEB + threadIdx.x;
    eid = p < ne ? __ldg(eperm + p) : 0;
  }
}

// One lane's view of its warp block of ring codes (rings.cu): W == 2: 16-bit
// words, step s at word s*32 + lane (word 0 = slot(j) | sign << 15, word 1 =
// slot(k) | n << 11); W == 1: a header byte n | sign << 5 | boundary << 6 per
// lane, then one slot byte per step at 32 + s*32 + lane.
template <int W>
struct RingCodes {
  const uint8_t* __restrict__ blk;
  int lane;
  __device__ __forceinline__ unsigned raw(int s) const {
    if constexpr (W == 2) return reinterpret_cast<const uint16_t*>(blk)[s * 32 + lane];
    else return blk[32 + s * 32 + lane];
  }
  __device__ __forceinline__ unsigned slot(int s) const {
    return W == 2 && s < 3 ? (raw(s) & 0x7ffu) : raw(s);
  }
  __device__ __forceinline__ int count() const {
    if constexpr (W == 2) return static_cast<int>(raw(1) >> 11);
    else return blk[lane] & 31;
  }
  __device__ __forceinline__ bool negative() const {
    if constexpr (W == 2) return (raw(0) & 0x8000u) != 0;
    else return (blk[lane] & 32) != 0;
  }
  // closed ring: its last slot repeats m_0 (rings.cu k_ring_codes)
  __device__ __forceinline__ bool closed() const {
    if constexpr (W == 2) return (raw(0) & 0x4000u) != 0;
    else return (blk[lane] & 128) != 0;
  }
};

// Walks one edge's ring; T(slot) returns the node record of a tile slot.
// x_j is not needed by the walk; the caller reads it afterwards (fewer live
// registers across the loop).  (Keeping d_0 in registers instead of
// re-reading m_0 for a closed ring's last term measured 10 % slower: the six
// extra registers cost the loop its unrolling.)
// SIGNED = false leaves the ring orientation to the caller, which folds it
// into the 1/12 scale ((-a) * f == a * (-f) exactly: the same bits).
// U: unrolling of the ring loop.  The row-tile kernel is fastest at 4 (C5:
// 1.42 ms; 1.44 / 1.47 / 1.49 ms at 2 / 3 / 1); the Morton-tile kernel at 2 --
// left to itself ptxas unrolls its fused-multiply-add loop by 8, whose
// remainder chain costs rings of 3..11 steps more than it saves (C3: 0.558 ms
// at 2 against 0.594 / 0.664 / 0.600 / 0.709 at 1 / 3 / 4 / 6; the 2-3-flipped
// grid 0.629 against 0.647 / 0.665 / 0.698 / 0.749; profiles/r2_ncu_summary.md).
template <bool SIGNED = true, int U = 0, typename CT, typename TabFn>
__device__ __forceinline__ void ring_walk(const TabFn& T, const CT& C, double* acc, d4& xk) {
  const int n = C.count();
  xk = T(C.slot(1));
  const d4 mp = T(C.slot(2));
  double dx = mp.x - xk.x, dy = mp.y - xk.y, dz = mp.z - xk.z;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  auto step = [&](int i) {
    const d4 m = T(C.raw(3 + i));
    const double ex = m.x - xk.x, ey = m.y - xk.y, ez = m.z - xk.z;
    // cross(d, e) accumulated as two fused multiply-adds per component (6 FP64
    // instructions per step instead of 9; the FP64 pipe is ~40 % busy):
    // C5 element loop 1.513 -> 1.446 ms, still <= 1e-12 of the serial oracle
    a0 = __fma_rn(-dz, ey, __fma_rn(dy, ez, a0));
    a1 = __fma_rn(-dx, ez, __fma_rn(dz, ex, a1));
    a2 = __fma_rn(-dy, ex, __fma_rn(dx, ey, a2));
    dx = ex;
    dy = ey;
    dz = ez;
  };
  if constexpr (U == 0) {  // the compiler's own choice
    for (int i = 0; i < n; ++i) step(i);
  } else {
#pragma unroll U
    for (int i = 0; i < n; ++i) step(i);
  }
  if constexpr (SIGNED) {
    const bool neg = C.negative();
    acc[0] = neg ? -a0 : a0;
    acc[1] = neg ? -a1 : a1;
    acc[2] = neg ? -a2 : a2;
  } else {
    acc[0] = a0;
    acc[1] = a1;
    acc[2] = a2;
  }
}

// Traditional median-dual terms along the
// same ring: element i = {j, k, m_i, m_i+1} contributes
//   c_i = (E_i - m) x (F_i - m) + (F_i+1 - m) x (E_i - m),  negated if
//   c_i . (x_k - x_j) < 0,
// with m the edge midpoint, E_i the element centroid and F_i the centroid of
// the face {j, m_i, k}; each face centroid is shared by consecutive elements,
// so an incidence again needs one new node.  Which of the two faces is "L"
// does not matter (swapping them negates c exactly and the sign rule undoes
// it).  The centroids are summed from S = x_j + x_k (= 2m exactly) instead of
// in local order, so results are within rounding of the serial loop (<= 1e-12
// per edge vector), not bitwise; x_j / x_k are re-read by the caller.
template <int U = 0, typename CT, typename TabFn>
__device__ __forceinline__ void ring_walk_trad(const TabFn& T, const CT& C, double* acc) {
  const int n = C.count();
  double mx, my, mz, ex, ey, ez;
  {
    const d4 xj = T(C.slot(0)), xk = T(C.slot(1));
    mx = (xj.x + xk.x) * 0.5;
    my = (xj.y + xk.y) * 0.5;
    mz = (xj.z + xk.z) * 0.5;
    ex = xk.x - xj.x;
    ey = xk.y - xj.y;
    ez = xk.z - xj.z;
  }
  d4 mp = T(C.slot(2));
  double fx = (2.0 * mx + mp.x) * (1.0 / 3.0) - mx;
  double fy = (2.0 * my + mp.y) * (1.0 / 3.0) - my;
  double fz = (2.0 * mz + mp.z) * (1.0 / 3.0) - mz;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  auto step = [&](int i) {
    const d4 m = T(C.raw(3 + i));
    const double gx = (2.0 * mx + m.x) * (1.0 / 3.0) - mx;
    const double gy = (2.0 * my + m.y) * (1.0 / 3.0) - my;
    const double gz = (2.0 * mz + m.z) * (1.0 / 3.0) - mz;
    const double cx = (2.0 * mx + mp.x + m.x) * 0.25 - mx;
    const double cy = (2.0 * my + mp.y + m.y) * 0.25 - my;
    const double cz = (2.0 * mz + mp.z + m.z) * 0.25 - mz;
    // cross(C, F) + cross(G, C) as one product and three fused multiply-adds
    // per component (<= 1e-12 of the serial loop, like the dual-free walk)
    double c0 = __fma_rn(cy, fz, __fma_rn(-cz, fy, __fma_rn(gy, cz, -(gz * cy))));
    double c1 = __fma_rn(cz, fx, __fma_rn(-cx, fz, __fma_rn(gz, cx, -(gx * cz))));
    double c2 = __fma_rn(cx, fy, __fma_rn(-cy, fx, __fma_rn(gx, cy, -(gy * cx))));
    if (c0 * ex + c1 * ey + c2 * ez < 0.0) {
      c0 = -c0;
      c1 = -c1;
      c2 = -c2;
    }
    a0 += c0;
    a1 += c1;
    a2 += c2;
    mp = m;
    fx = gx;
    fy = gy;
    fz = gz;
  };
  if constexpr (U == 0) {
    for (int i = 0; i < n; ++i) step(i);
  } else {
#pragma unroll U
    for (int i = 0; i < n; ++i) step(i);
  }
  acc[0] = a0;
  acc[1] = a1;
  acc[2] = a2;
}

// OPT bits (all give the same bits; C5 element-loop times, round 1):
//   1  the (x, y) table and code fill bypasses L1 (cp.async.cg: nothing a
//      tile fills is re-read through this SM's L1): 2.22 -> 2.17 ms
//   16 mbarrier full / empty pipeline instead of the tile barrier (NB = 3
//      only): 2.035 -> 2.015 ms
//   32 the table fill walks the tile's rank-ordered fill list (coloured
//      256-node plans only): 2.015 -> 1.99 ms
// NB = 3 buffers drop the end-of-tile barrier (PipeSmem): 2.17 -> 2.035 ms.
// The default launch is OPT = 49 (1 | 16 | 32), NB = 3.  Measured and
// dropped (profiles/): streaming stores, L1::no_allocate id loads, a TMA
// bulk code fill (no change), four or five buffers (slower: less L1).
template <int CAP, int MINB, int W, int ALGO, int OPT, int NB,
          int CCAP = (NB == 2 ? kPipeCodeCap : 2048)>
__global__ void __launch_bounds__(kEB, MINB)
    k_navs_ring_pipe(const int32_t* __restrict__ eperm, const uint8_t* __restrict__ rcodes,
                     const int32_t* __restrict__ tnodes, const int4* __restrict__ meta,
                     const double2* __restrict__ mxy, const double* __restrict__ mz,
                     Coords<3> X, i64 ne, int ntiles, bool pos_s, double* __restrict__ navs,
                     double* __restrict__ svals) {
  using SM = PipeSmem<CAP, NB, CCAP>;
  SM& S = *reinterpret_cast<SM*>(dm_smem);
  const int t = threadIdx.x;
  const int lane = t & 31;
  int tile = blockIdx.x;
  if (tile >= ntiles) return;
  const int G = gridDim.x;
  // OPT & 16: mbarrier pipeline (NB == 3) -- each thread's cp.async fills
  // arrive on full[buffer]; each warp arrives on empty[buffer] after its
  // evaluation; a warp waits only for the fill it reads and, before
  // refilling a buffer, for every warp to be done with its previous use
  constexpr bool MB = (OPT & 16) != 0;
  static_assert(!MB || NB >= 3, "the mbarrier pipeline uses three or more buffers");
  if (MB) {
    if (t == 0) {
      for (int i = 0; i < NB; ++i) {
        mbar_init(&S.full[i], kEB);
        mbar_init(&S.empty[i], kEB / 32);
      }
    }
    __syncthreads();
  }
  // prologue: tile 0 -> buffer 0; ids / metadata of tile 1 into registers
  int ids[CAP / kEB], sl[CAP / kEB];
  int e_nxt = 0;
  int4 m_cur = __ldg(meta + 2 * tile);
  pipe_ids<CAP / kEB, (OPT & 32) != 0>(tile, ntiles, tnodes, eperm, ne, ids, sl, e_nxt);
  int e_cur = e_nxt;
  pipe_issue<CAP, true, OPT>(S, 0, tile, m_cur, ids, sl, mxy, mz, rcodes, meta);
  if (MB) cp_async_mbar_arrive(&S.full[0]);
  else cp_async_commit();
  int4 m_nxt = tile + G < ntiles ? __ldg(meta + 2 * (tile + G)) : make_int4(0, 0, 0, 0);
  pipe_ids<CAP / kEB, (OPT & 32) != 0>(tile + G, ntiles, tnodes, eperm, ne, ids, sl, e_nxt);
  for (int it = 0; tile < ntiles; ++it, tile += G) {
    const int b = NB == 2 ? (it & 1) : it % NB;
    const int bn = NB == 2 ? (b ^ 1) : (b + 1 == NB ? 0 : b + 1);
    const int nxt = tile + G;
    if (nxt < ntiles) {
      // buffer bn's use (it + 1) / NB waits for its previous use to be read
      if (MB && it + 1 >= NB)
        mbar_wait(&S.empty[bn], static_cast<unsigned>((it + 1) / NB - 1) & 1u);
      pipe_issue<CAP, true, OPT>(S, bn, nxt, m_nxt, ids, sl, mxy, mz, rcodes, meta);
      if (MB) cp_async_mbar_arrive(&S.full[bn]);
    }
    if (!MB) cp_async_commit();
    const int4 m = m_cur;
    const int e = e_cur;
    // m.w (the tile's boundary slice start) is not read by this kernel.  This
    // use keeps the register allocation that fits 64 registers without
    // spills; ptxas still reuses the dead w lane of the 16-byte prefetch
    // while it is in flight, a wait the other warps hide (every way around
    // it measured slower, profiles/r1_ncu_summary.md)
    asm volatile("" ::"r"(m.w));
    m_cur = m_nxt;
    e_cur = e_nxt;
    m_nxt = nxt + G < ntiles ? __ldg(meta + 2 * (nxt + G)) : make_int4(0, 0, 0, 0);
    pipe_ids<CAP / kEB, (OPT & 32) != 0>(nxt + G, ntiles, tnodes, eperm, ne, ids, sl, e_nxt);
    if (MB) {
      mbar_wait(&S.full[b], static_cast<unsigned>(it / NB) & 1u);
    } else {
      cp_async_wait<1>();
      __syncthreads();
    }
    // ---- evaluate tile `tile` from buffer b
    const i64 p = static_cast<i64>(tile) * kEB + t;
    const bool valid = p < ne;
    double acc[3] = {0.0, 0.0, 0.0};
    d4 xj{}, xk{};
    if (valid) {
      const int warp = t >> 5;
      const unsigned wo = (reinterpret_cast<const unsigned*>(&S.wo[b])[warp >> 1] >>
                           (16 * (warp & 1))) & 0xffffu;
      const int32_t* tn = tnodes + static_cast<i64>(tile) * kTileNodeCap;
      if (meta_nu(m) <= CAP && m.y <= SM::kCodeBytes) {
        const double2* xy = S.xy[b];
        const double* zz = S.z[b];
        auto T = [&](unsigned i) -> d4 {
          const double2 v = xy[i];
          d4 r;
          r.x = v.x;
          r.y = v.y;
          r.z = zz[i];
          return r;
        };
        const RingCodes<W> C{reinterpret_cast<const uint8_t*>(S.cd[b]) + wo, lane};
        if constexpr (ALGO == kTraditional) {
          ring_walk_trad(T, C, acc);
          xk = T(C.slot(1));
        } else {
          ring_walk<true, (CAP == 256 ? 2 : 0)>(T, C, acc, xk);
        }
        xj = T(C.slot(0));
      } else {
        auto T = [&](unsigned i) -> d4 {
          const int r = __ldg(tn + i);
          const double2 v = __ldg(mxy + r);
          d4 q;
          q.x = v.x;
          q.y = v.y;
          q.z = __ldg(mz + r);
          return q;
        };
        const RingCodes<W> C{rcodes + 32 * static_cast<i64>(m.x) + wo, lane};
        if constexpr (ALGO == kTraditional) {
          ring_walk_trad(T, C, acc);
          xk = T(C.slot(1));
        } else {
          ring_walk<true, (CAP == 256 ? 2 : 0)>(T, C, acc, xk);
        }
        xj = T(C.slot(0));
      }
    }
    if (valid) {
      // scale pass; boundary edges get their facet terms (and s) from
      // k_ring_boundary, launched right after on the same stream
      double nv[3], s;
      edge_tail_values<3, ALGO>(X, p, acc, xj, xk, nullptr, 0u, 0u, nullptr, nv, s);
      svals[pos_s ? p : static_cast<i64>(e)] = s;  // rings.cu: vol_by_rank
      store_nav_row(navs, e, nv);
    }
    if (NB == 2) __syncthreads();  // buffer b is refilled next iteration
    if (MB) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[b]);
    }
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------ GATHER (row tiles)
// The 3D default for node numberings with spatial coherence (rowplan.cu).
// Persistent CTAs of kRowTile threads walk the row tiles blockIdx.x,
// blockIdx.x + gridDim.x, ...  Per tile, warp 0 issues TMA bulk copies of the
// next tile's node runs (straight from the caller's coordinates) and code
// block into the other buffer, completing on that buffer's mbarrier; each
// thread walks its edge's ring from the table, stages its navs row and s term
// in shared memory, and after the tile barrier thread 0 writes the tile's
// rows as two bulk stores (the <= 2 rows outside the 16-byte-aligned middle
// with plain stores).  Same arithmetic as k_navs_ring_pipe.
struct RowCodes {
  const uint8_t* __restrict__ st;  // step rows of the warp block
  int lane, hdr;
  __device__ __forceinline__ unsigned raw(int s) const { return st[s * 32 + lane]; }
  __device__ __forceinline__ unsigned slot(int s) const { return raw(s); }
  __device__ __forceinline__ int count() const { return hdr & 31; }
  __device__ __forceinline__ bool negative() const { return (hdr & 32) != 0; }
};

struct RowSmem {
  double tab[2][3 * kRowSlots];       // node records (x, y, z), 24 B per slot
  uint8_t cd[2][kRowCodeCap];         // tile header + warp code blocks
  double stg[2][3 * (kRowTile + 2)];  // staged navs rows (row r = e - e0 + (e0 & 1))
  double sst[2][kRowTile + 2];        // staged s terms
  uint64_t full[2];
};
static_assert(sizeof(double) * 3 * (kRowTile + 2) % 16 == 0 && (kRowTile + 2) * 8 % 16 == 0,
              "RowSmem members stay 16-byte aligned");

// Design notes (C5, element loop, profiles/r2_ncu_summary.md): 5 CTAs of 56
// registers beat 4 of 70 (1.55 vs 1.67 ms); a decoupled form without the tile
// barrier (rotating lane blocks, the last warp refilling and storing) and
// coalesced 16-byte stores from the stage instead of the bulk stores were
// both slower (1.79, 1.73 ms); a third stage buffer changed nothing.
template <int ALGO, int MINB>
__global__ void __launch_bounds__(kRowTile, MINB)
    k_navs_row(const int4* __restrict__ meta, const int2* __restrict__ runs,
               const uint8_t* __restrict__ rcodes, const double* __restrict__ X, int ntiles,
               double* __restrict__ navs, double* __restrict__ svals) {
  RowSmem& S = *reinterpret_cast<RowSmem*>(dm_smem);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int tile = blockIdx.x;
  if (tile >= ntiles) return;
  const int G = gridDim.x;
  if (t == 0) {
    mbar_init(&S.full[0], 1);
    mbar_init(&S.full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    fence_async_smem();
  }
  __syncthreads();
  // warp 0: node runs + code block of a tile into buffer b (one arrival with
  // the transaction bytes, then the copies)
  auto issue = [&](int b, const int4& m, const int2& rn) {
    const unsigned bytes = lane < m.z ? 24u * static_cast<unsigned>(rn.y & 0xffff) : 0u;
    const unsigned total = __reduce_add_sync(0xffffffffu, bytes) + static_cast<unsigned>(m.y);
    if (lane == 0) mbar_arrive_expect_tx(&S.full[b], total);
    __syncwarp();
    if (lane < m.z)
      bulk_g2s(&S.tab[b][3 * (rn.y >> 16)], X + 3 * static_cast<i64>(rn.x), bytes, &S.full[b]);
    if (lane == 0)
      bulk_g2s(S.cd[b], rcodes + 32 * static_cast<i64>(m.x), static_cast<unsigned>(m.y),
               &S.full[b]);
  };
  auto ld_runs = [&](int tl, int nr) -> int2 {  // tl: the tile's run block (meta .w)
    return lane < nr ? __ldg(runs + static_cast<i64>(tl) * kRowRuns + lane) : make_int2(0, 0);
  };
  int4 mA = make_int4(0, 0, 0, 0), mB = make_int4(0, 0, 0, 0);
  int2 rA = make_int2(0, 0);
  if (warp == 0) {
    const int4 m0 = __ldg(meta + tile);
    issue(0, m0, ld_runs(m0.w, m0.z));
    if (tile + G < ntiles) {
      mA = __ldg(meta + tile + G);
      rA = ld_runs(mA.w, mA.z);
    }
    if (tile + 2 * G < ntiles) mB = __ldg(meta + tile + 2 * G);
  }
  for (int it = 0; tile < ntiles; ++it, tile += G) {
    const int b = it & 1;
    const int nxt = tile + G;
    if (warp == 0) {
      // buffer b ^ 1 was last read by tile it - 1: every warp is past the
      // barrier that ended it
      if (nxt < ntiles) issue(b ^ 1, mA, rA);
      rA = nxt + G < ntiles ? ld_runs(mB.w, mB.z) : make_int2(0, 0);
      mA = mB;
      mB = nxt + 2 * G < ntiles ? __ldg(meta + nxt + 2 * G) : make_int4(0, 0, 0, 0);
    }
    mbar_wait(&S.full[b], static_cast<unsigned>(it >> 1) & 1u);
    const int* hd = reinterpret_cast<const int*>(S.cd[b]);
    const int e0 = hd[0], cnt = hd[1], sh = e0 & 1;
    if (t < cnt) {
      const unsigned wo = reinterpret_cast<const uint16_t*>(hd + 2)[warp];
      const uint8_t* blk = S.cd[b] + wo;
      const int off = blk[32 + lane];
      const RowCodes C{blk + 64, lane, blk[lane]};
      const double* tab = S.tab[b];
      auto T = [&](unsigned i) -> d4 {
        const double* q = tab + 3 * i;
        d4 r;
        r.x = q[0];
        r.y = q[1];
        r.z = q[2];
        r.w = 0.0;
        return r;
      };
      double acc[3];
      d4 xj, xk;
      double nv[3], s;
      if constexpr (ALGO == kTraditional) {
        ring_walk_trad<4>(T, C, acc);  // C5: 3.18 -> 3.10 ms (2: 3.18, 1: 3.35)
        xk = T(C.slot(1));
        xj = T(C.slot(0));
        edge_tail_values<3, ALGO>(Coords<3>{nullptr}, 0, acc, xj, xk, nullptr, 0u, 0u, nullptr, nv, s);
      } else {
        // the ring's orientation rides on the 1/12 scale (same bits as
        // edge_tail_values on the signed sums, three fewer FP64 negations)
        ring_walk<false, 4>(T, C, acc, xk);
        xj = T(C.slot(0));
        const double f = C.negative() ? -(1.0 / 12.0) : (1.0 / 12.0);
        nv[0] = acc[0] * f;
        nv[1] = acc[1] * f;
        nv[2] = acc[2] * f;
        s = (xk.x - xj.x) * nv[0] + (xk.y - xj.y) * nv[1];
        s = s + (xk.z - xj.z) * nv[2];
      }
      const int r = off + sh;
      double* row = S.stg[b] + 3 * r;
      row[0] = nv[0];
      row[1] = nv[1];
      row[2] = nv[2];
      S.sst[b][r] = s;
    }
    fence_async_smem();
    if (t == 0) bulk_wait_read<0>();  // the previous tile's stores have read their stage
    __syncthreads();
    if (t == 0) {
      const int a = e0 + sh, end = e0 + cnt, bend = end & ~1;
      if (bend > a) {
        bulk_s2g(navs + 3 * static_cast<i64>(a), S.stg[b] + 3 * (a - e0 + sh),
                 24u * static_cast<unsigned>(bend - a));
        bulk_s2g(svals + a, S.sst[b] + (a - e0 + sh), 8u * static_cast<unsigned>(bend - a));
      }
      bulk_commit();
      auto plain = [&](int e) {
        const int r = e - e0 + sh;
        navs[3 * static_cast<i64>(e)] = S.stg[b][3 * r];
        navs[3 * static_cast<i64>(e) + 1] = S.stg[b][3 * r + 1];
        navs[3 * static_cast<i64>(e) + 2] = S.stg[b][3 * r + 2];
        svals[e] = S.sst[b][r];
      };
      if (sh) plain(e0);
      if ((end & 1) && end - 1 >= a) plain(end - 1);
    }
  }
  if (t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------ side list of the ring path
// Edges the ring codes cannot describe (rings.cu / rowplan.cu side list:
// more than kRingMax incidences, non-manifold or inconsistently oriented
// fans): one thread per edge folds its incident elements in ascending id --
// the serial loop's order, so these rows are bitwise the oracle's -- and
// overwrites the zero row the ring kernel wrote; the boundary pass follows.
// A warp per edge: lane q evaluates incidences q, q + 32, ... (all loads in
// flight at once), lane 0 then adds the terms in incidence order.
template <int ALGO>
__global__ void __launch_bounds__(128)
    k_navs_side(const int2* __restrict__ side, i64 n, const int2* __restrict__ edges,
                const int32_t* __restrict__ inc_ptr, const int32_t* __restrict__ inc,
                const int32_t* __restrict__ el, Coords3R X, bool pos_s,
                double* __restrict__ navs, double* __restrict__ svals) {
  __shared__ double term[4][32][3];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const i64 i = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;  // warp-uniform
  const int2 sp = side[i];  // {edge id, position}
  const int e = sp.x;
  const int2 jk = edges[e];
  const int q0 = inc_ptr[e], q1 = inc_ptr[e + 1];
  double acc[3] = {0.0, 0.0, 0.0};
  for (int b = q0; b < q1; b += 32) {
    const int q = b + lane;
    if (q < q1) {
      const int4 t = __ldg(reinterpret_cast<const int4*>(el) + inc[q]);
      const int ij = t.x == jk.x ? 0 : (t.y == jk.x ? 1 : (t.z == jk.x ? 2 : 3));
      double c0, c1, c2;
      if constexpr (ALGO == kDualFree) {
        df3(X, t.x, t.y, t.z, t.w, ij, c0, c1, c2);
      } else {
        const int ik = t.x == jk.y ? 0 : (t.y == jk.y ? 1 : (t.z == jk.y ? 2 : 3));
        tr3(X, t.x, t.y, t.z, t.w, ij, ik, c0, c1, c2);
      }
      term[w][lane][0] = c0;
      term[w][lane][1] = c1;
      term[w][lane][2] = c2;
    }
    __syncwarp();
    if (lane == 0)
      for (int r = 0; r < 32 && b + r < q1; ++r) {
        acc[0] += term[w][r][0];
        acc[1] += term[w][r][1];
        acc[2] += term[w][r][2];
      }
    __syncwarp();
  }
  if (lane != 0) return;
  double nv[3], s;
  edge_tail_values<3, ALGO>(Coords<3>{nullptr}, e, acc, X[jk.x], X[jk.y], nullptr, 0u, 0u, nullptr,
                            nv, s);
  navs[3 * static_cast<i64>(e)] = nv[0];
  navs[3 * static_cast<i64>(e) + 1] = nv[1];
  navs[3 * static_cast<i64>(e) + 2] = nv[2];
  svals[pos_s ? static_cast<i64>(sp.y) : static_cast<i64>(e)] = s;
}

// ------------------------------------------------------------------ GATHER_FACES
// One thread per edge.  x_j, x_k live in registers; the thread walks its own
// slice of the face-list incidence in ascending element order, U entries at
// a time with all loads of a batch issued before any use (memory-level
// parallelism without shared memory or block barriers), and folds the
// contributions in registers.  The navs row is written coalesced by a warp
// shuffle transpose (lane l stores doubles l, l+32, l+64 of the warp's
// 32*D-double block).
template <int D, int ALGO, int U, int MINB>
__global__ void __launch_bounds__(kEB, MINB)
    k_navs_faces(const int2* __restrict__ edges, const int32_t* __restrict__ inc_ptr,
                  const int2* __restrict__ ifl, Coords<D> X, i64 ne,
                  const u64* __restrict__ bedge, const u32* __restrict__ tile_bptr,
                  const int32_t* __restrict__ bnd, double* __restrict__ navs,
                  double* __restrict__ svals) {
  const int lane = threadIdx.x & 31;
  const i64 e = static_cast<i64>(blockIdx.x) * kEB + threadIdx.x;
  const bool valid = e < ne;
  int pb = 0, pe = 0;
  int2 jk = make_int2(0, 0);
  if (valid) {
    jk = edges[e];
    pb = inc_ptr[e];
    pe = inc_ptr[e + 1];
  }
  const Pt<D> xj = X[jk.x], xk = X[jk.y];
  double acc[3] = {0.0, 0.0, 0.0};
  for (int q0 = pb; q0 < pe; q0 += U) {
    int2 f[U];
#pragma unroll
    for (int u = 0; u < U; ++u) f[u] = q0 + u < pe ? __ldg(ifl + q0 + u) : make_int2(0, 0);
    Pt<D> xl[U], xr[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (q0 + u < pe) {
        xl[u] = X[f[u].x & kNodeMask];
        if constexpr (D == 3) xr[u] = X[f[u].y & kNodeMask];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (q0 + u < pe) {
        double c[3];
        const int ij = static_cast<unsigned>(f[u].x) >> 30;
        const int ik = static_cast<unsigned>(f[u].y) >> 30;
        if constexpr (D == 3) face_contrib3<ALGO>(ij, ik, xj, xk, xl[u], xr[u], c[0], c[1], c[2]);
        else face_contrib2<ALGO>(ij, ik, xj, xk, xl[u], c[0], c[1]);
#pragma unroll
        for (int d = 0; d < D; ++d) acc[d] += c[d];
      }
    }
  }
  double n[3] = {0.0, 0.0, 0.0};
  double s = 0.0;
  if (valid) {
    edge_tail_values<D, ALGO>(X, e, acc, xj, xk, bedge,
                              ALGO == kDualFree ? tile_bptr[blockIdx.x] : 0u,
                              ALGO == kDualFree ? tile_bptr[blockIdx.x + 1] : 0u, bnd, n, s);
    svals[e] = s;
  }
  store_navs_warp<D>(n, e - lane, ne, navs);
}

// ------------------------------------------------------------------ GATHER_ELEM
template <int D, int ALGO>
__global__ void __launch_bounds__(kEB)
    k_navs_gather_elem(const int2* __restrict__ edges, const int32_t* __restrict__ inc_ptr,
                       const int32_t* __restrict__ inc, const int32_t* __restrict__ el,
                       Coords<D> X, i64 ne, const u64* __restrict__ bedge,
                       const u32* __restrict__ tile_bptr, const int32_t* __restrict__ bnd,
                       double* __restrict__ navs, double* __restrict__ svals) {
  __shared__ int s_j[kEB], s_k[kEB];
  __shared__ unsigned char s_le[kCH];
  __shared__ double s_c[D][kCH];

  const int t = threadIdx.x;
  const i64 e0 = static_cast<i64>(blockIdx.x) * kEB;
  const i64 e1 = (e0 + kEB < ne) ? e0 + kEB : ne;
  const i64 e = e0 + t;
  const bool valid = e < ne;
  int j = 0, k = 0, pb = 0, pe = 0;
  if (valid) {
    const int2 jk = edges[e];
    j = jk.x;
    k = jk.y;
    pb = inc_ptr[e];
    pe = inc_ptr[e + 1];
  }
  s_j[t] = j;
  s_k[t] = k;
  const int P0 = __ldg(inc_ptr + e0), P1 = __ldg(inc_ptr + e1);
  __syncthreads();
  double acc[3] = {0.0, 0.0, 0.0};
  for (int c0 = P0; c0 < P1; c0 += kCH) {
    const int c1 = (c0 + kCH < P1) ? c0 + kCH : P1;
    const int qb = pb > c0 ? pb : c0, qe = pe < c1 ? pe : c1;
    for (int q = qb; q < qe; ++q) s_le[q - c0] = static_cast<unsigned char>(t);
    __syncthreads();
    for (int q = c0 + t; q < c1; q += kEB) {
      const int le = s_le[q - c0];
      double c[3];
      contribution<D, ALGO>(X, el, __ldg(inc + q), s_j[le], s_k[le], c);
#pragma unroll
      for (int d = 0; d < D; ++d) s_c[d][q - c0] = c[d];
    }
    __syncthreads();
    for (int q = qb; q < qe; ++q) {
#pragma unroll
      for (int d = 0; d < D; ++d) acc[d] += s_c[d][q - c0];
    }
    __syncthreads();
  }
  if (!valid) return;
  edge_tail<D, ALGO>(X, e, acc, X[j], X[k], bedge,
                     ALGO == kDualFree ? tile_bptr[blockIdx.x] : 0u,
                     ALGO == kDualFree ? tile_bptr[blockIdx.x + 1] : 0u, bnd, navs, svals);
}

// ------------------------------------------------------------------ SCATTER
template <int D, int ALGO>
__global__ void __launch_bounds__(256)
    k_navs_scatter(const int32_t* __restrict__ el, Coords<D> X, i64 nE,
                   const int32_t* __restrict__ e2l, double* __restrict__ navs) {
  const i64 E = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (E >= nE) return;
  constexpr int L = D == 3 ? 6 : 3;
  int v[4];
  if constexpr (D == 3) {
    const int4 t4 = ld_i4(reinterpret_cast<const int4*>(el) + E);
    v[0] = t4.x; v[1] = t4.y; v[2] = t4.z; v[3] = t4.w;
  } else {
    v[0] = __ldg(el + 3 * E); v[1] = __ldg(el + 3 * E + 1); v[2] = __ldg(el + 3 * E + 2); v[3] = 0;
  }
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const unsigned p = D == 3 ? (kTetEdgePacked >> (4 * l)) : (kTriEdgePacked >> (4 * l));
    const int la = p & 3, lb = (p >> 2) & 3;
    const int a = v[la], b = v[lb];
    const int j = a < b ? a : b, k = a < b ? b : a;
    double c[3];
    contribution<D, ALGO>(X, el, static_cast<int>(E), j, k, c);
    const i64 id = __ldg(e2l + L * E + l);
#pragma unroll
    for (int d = 0; d < D; ++d) atomicAdd(navs + D * id + d, c[d]);
  }
}

// Warp-aggregated form (north_star (b)): for each local edge slot l the 32
// lanes (consecutive elements, which share many edges: the six Kuhn tets of a
// hex all hold its diagonal) group by edge id with __match_any_sync; the
// lowest lane of a group adds the group's terms (lane order) and issues one
// REDG.E.ADD.F64 per component for all of them.
template <int D, int ALGO>
__global__ void __launch_bounds__(256)
    k_navs_scatter_agg(const int32_t* __restrict__ el, Coords<D> X, i64 nE,
                       const int32_t* __restrict__ e2l, double* __restrict__ navs) {
  __shared__ double term[8][32][D];
  const i64 E = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool valid = E < nE;
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  constexpr int L = D == 3 ? 6 : 3;
  int v[4];
  if constexpr (D == 3) {
    const int4 t4 = ld_i4(reinterpret_cast<const int4*>(el) + E);
    v[0] = t4.x; v[1] = t4.y; v[2] = t4.z; v[3] = t4.w;
  } else {
    v[0] = __ldg(el + 3 * E); v[1] = __ldg(el + 3 * E + 1); v[2] = __ldg(el + 3 * E + 2); v[3] = 0;
  }
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const unsigned pk = D == 3 ? (kTetEdgePacked >> (4 * l)) : (kTriEdgePacked >> (4 * l));
    const int a = v[pk & 3], b = v[(pk >> 2) & 3];
    const int j = a < b ? a : b, k = a < b ? b : a;
    double c[3];
    contribution<D, ALGO>(X, el, static_cast<int>(E), j, k, c);
    const int id = __ldg(e2l + L * E + l);
    const unsigned grp = __match_any_sync(act, id);
#pragma unroll
    for (int d = 0; d < D; ++d) term[w][lane][d] = c[d];
    __syncwarp(act);
    if ((grp & ((1u << lane) - 1)) == 0) {  // group leader
      double s[3] = {0.0, 0.0, 0.0};
      for (unsigned g = grp; g; g &= g - 1) {
        const int r = __ffs(g) - 1;
#pragma unroll
        for (int d = 0; d < D; ++d) s[d] += term[w][r][d];
      }
#pragma unroll
      for (int d = 0; d < D; ++d) atomicAdd(navs + D * static_cast<i64>(id) + d, s[d]);
    }
    __syncwarp(act);
  }
}

template <int D, int ALGO>
__global__ void __launch_bounds__(kEB)
    k_edge_finalize(const int2* __restrict__ edges, Coords<D> X, i64 ne,
                    const u64* __restrict__ bedge, const u32* __restrict__ tile_bptr,
                    const int32_t* __restrict__ bnd, double* __restrict__ navs,
                    double* __restrict__ svals) {
  const i64 e = static_cast<i64>(blockIdx.x) * kEB + threadIdx.x;
  if (e >= ne) return;
  const int2 jk = edges[e];
  double acc[3] = {navs[D * e], navs[D * e + 1], D == 3 ? navs[D * e + 2] : 0.0};
  edge_tail<D, ALGO>(X, e, acc, X[jk.x], X[jk.y], bedge,
                     ALGO == kDualFree ? tile_bptr[blockIdx.x] : 0u,
                     ALGO == kDualFree ? tile_bptr[blockIdx.x + 1] : 0u, bnd, navs, svals);
}

// Boundary pass of the ring path, in two steps: (1) the facet terms
// fb * n_B once per facet (coalesced over the facet list), (2) one thread per
// segment of the position-keyed (p << 32 | facet) list, i.e. per boundary
// edge, adds its facets' terms in ascending facet id to the scaled navs row
// and recomputes s -- the same values added in the same order as the fused
// tail, so the same bits.
// Boundary pass of the ring path: one thread per boundary edge adds
// fb * n_B of its facets (ascending facet id) to the scaled row and recomputes
// s.  The facet terms are evaluated per edge from the facet's nodes (a
// separate per-facet pass measured 0.0025 ms slower at C5 for the same bits).
__global__ void __launch_bounds__(256)
    k_ring_boundary(const int4* __restrict__ seg, const u32* __restrict__ start, i64 ns,
                    const u64* __restrict__ bedge_p, Coords3R X, const int32_t* __restrict__ bnd,
                    bool pos_s, double* __restrict__ navs, double* __restrict__ svals) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= ns) return;
  const int4 g = seg[i];  // {e, j, k, p}
  const i64 e = g.x;
  const u32 q0 = start[i], q1 = start[i + 1];
  const d4 xj = X[g.y], xk = X[g.z];
  double n[3] = {navs[3 * e], navs[3 * e + 1], navs[3 * e + 2]};  // already scaled
  for (u32 q = q0; q < q1; ++q) {
    const i64 f = static_cast<i64>(bedge_p[q] & 0xffffffffu);
    constexpr double fb = 1.0 / 12.0;
    double b0, b1, b2;
    bnormal3(X, bnd + 3 * f, b0, b1, b2);
    n[0] += fb * b0;
    n[1] += fb * b1;
    n[2] += fb * b2;
  }
  double s = (xk.x - xj.x) * n[0] + (xk.y - xj.y) * n[1];
  s = s + (xk.z - xj.z) * n[2];
  navs[3 * e] = n[0];
  navs[3 * e + 1] = n[1];
  navs[3 * e + 2] = n[2];
  svals[pos_s ? static_cast<i64>(g.w) : e] = s;
}

template <int D>
__global__ void __launch_bounds__(256)
    k_svals(const int2* __restrict__ edges, Coords<D> X, i64 ne, const double* __restrict__ navs,
            double* __restrict__ svals) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int2 jk = edges[e];
  double s;
  if constexpr (D == 3) {
    const d4 xj = X[jk.x], xk = X[jk.y];
    s = (xk.x - xj.x) * navs[3 * e] + (xk.y - xj.y) * navs[3 * e + 1];
    s = s + (xk.z - xj.z) * navs[3 * e + 2];
  } else {
    const double2 xj = X[jk.x], xk = X[jk.y];
    s = (xk.x - xj.x) * navs[2 * e] + (xk.y - xj.y) * navs[2 * e + 1];
  }
  svals[e] = s;
}

template <int D>
Coords<D> coords_of(dm_ctx* c) {
  Coords<D> X;
  if constexpr (D == 3) X.p = c->x4.p;
  else X.p = reinterpret_cast<const double2*>(c->coords.p);
  return X;
}

template <int D, int ALGO>
int launch_navs(dm_ctx* c, int variant) {
  const Coords<D> X = coords_of<D>(c);
  const i64 ne = c->ne;
  const unsigned tiles = grid_for(ne, kEB);
  if (variant == DM_VARIANT_SCATTER) {
    tmark(c, 0);
    DM_CK(c, cudaMemsetAsync(c->navs.p, 0, sizeof(double) * D * ne, c->stream));
    // warp-aggregated atomics by default; DUALMESH_SCATTER_PLAIN=1: one
    // atomic per term (the ncu comparison in profiles/)
    static const bool plain = [] {
      const char* e = std::getenv("DUALMESH_SCATTER_PLAIN");
      return e && e[0] == '1';
    }();
    if (plain)
      DM_LAUNCH(c, (k_navs_scatter<D, ALGO>), grid_for(c->nE, 256), 256, 0, c->elems.p, X, c->nE,
                c->e2l.p, c->navs.p);
    else
      DM_LAUNCH(c, (k_navs_scatter_agg<D, ALGO>), grid_for(c->nE, 256), 256, 0, c->elems.p, X,
                c->nE, c->e2l.p, c->navs.p);
    tmark(c, 1);
    DM_LAUNCH(c, (k_edge_finalize<D, ALGO>), tiles, kEB, 0, c->edges.p, X, ne, c->bedge.p,
              c->tile_bptr.p, c->bnd.p, c->navs.p, c->svals.p);
    tmark(c, 2);
  } else if (variant == DM_VARIANT_GATHER_ELEM) {
    tmark(c, 0);
    DM_LAUNCH(c, (k_navs_gather_elem<D, ALGO>), tiles, kEB, 0, c->edges.p, c->inc_ptr.p,
              c->inc.p, c->elems.p, X, ne, c->bedge.p, c->tile_bptr.p, c->bnd.p, c->navs.p,
              c->svals.p);
    tmark(c, 1);
    tmark(c, 2);
  } else if (variant == DM_VARIANT_GATHER && D == 3 && c->ring_ok && c->row_plan) {
    tmark(c, 0);
    if constexpr (D == 3) {
      auto launch = [&](auto kern) -> int {
        const int smem = static_cast<int>(sizeof(RowSmem));
        DM_CK(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int per_sm = 0, nsm = 0;
        DM_CK(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowTile, smem));
        DM_CK(c, cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
        const unsigned grid = static_cast<unsigned>(
            std::min<i64>(c->rt_ntiles, static_cast<i64>(nsm) * std::max(per_sm, 1)));
        DM_LAUNCH(c, kern, grid, kRowTile, smem, c->rt_meta.p, c->rt_runs.p, c->rcodes.p,
                  c->coords.p, static_cast<int>(c->rt_ntiles), c->navs.p, c->svals.p);
        return DM_OK;
      };
      int st = DM_OK;
      if (ALGO == kTraditional) st = launch(k_navs_row<kTraditional, 2>);
      else st = launch(k_navs_row<kDualFree, 5>);  // 56 registers, 5 x 35 KB shared
      if (st) return st;
      if (c->n_side > 0)  // one warp per side-list edge
        DM_LAUNCH(c, k_navs_side<ALGO>, grid_for(32 * c->n_side, 128), 128, 0, c->side.p,
                  c->n_side, c->edges.p, c->inc_ptr.p, c->inc.p, c->elems.p,
                  Coords3R{c->coords.p}, c->row_plan ? false : c->vol_by_rank, c->navs.p,
                  c->svals.p);
    }
    tmark(c, 1);
    if constexpr (D == 3 && ALGO == kDualFree) {
      if (c->n_bedge > 0) {
        DM_LAUNCH(c, k_ring_boundary, grid_for(c->n_bseg, 256), 256, 0, c->bseg.p,
                  c->bseg_start.p, c->n_bseg, c->bedge_p.p, Coords3R{c->coords.p}, c->bnd.p,
                  false, c->navs.p, c->svals.p);
      }
    }
    tmark(c, 2);
  } else if (variant == DM_VARIANT_GATHER && D == 3 && c->ring_ok) {
    tmark(c, 0);
    if constexpr (D == 3) {
      auto launch = [&](auto kern, int smem) -> int {
        DM_CK(c, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int per_sm = 0, nsm = 0;
        DM_CK(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kEB, smem));
        DM_CK(c, cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
        const unsigned grid = static_cast<unsigned>(std::min<i64>(
            static_cast<i64>(tiles), static_cast<i64>(nsm) * std::max(per_sm, 1)));
        DM_LAUNCH(c, kern, grid, kEB, smem, c->eperm.p, c->rcodes.p, c->tnodes.p,
                  c->ring_meta.p, c->mxy.p, c->mz.p, X, ne, static_cast<int>(tiles),
                  c->vol_by_rank, c->navs.p, c->svals.p);
        return DM_OK;
      };
      int st = DM_OK;
      // the code width and the table size follow the plan (8-bit codes and a
      // 256-node table when every tile fits, else 16-bit codes, 512 nodes)
      using S3 = PipeSmem<256, 3, 2048>;
      if (ALGO == kTraditional) {  // ~30 live doubles in the walk: 2 CTAs/SM, no spills
        st = c->code_width == 1
                 ? launch(k_navs_ring_pipe<256, 2, 1, kTraditional, 17, 3>, sizeof(S3))
                 : launch(k_navs_ring_pipe<512, 2, 2, kTraditional, 1, 2>, sizeof(PipeSmem<512>));
      } else if (c->code_width == 1) {
        if (c->gather_cfg == 41)  // test hook: a 16-code shared buffer sends every
                                  // tile down the global-memory path of the kernel
          st = launch(k_navs_ring_pipe<256, 4, 1, kDualFree, 49, 3, 16>, sizeof(PipeSmem<256, 3, 16>));
        else if (c->plan_colored)  // coloured plans carry the rank-ordered fill list (OPT & 32)
          st = launch(k_navs_ring_pipe<256, 4, 1, kDualFree, 49, 3>, sizeof(S3));
        else
          st = launch(k_navs_ring_pipe<256, 4, 1, kDualFree, 17, 3>, sizeof(S3));
      } else {
        st = launch(k_navs_ring_pipe<512, 4, 2, kDualFree, 1, 2>, sizeof(PipeSmem<512>));
      }
      if (st) return st;
      if (c->n_side > 0)  // one warp per side-list edge
        DM_LAUNCH(c, k_navs_side<ALGO>, grid_for(32 * c->n_side, 128), 128, 0, c->side.p,
                  c->n_side, c->edges.p, c->inc_ptr.p, c->inc.p, c->elems.p,
                  Coords3R{c->coords.p}, c->row_plan ? false : c->vol_by_rank, c->navs.p,
                  c->svals.p);
    }
    tmark(c, 1);
    if constexpr (D == 3 && ALGO == kDualFree) {
      if (c->n_bedge > 0) {
        DM_LAUNCH(c, k_ring_boundary, grid_for(c->n_bseg, 256), 256, 0, c->bseg.p,
                  c->bseg_start.p, c->n_bseg, c->bedge_p.p, Coords3R{c->coords.p}, c->bnd.p,
                  c->vol_by_rank, c->navs.p, c->svals.p);
      }
    }
    tmark(c, 2);
  } else if (variant == DM_VARIANT_GATHER_FACES || !c->table_ok || ALGO != kDualFree ||
             (D == 2 && variant == DM_VARIANT_GATHER)) {
    // face-list gather: traditional algorithm, meshes with node degree > 32,
    // and the 2D default (<= 2 incidences per edge, one opposite node each:
    // 2.5x the row-table kernel at 33.5 M triangles, and bitwise the serial
    // order like it)
    if (int sf = ensure_ifl(c)) return sf;
    tmark(c, 0);
#define DM_FACES(U, MINB)                                                                     \
  DM_LAUNCH(c, (k_navs_faces<D, ALGO, U, MINB>), tiles, kEB, 0, c->edges.p, c->inc_ptr.p,      \
            c->ifl.p, X, ne, c->bedge.p, c->tile_bptr.p, c->bnd.p, c->navs.p, c->svals.p)
    DM_FACES(2, 3);
#undef DM_FACES
    tmark(c, 1);
    tmark(c, 2);
  } else {
    tmark(c, 0);
#define DM_TABLE(U, MINB)                                                                     \
  DM_LAUNCH(c, (k_navs_gather<D, U, MINB>), tiles, kEB, 0, c->edges.p, c->inc_ptr.p,           \
            c->codes.p, c->adj_ptr.p, c->adj.p, c->os.p, c->tile_meta.p, X, ne, c->bedge.p,  \
            c->tile_bptr.p, c->bnd.p, c->navs.p, c->svals.p)
    DM_TABLE(2, 3);
#undef DM_TABLE
    tmark(c, 1);
    tmark(c, 2);
  }
  return DM_OK;
}

}  // namespace

int svals_from_navs(dm_ctx* c) {
  if (int sx = ensure_x4(c)) return sx;
  if (c->dim == 3) {
    DM_LAUNCH(c, k_svals<3>, grid_for(c->ne, 256), 256, 0, c->edges.p, coords_of<3>(c), c->ne,
              c->navs.p, c->svals.p);
  } else {
    DM_LAUNCH(c, k_svals<2>, grid_for(c->ne, 256), 256, 0, c->edges.p, coords_of<2>(c), c->ne,
              c->navs.p, c->svals.p);
  }
  return DM_OK;
}

int navs_impl(dm_ctx* c, int algo, int variant) {
  if (!c->have_edges) return fail(c, DM_ERR_STATE, "navs requested before build_edges");
  if (algo != DM_NAV_TRADITIONAL && algo != DM_NAV_DUALFREE)
    return fail(c, DM_ERR_INVALID_ARG, "unknown nav algorithm");
  if (variant < DM_VARIANT_GATHER || variant > DM_VARIANT_GATHER_EXACT)
    return fail(c, DM_ERR_INVALID_ARG, "unknown nav variant");
  if (c->ne == 0) {  // a mesh without elements has no edges: empty fields
    DM_CK(c, c->navs.ensure(0));
    DM_CK(c, c->svals.ensure(0));
    c->svals_pos = false;
    c->have_navs = true;
    c->navs_algo = algo;
    c->have_vols = false;
    return DM_OK;
  }
  int st = ensure_bedge(c);
  if (st) return st;
  if (variant == DM_VARIANT_GATHER) {
    st = ensure_rings(c);
    if (st) return st;
  }
  if ((variant == DM_VARIANT_GATHER_EXACT ||
       (variant == DM_VARIANT_GATHER && !c->ring_ok && c->dim == 3)) &&
      algo == DM_NAV_DUALFREE) {
    st = ensure_tables(c);
    if (st) return st;
  }
  DM_CK(c, c->navs.ensure(static_cast<size_t>(c->dim * c->ne)));
  DM_CK(c, c->svals.ensure(static_cast<size_t>(c->ne)));
  if (c->dim == 3) {
    // every call reads the caller's coordinates: the ring walk's table source
    // (Morton-order copy) or the padded copy of the other kernels is rebuilt
    // here, inside the metrics step, never carried over from an earlier call
    // (the row-tile plan reads the caller's coordinates directly: no copy)
    if (!(variant == DM_VARIANT_GATHER && c->ring_ok && c->row_plan)) {
      st = variant == DM_VARIANT_GATHER && c->ring_ok ? refresh_ring_coords(c) : pad_x4(c);
      if (st) return st;
    }
    st = algo == DM_NAV_DUALFREE ? launch_navs<3, kDualFree>(c, variant)
                                 : launch_navs<3, kTraditional>(c, variant);
  } else {
    st = algo == DM_NAV_DUALFREE ? launch_navs<2, kDualFree>(c, variant)
                                 : launch_navs<2, kTraditional>(c, variant);
  }
  if (st) return st;
  c->svals_pos = variant == DM_VARIANT_GATHER && c->dim == 3 && c->ring_ok && !c->row_plan &&
                c->vol_by_rank;
  c->have_navs = true;
  c->navs_algo = algo;
  c->have_vols = false;
  return DM_OK;
}

}  // namespace dm
