// edges.cu -- K1: GPU edge extraction, bit-exact with the reference
// build_edges (proj/src/mesh.cpp:256-285) and EdgeList::edge_of
// (mesh.cpp:58-73), plus the element->local-edge map and the edge->element
// CSR incidence of north_star (a).
//
// Algorithm (MSD bucket sort instead of the reference's hash set + sort):
//   items     : one per (element e, local edge l) = L*N_E, local order of
//               mesh.cpp:17 (3D) / mesh.cpp:263-265 (2D)
//   bucket    : the origin j = min(a,b) of the pair (counting sort, atomics)
//   payload   : (k << 32) | (e*L + l), k = max(a,b)
//   per bucket: rank sort of the payloads -> (k, e*L+l) ascending, counting
//               the distinct k on the way
// The concatenated buckets are then sorted by (j, k, e) -- exactly the
// lexicographic edge order of the reference with, per edge, its incident
// elements in ascending id.  Atomic placement order is erased by the sort
// (payloads are unique), so every output is deterministic.
#include <cstdlib>

#include "dm_internal.cuh"

namespace dm {
namespace {

template <int D>
__device__ __forceinline__ void load_elem(const int32_t* el, i64 e, int* v) {
  if (D == 3) {
    int4 t = ld_i4(reinterpret_cast<const int4*>(el) + e);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
    v[0] = __ldg(el + 3 * e); v[1] = __ldg(el + 3 * e + 1); v[2] = __ldg(el + 3 * e + 2);
  }
}

template <int D>
__device__ __forceinline__ void local_edge(int l, int& la, int& lb) {
  const unsigned p = D == 3 ? (kTetEdgePacked >> (4 * l)) : (kTriEdgePacked >> (4 * l));
  la = p & 3;
  lb = (p >> 2) & 3;
}

// Count items per origin bucket.
template <int D>
__global__ void k_count(const int32_t* el, i64 nE, u32* cnt) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nE) return;
  constexpr int L = D == 3 ? 6 : 3;
  int v[4];
  load_elem<D>(el, e, v);
#pragma unroll
  for (int l = 0; l < L; ++l) {
    int la, lb;
    local_edge<D>(l, la, lb);
    const int a = v[la], b = v[lb];
    atomicAdd(cnt + (a < b ? a : b), 1u);
  }
}

template <int D>
__global__ void k_scatter(const int32_t* el, i64 nE, const u32* bstart, u32* fill, u64* out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nE) return;
  constexpr int L = D == 3 ? 6 : 3;
  int v[4];
  load_elem<D>(el, e, v);
#pragma unroll
  for (int l = 0; l < L; ++l) {
    int la, lb;
    local_edge<D>(l, la, lb);
    const int a = v[la], b = v[lb];
    const int j = a < b ? a : b, k = a < b ? b : a;
    const u32 pos = bstart[j] + atomicAdd(fill + j, 1u);
    out[pos] = (static_cast<u64>(static_cast<u32>(k)) << 32) | static_cast<u64>(e * L + l);
  }
}

// Face-list incidence entry for element E seen from its local edge l:
//   x = node at il | ij << 30,  y = node at ir | ik << 30   (3D)
//   x = node at im | ij << 30,  y = ik << 30                 (2D)
// where ij / ik are the local slots of the origin j = min and of k, and
// il < ir (3D) / im (2D) are the remaining local slots.  With x_j and x_k
// known per edge, this is everything the dual-free and traditional
// contributions need (geometry.cuh), in the reference's local order.
template <int D>
__device__ __forceinline__ int2 make_ifl(const int32_t* el, int E, int l) {
  int v[4];
  load_elem<D>(el, E, v);
  int la, lb;
  local_edge<D>(l, la, lb);
  const int ij = v[la] < v[lb] ? la : lb, ik = v[la] < v[lb] ? lb : la;
  if (D == 3) {
    const unsigned rest = 0xFu & ~((1u << ij) | (1u << ik));
    const int il = __ffs(rest) - 1, ir = __ffs(rest & (rest - 1)) - 1;
    return make_int2(v[il] | (ij << 30), v[ir] | (ik << 30));
  }
  const int im = 3 - la - lb;
  return make_int2(v[im] | (ij << 30), ik << 30);
}

// Warp per bucket: emit edges, inc_ptr, inc and e2l.  Each chunk's items
// are loaded before the previous chunk is stored, and each item's
// predecessor comes by shuffle.
template <int L>
__global__ void k_emit(const u64* __restrict__ items, const u32* __restrict__ bstart,
                       const u32* __restrict__ os, i64 nv, int2* __restrict__ edges,
                       int32_t* __restrict__ inc_ptr, int32_t* __restrict__ inc,
                       int32_t* __restrict__ e2l) {
  constexpr unsigned F = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const i64 j = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (j >= nv) return;
  const u32 b = bstart[j], n = bstart[j + 1] - b;
  u32 id_base = os[j];  // edge id of the first head in this chunk
  u64 nxt = lane < n ? items[b + lane] : 0;
  u32 prev_hi = ~0u;  // high word of the item before this chunk
  for (u32 i0 = 0; i0 < n; i0 += 32) {
    const u32 i = i0 + lane;
    const u64 it = nxt;
    if (i0 + 32 < n) nxt = i + 32 < n ? items[b + i + 32] : 0;
    const u32 hi = static_cast<u32>(it >> 32);
    u32 up = __shfl_up_sync(F, hi, 1);
    if (lane == 0) up = prev_hi;
    prev_hi = __shfl_sync(F, hi, 31);
    const bool head = i < n && (i == 0 || hi != up);
    const unsigned hm = __ballot_sync(F, head);
    if (i < n) {
      // heads at or before this lane within the chunk
      const int before = __popc(hm & (0xffffffffu >> (31 - lane)));
      const int32_t id = static_cast<int32_t>(id_base + before - 1);
      const u32 val = static_cast<u32>(it);
      if (head) {
        edges[id] = make_int2(static_cast<int>(j), static_cast<int>(hi));
        inc_ptr[id] = static_cast<int32_t>(b + i);
      }
      inc[b + i] = static_cast<int32_t>(val / L);
      e2l[val] = id;
    }
    id_base += __popc(hm);
  }
}

// Face-list incidence, on demand (only the FACES / traditional fallbacks read
// it): thread per edge over its incidence slice.  The local edge l of slot q
// is recovered from the element's nodes -- the first local edge of element E
// joining (j, k) after the one of the previous slot if that slot was E too --
// so ifl[q] equals make_ifl(E, l) of the (E, l) item that K1 sorted into q.
template <int D>
__global__ void k_build_ifl(const int2* __restrict__ edges, const int32_t* __restrict__ inc_ptr,
                            const int32_t* __restrict__ inc, const int32_t* __restrict__ el,
                            i64 ne, int2* __restrict__ ifl) {
  constexpr int L = D == 3 ? 6 : 3;
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int2 jk = edges[e];
  int prevE = -1, prevl = -1;
  for (int q = inc_ptr[e]; q < inc_ptr[e + 1]; ++q) {
    const int E = inc[q];
    int v[4];
    load_elem<D>(el, E, v);
    int l = E == prevE ? prevl + 1 : 0;
    for (; l < L; ++l) {
      int la, lb;
      local_edge<D>(l, la, lb);
      const int a = v[la], b = v[lb];
      if ((a == jk.x && b == jk.y) || (a == jk.y && b == jk.x)) break;
    }
    ifl[q] = make_ifl<D>(el, E, l < L ? l : L - 1);
    prevE = E;
    prevl = l;
  }
}

__global__ void k_set_i32(int32_t* p, int32_t v) { *p = v; }

}  // namespace

int build_edges_impl(dm_ctx* c) {
  const int D = c->dim;
  const int L = D == 3 ? 6 : 3;
  const i64 M = static_cast<i64>(L) * c->nE;
  if (M >= (1ll << 31) || c->nv >= (1ll << 30))
    return fail(c, DM_ERR_UNSUPPORTED, "mesh exceeds the 32-bit item space of the device layout");
  c->have_edges = c->have_in = c->have_bedge = c->have_n2e = c->have_ifl = c->have_tables =
      c->have_rings = false;
  c->have_navs = c->have_vols = false;
  if (c->nE == 0) {
    // no elements: the reference returns an empty edge list whose origin CSR
    // is nv + 1 zeros (mesh.cpp:256-285)
    c->ne = 0;
    DM_CK(c, c->os.ensure(static_cast<size_t>(c->nv + 1)));
    DM_CK(c, cudaMemsetAsync(c->os.p, 0, (c->nv + 1) * sizeof(u32), c->stream));
    DM_CK(c, c->edges.ensure(0));
    DM_CK(c, c->inc_ptr.ensure(1));
    DM_CK(c, cudaMemsetAsync(c->inc_ptr.p, 0, sizeof(int32_t), c->stream));
    DM_CK(c, c->inc.ensure(0));
    DM_CK(c, c->e2l.ensure(0));
    DM_CK(c, cudaStreamSynchronize(c->stream));
    c->have_edges = true;
    return DM_OK;
  }
  // DUALMESH_K1_LEGACY=1: the item-sort path for every mesh (A/B and tests)
  const char* legacy = std::getenv("DUALMESH_K1_LEGACY");
  if (!(legacy && *legacy == '1')) {
    const int sb = build_edges_buckets(c);
    if (sb != kK1Unsupported) {
      c->have_edges = sb == DM_OK;
      return sb;
    }
  }
  const i64 nv = c->nv;

  DM_CK(c, c->cnt.ensure(static_cast<size_t>(nv + 1)));
  DM_CK(c, c->fill.ensure(static_cast<size_t>(nv + 1)));
  DM_CK(c, c->tmp64.ensure(static_cast<size_t>(M)));
  DM_CK(c, cudaMemsetAsync(c->cnt.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_CK(c, cudaMemsetAsync(c->fill.p, 0, (nv + 1) * sizeof(u32), c->stream));
  const unsigned ge = grid_for(c->nE, 256);
  if (D == 3) {
    DM_LAUNCH(c, k_count<3>, ge, 256, 0, c->elems.p, c->nE, c->cnt.p);
  } else {
    DM_LAUNCH(c, k_count<2>, ge, 256, 0, c->elems.p, c->nE, c->cnt.p);
  }
  int st = scan_exclusive(c, c->cnt.p, c->cnt.p, nv);  // cnt := bucket starts
  if (st) return st;
  if (D == 3) {
    DM_LAUNCH(c, k_scatter<3>, ge, 256, 0, c->elems.p, c->nE, c->cnt.p, c->fill.p, c->tmp64.p);
  } else {
    DM_LAUNCH(c, k_scatter<2>, ge, 256, 0, c->elems.p, c->nE, c->cnt.p, c->fill.p, c->tmp64.p);
  }
  // sort each bucket; fill := distinct k per bucket (edges per origin)
  st = segment_sort_unique_u64(c, c->tmp64.p, c->cnt.p, nv, c->fill.p);
  if (st) return st;
  DM_CK(c, c->os.ensure(static_cast<size_t>(nv + 1)));
  st = scan_exclusive(c, c->fill.p, c->os.p, nv);
  if (st) return st;
  u32 ne32 = 0;
  DM_CK(c, cudaMemcpyAsync(&ne32, c->os.p + nv, sizeof(u32), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  c->ne = ne32;
  DM_CK(c, c->edges.ensure(static_cast<size_t>(c->ne)));
  DM_CK(c, c->inc_ptr.ensure(static_cast<size_t>(c->ne + 1)));
  DM_CK(c, c->inc.ensure(static_cast<size_t>(M)));
  DM_CK(c, c->e2l.ensure(static_cast<size_t>(M)));
  if (D == 3) {
    DM_LAUNCH(c, k_emit<6>, grid_for(nv * 32, 256), 256, 0, c->tmp64.p, c->cnt.p, c->os.p, nv,
              c->edges.p, c->inc_ptr.p, c->inc.p, c->e2l.p);
  } else {
    DM_LAUNCH(c, k_emit<3>, grid_for(nv * 32, 256), 256, 0, c->tmp64.p, c->cnt.p, c->os.p, nv,
              c->edges.p, c->inc_ptr.p, c->inc.p, c->e2l.p);
  }
  DM_LAUNCH(c, k_set_i32, 1, 1, 0, c->inc_ptr.p + c->ne, static_cast<int32_t>(M));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  // tmp64 stays allocated: re-extraction (remeshing loops) must not pay a
  // cudaMalloc/cudaFree pair, which stalls the device for up to ~0.3 s
  c->have_edges = true;
  return DM_OK;
}

// ------------------------------------------------------------ derived CSRs
namespace {

// incoming edges: bucket by destination k, payload edge id
__global__ void k_in_count(const int2* edges, i64 ne, u32* cnt) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e < ne) atomicAdd(cnt + edges[e].y, 1u);
}
__global__ void k_in_scatter(const int2* edges, i64 ne, const u32* start, u32* fill, u32* out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int k = edges[e].y;
  out[start[k] + atomicAdd(fill + k, 1u)] = static_cast<u32>(e);
}

// node -> element: bucket by every node of every element, payload element id
template <int D>
__global__ void k_n2e_count(const int32_t* el, i64 nE, u32* cnt) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < nE * (D + 1)) atomicAdd(cnt + el[t], 1u);
}
template <int D>
__global__ void k_n2e_scatter(const int32_t* el, i64 nE, const u32* start, u32* fill, u32* out) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nE * (D + 1)) return;
  const int v = el[t];
  out[start[v] + atomicAdd(fill + v, 1u)] = static_cast<u32>(t / (D + 1));
}

// boundary (edge, facet) pairs: bucket by the edge's origin, payload (edge<<32 | b)
__device__ __forceinline__ int dev_edge_of(const int2* edges, const u32* os, i64 nv, int a, int b) {
  if (a > b) { int t = a; a = b; b = t; }
  if (a < 0 || a >= nv) return -1;
  u32 lo = os[a], hi = os[a + 1];
  const u32 end = hi;
  while (lo < hi) {
    const u32 mid = lo + (hi - lo) / 2;
    if (edges[mid].y < b) lo = mid + 1;
    else hi = mid;
  }
  return (lo < end && edges[lo].y == b) ? static_cast<int>(lo) : -1;
}

template <int D>
__global__ void k_bedge_count(const int32_t* bnd, i64 nB, const int2* edges, const u32* os, i64 nv,
                              u32* cnt, int* flag) {
  constexpr int NEB = D == 3 ? 3 : 1;
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nB * NEB) return;
  const i64 b = t / NEB;
  const int q = static_cast<int>(t % NEB);
  const int a = bnd[D * b + q], c = bnd[D * b + (q + 1) % D];
  const int id = dev_edge_of(edges, os, nv, a, c);
  if (id < 0) {
    atomicExch(flag, 1);
    return;
  }
  atomicAdd(cnt + (a < c ? a : c), 1u);
}
template <int D>
__global__ void k_bedge_scatter(const int32_t* bnd, i64 nB, const int2* edges, const u32* os,
                                i64 nv, const u32* start, u32* fill, u64* out) {
  constexpr int NEB = D == 3 ? 3 : 1;
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nB * NEB) return;
  const i64 b = t / NEB;
  const int q = static_cast<int>(t % NEB);
  const int a = bnd[D * b + q], c = bnd[D * b + (q + 1) % D];
  const int id = dev_edge_of(edges, os, nv, a, c);
  if (id < 0) return;
  const int j = a < c ? a : c;
  out[start[j] + atomicAdd(fill + j, 1u)] = (static_cast<u64>(id) << 32) | static_cast<u64>(b);
}

__global__ void k_edge_of(const int2* edges, const u32* os, i64 nv, const int32_t* a,
                          const int32_t* b, i64 n, int32_t* out) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = dev_edge_of(edges, os, nv, a[i], b[i]);
}

}  // namespace

// tile_bptr[t] = first entry of the sorted (key << 32 | facet) list whose key
// is >= t * kTileEdges (t = 0..ntiles).
__global__ void k_tile_bptr(const u64* bedge, u32 n, i64 ne, i64 ntiles, u32* tile_bptr) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t > ntiles) return;
  const i64 e = t * kTileEdges < ne ? t * kTileEdges : ne;
  u32 lo = 0, hi = n;
  while (lo < hi) {
    const u32 mid = (lo + hi) >> 1;
    if ((bedge[mid] >> 32) < static_cast<u64>(e)) lo = mid + 1;
    else hi = mid;
  }
  tile_bptr[t] = lo;
}


int ensure_incoming(dm_ctx* c) {
  if (c->have_in) return DM_OK;
  if (!c->have_edges) return fail(c, DM_ERR_STATE, "edges not built");
  const i64 nv = c->nv, ne = c->ne;
  DM_CK(c, c->in_ptr.ensure(static_cast<size_t>(nv + 1)));
  DM_CK(c, c->in_list.ensure(static_cast<size_t>(ne)));
  DM_CK(c, c->fill.ensure(static_cast<size_t>(nv + 1)));
  DM_CK(c, cudaMemsetAsync(c->in_ptr.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_CK(c, cudaMemsetAsync(c->fill.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_LAUNCH(c, k_in_count, grid_for(ne, 256), 256, 0, c->edges.p, ne, c->in_ptr.p);
  int st = scan_exclusive(c, c->in_ptr.p, c->in_ptr.p, nv);
  if (st) return st;
  DM_LAUNCH(c, k_in_scatter, grid_for(ne, 256), 256, 0, c->edges.p, ne, c->in_ptr.p, c->fill.p,
            reinterpret_cast<u32*>(c->in_list.p));
  st = segment_sort_u32(c, reinterpret_cast<u32*>(c->in_list.p), c->in_ptr.p, nv);
  if (st) return st;
  c->have_in = true;
  return DM_OK;
}

int ensure_ifl(dm_ctx* c) {
  if (c->have_ifl) return DM_OK;
  if (!c->have_edges) return fail(c, DM_ERR_STATE, "edges not built");
  const i64 L = c->dim == 3 ? 6 : 3;
  DM_CK(c, c->ifl.ensure(static_cast<size_t>(std::max<i64>(L * c->nE, 1))));
  if (c->dim == 3)
    DM_LAUNCH(c, k_build_ifl<3>, grid_for(c->ne, 256), 256, 0, c->edges.p, c->inc_ptr.p, c->inc.p,
              c->elems.p, c->ne, c->ifl.p);
  else
    DM_LAUNCH(c, k_build_ifl<2>, grid_for(c->ne, 256), 256, 0, c->edges.p, c->inc_ptr.p, c->inc.p,
              c->elems.p, c->ne, c->ifl.p);
  c->have_ifl = true;
  return DM_OK;
}

int ensure_n2e(dm_ctx* c) {
  if (c->have_n2e) return DM_OK;
  const i64 nv = c->nv, nt = c->nE * (c->dim + 1);
  DM_CK(c, c->n2e_ptr.ensure(static_cast<size_t>(nv + 1)));
  DM_CK(c, c->n2e.ensure(static_cast<size_t>(nt)));
  DM_CK(c, c->fill.ensure(static_cast<size_t>(nv + 1)));
  DM_CK(c, cudaMemsetAsync(c->n2e_ptr.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_CK(c, cudaMemsetAsync(c->fill.p, 0, (nv + 1) * sizeof(u32), c->stream));
  if (c->dim == 3) {
    DM_LAUNCH(c, k_n2e_count<3>, grid_for(nt, 256), 256, 0, c->elems.p, c->nE, c->n2e_ptr.p);
  } else {
    DM_LAUNCH(c, k_n2e_count<2>, grid_for(nt, 256), 256, 0, c->elems.p, c->nE, c->n2e_ptr.p);
  }
  int st = scan_exclusive(c, c->n2e_ptr.p, c->n2e_ptr.p, nv);
  if (st) return st;
  u32* out = reinterpret_cast<u32*>(c->n2e.p);
  if (c->dim == 3) {
    DM_LAUNCH(c, k_n2e_scatter<3>, grid_for(nt, 256), 256, 0, c->elems.p, c->nE, c->n2e_ptr.p,
              c->fill.p, out);
  } else {
    DM_LAUNCH(c, k_n2e_scatter<2>, grid_for(nt, 256), 256, 0, c->elems.p, c->nE, c->n2e_ptr.p,
              c->fill.p, out);
  }
  st = segment_sort_u32(c, out, c->n2e_ptr.p, nv);
  if (st) return st;
  c->have_n2e = true;
  return DM_OK;
}

int ensure_bedge(dm_ctx* c) {
  if (c->have_bedge) return DM_OK;
  if (!c->have_edges) return fail(c, DM_ERR_STATE, "edges not built");
  const int D = c->dim;
  const int NEB = D == 3 ? 3 : 1;
  const i64 nv = c->nv, n = c->nB * NEB;
  DM_CK(c, c->cnt.ensure(static_cast<size_t>(nv + 1)));
  DM_CK(c, c->fill.ensure(static_cast<size_t>(nv + 1)));
  DM_CK(c, c->bedge.ensure(static_cast<size_t>(n)));
  DM_CK(c, c->flag.ensure(4));
  DM_CK(c, cudaMemsetAsync(c->cnt.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_CK(c, cudaMemsetAsync(c->fill.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_CK(c, cudaMemsetAsync(c->flag.p, 0, sizeof(int), c->stream));
  if (D == 3) {
    DM_LAUNCH(c, k_bedge_count<3>, grid_for(n, 256), 256, 0, c->bnd.p, c->nB, c->edges.p, c->os.p,
              nv, c->cnt.p, c->flag.p);
  } else {
    DM_LAUNCH(c, k_bedge_count<2>, grid_for(n, 256), 256, 0, c->bnd.p, c->nB, c->edges.p, c->os.p,
              nv, c->cnt.p, c->flag.p);
  }
  int f = 0;
  int st = read_flag(c, &f);
  if (st) return st;
  if (f)
    return fail(c, DM_ERR_EDGE_ABSENT, "boundary element references an edge absent from EdgeList");
  st = scan_exclusive(c, c->cnt.p, c->cnt.p, nv);
  if (st) return st;
  if (D == 3) {
    DM_LAUNCH(c, k_bedge_scatter<3>, grid_for(n, 256), 256, 0, c->bnd.p, c->nB, c->edges.p,
              c->os.p, nv, c->cnt.p, c->fill.p, c->bedge.p);
  } else {
    DM_LAUNCH(c, k_bedge_scatter<2>, grid_for(n, 256), 256, 0, c->bnd.p, c->nB, c->edges.p,
              c->os.p, nv, c->cnt.p, c->fill.p, c->bedge.p);
  }
  st = segment_sort_unique_u64(c, c->bedge.p, c->cnt.p, nv, nullptr);
  if (st) return st;
  // per-tile slices of the sorted (edge, facet) list, so no kernel searches it
  const i64 ntiles = (c->ne + kTileEdges - 1) / kTileEdges;
  DM_CK(c, c->tile_bptr.ensure(static_cast<size_t>(ntiles + 1)));
  DM_LAUNCH(c, k_tile_bptr, grid_for(ntiles + 1, 256), 256, 0, c->bedge.p, static_cast<u32>(n),
            c->ne, ntiles, c->tile_bptr.p);
  c->n_bedge = n;
  c->have_bedge = true;
  return DM_OK;
}

}  // namespace dm

// ------------------------------------------------------------ C-ABI pieces
extern "C" int dm_edge_of(dm_ctx* c, const int32_t* a, const int32_t* b, int64_t n, int32_t* out) {
  using namespace dm;
  if (!c || (n > 0 && (!a || !b || !out)) || n < 0) return DM_ERR_INVALID_ARG;
  if (!c->have_edges) return fail(c, DM_ERR_STATE, "dm_edge_of before dm_build_edges");
  if (n == 0) return DM_OK;
  DevBuf<int32_t> da, db, dout;
  DM_CK(c, da.ensure(n));
  DM_CK(c, db.ensure(n));
  DM_CK(c, dout.ensure(n));
  DM_CK(c, cudaMemcpyAsync(da.p, a, n * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  DM_CK(c, cudaMemcpyAsync(db.p, b, n * sizeof(int32_t), cudaMemcpyHostToDevice, c->stream));
  DM_LAUNCH(c, k_edge_of, grid_for(n, 256), 256, 0, c->edges.p, c->os.p, c->nv, da.p, db.p, n,
            dout.p);
  DM_CK(c, cudaMemcpyAsync(out, dout.p, n * sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}
