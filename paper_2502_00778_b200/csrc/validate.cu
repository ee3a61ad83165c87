// validate.cu -- validate_mesh and derive_boundary_faces on the GPU
// (reference proj/src/mesh.cpp:129-254 and 287-323).
//
// Faces are keyed like the reference's FaceKey (sorted node ids,
// mesh.cpp:31-54) but found by a bucket sort instead of a hash map: every
// element face (e, i) -- the face opposite local node i in the reference's
// outward vertex order (mesh.cpp:15,97-110, 190-197) -- goes to the bucket of
// its smallest node with key (mid << 32 | max) and value e*(D+1)+i; each
// bucket is sorted by (key, value).  Equal keys are then contiguous with the
// lowest (element, face) first, which is the "first owner" the reference's
// try_emplace keeps.  Boundary facets are bucketed the same way (value b).
// Every check of the reference is then a per-item kernel; the offending ids
// are collected per violation class and the C++ layer formats the messages
// in the reference's order (host_api.cpp).
#include <algorithm>
#include <vector>

#include "dm_internal.cuh"

namespace dm {
namespace {

struct Faces {
  DevBuf<u32> fptr;  // face buckets, nv+1
  DevBuf<u64> fkey;
  DevBuf<u32> fval;  // e*(D+1)+i
  DevBuf<u32> bptr;  // boundary buckets, nv+1
  DevBuf<u64> bkey;
  DevBuf<u32> bval;  // boundary facet id
};

template <int D>
__device__ __forceinline__ void face_nodes(const int32_t* el, i64 e, int i, int* o) {
  // outward order of the face opposite local node i (ref mesh.cpp:97-110, 188-197)
  const int32_t* t = el + (D + 1) * e;
  if (D == 3) {
    const unsigned f = (kOppPacked >> (6 * i)) & 63u;
    o[0] = t[f & 3];
    o[1] = t[(f >> 2) & 3];
    o[2] = t[(f >> 4) & 3];
  } else {
    o[0] = t[(i + 1) % 3];
    o[1] = t[(i + 2) % 3];
    o[2] = 0;
  }
}

template <int D>
__device__ __forceinline__ void sorted_key(const int* o, int& a, u64& key) {
  int x = o[0], y = o[1], z = D == 3 ? o[2] : 0;
  if (D == 3) {
    if (x > y) { const int t = x; x = y; y = t; }
    if (y > z) { const int t = y; y = z; z = t; }
    if (x > y) { const int t = x; x = y; y = t; }
    a = x;
    key = (static_cast<u64>(static_cast<u32>(y)) << 32) | static_cast<u32>(z);
  } else {
    if (x > y) { const int t = x; x = y; y = t; }
    a = x;
    key = static_cast<u64>(static_cast<u32>(y)) << 32;
  }
}

__device__ __forceinline__ void push(i64* list, unsigned long long* cnt, i64 cap, i64 v) {
  const unsigned long long p = atomicAdd(cnt, 1ull);
  if (static_cast<i64>(p) < cap) list[p] = v;
}

template <int D>
__global__ void k_range(const int32_t* el, i64 nE, const int32_t* bnd, i64 nB, i64 nv, i64* lists,
                        i64 cap, unsigned long long* cnt) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < nE) {
    bool bad = false;
    for (int i = 0; i <= D; ++i) {
      const int v = el[(D + 1) * t + i];
      bad |= v < 0 || v >= nv;
    }
    if (bad) push(lists + DM_V_OUT_OF_RANGE_ELEM * cap, cnt + DM_V_OUT_OF_RANGE_ELEM, cap, t);
  } else if (t < nE + nB) {
    const i64 b = t - nE;
    bool bad = false;
    for (int i = 0; i < D; ++i) {
      const int v = bnd[D * b + i];
      bad |= v < 0 || v >= nv;
    }
    if (bad) push(lists + DM_V_OUT_OF_RANGE_BND * cap, cnt + DM_V_OUT_OF_RANGE_BND, cap, b);
  }
}

template <int D>
__global__ void k_signs(const int32_t* el, const double* x, i64 nE, int8_t* signs, i64* lists,
                        i64 cap, unsigned long long* cnt) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= nE) return;
  const int32_t* t = el + (D + 1) * e;
  double v;
  if (D == 2) {  // ref mesh.cpp:77-81
    const double *a = x + 2 * (i64)t[0], *b = x + 2 * (i64)t[1], *c = x + 2 * (i64)t[2];
    v = 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]));
  } else {  // ref mesh.cpp:83-91
    const double *a = x + 3 * (i64)t[0], *b = x + 3 * (i64)t[1], *c = x + 3 * (i64)t[2],
                 *d = x + 3 * (i64)t[3];
    double uv0, uv1, uv2;
    cross3(b[0] - a[0], b[1] - a[1], b[2] - a[2], c[0] - a[0], c[1] - a[1], c[2] - a[2], uv0, uv1,
           uv2);
    v = (uv0 * (d[0] - a[0]) + uv1 * (d[1] - a[1]) + uv2 * (d[2] - a[2])) / 6.0;
  }
  signs[e] = static_cast<int8_t>(v > 0.0 ? 1 : (v < 0.0 ? -1 : 0));
  if (!(v > 0.0)) push(lists + DM_V_NONPOSITIVE * cap, cnt + DM_V_NONPOSITIVE, cap, e);
}

template <int D>
__global__ void k_face_count(const int32_t* el, i64 nE, u32* cnt) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nE * (D + 1)) return;
  int o[3], a;
  u64 key;
  face_nodes<D>(el, t / (D + 1), static_cast<int>(t % (D + 1)), o);
  sorted_key<D>(o, a, key);
  atomicAdd(cnt + a, 1u);
}

template <int D>
__global__ void k_face_scatter(const int32_t* el, i64 nE, const u32* start, u32* fill, u64* keys,
                               u32* vals) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nE * (D + 1)) return;
  int o[3], a;
  u64 key;
  face_nodes<D>(el, t / (D + 1), static_cast<int>(t % (D + 1)), o);
  sorted_key<D>(o, a, key);
  const u32 p = start[a] + atomicAdd(fill + a, 1u);
  keys[p] = key;
  vals[p] = static_cast<u32>(t);
}

template <int D>
__global__ void k_bnd_count(const int32_t* bnd, i64 nB, u32* cnt) {
  const i64 b = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nB) return;
  int o[3] = {bnd[D * b], bnd[D * b + 1], D == 3 ? bnd[D * b + 2] : 0}, a;
  u64 key;
  sorted_key<D>(o, a, key);
  atomicAdd(cnt + a, 1u);
}

template <int D>
__global__ void k_bnd_scatter(const int32_t* bnd, i64 nB, const u32* start, u32* fill, u64* keys,
                              u32* vals) {
  const i64 b = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nB) return;
  int o[3] = {bnd[D * b], bnd[D * b + 1], D == 3 ? bnd[D * b + 2] : 0}, a;
  u64 key;
  sorted_key<D>(o, a, key);
  const u32 p = start[a] + atomicAdd(fill + a, 1u);
  keys[p] = key;
  vals[p] = static_cast<u32>(b);
}

// first index of key in bucket [lo, hi), or hi
__device__ __forceinline__ u32 find_key(const u64* keys, u32 lo, u32 hi, u64 key) {
  const u32 end = hi;
  while (lo < hi) {
    const u32 mid = (lo + hi) >> 1;
    if (keys[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return (lo < end && keys[lo] == key) ? lo : end;
}

// Face incidence > 2 (ref mesh.cpp:199-202): the 3rd, 4th, ... owners of a
// key in (element, face) order are reported (value = e*(D+1)+i).
template <int D>
__global__ void k_overshared(const u64* keys, const u32* vals, const u32* fptr, i64 nv, i64* lists,
                             i64 cap, unsigned long long* cnt) {
  const i64 a = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= nv) return;
  const u32 lo = fptr[a], hi = fptr[a + 1];
  u32 run = 0;
  for (u32 q = lo; q < hi; ++q) {
    run = (q > lo && keys[q] == keys[q - 1]) ? run + 1 : 0;
    if (run >= 2) push(lists + DM_V_FACE_OVERSHARED * cap, cnt + DM_V_FACE_OVERSHARED, cap, vals[q]);
  }
}

// Per boundary facet (ref mesh.cpp:206-243), visiting the sorted boundary
// buckets so a duplicate is any facet with an equal key and a smaller id.
template <int D>
__global__ void k_bnd_check(const u64* bkeys, const u32* bvals, const u32* bptr, const u64* fkeys,
                            const u32* fvals, const u32* fptr, const int32_t* el,
                            const int32_t* bnd, const double* x, i64 nv, i64* lists, i64 cap,
                            unsigned long long* cnt) {
  const i64 a = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= nv) return;
  const u32 lo = bptr[a], hi = bptr[a + 1];
  for (u32 q = lo; q < hi; ++q) {
    const u64 key = bkeys[q];
    const i64 b = bvals[q];
    const u32 f = find_key(fkeys, fptr[a], fptr[a + 1], key);
    if (f == fptr[a + 1]) {
      push(lists + DM_V_BND_NOT_FACE * cap, cnt + DM_V_BND_NOT_FACE, cap, b << 32);
      continue;
    }
    u32 n = 1;
    while (f + n < fptr[a + 1] && fkeys[f + n] == key) ++n;
    const i64 owner = fvals[f] / (D + 1);
    if (n != 1) {
      push(lists + DM_V_BND_INTERIOR * cap, cnt + DM_V_BND_INTERIOR, cap, (b << 32) | owner);
      continue;
    }
    if (q > lo && bkeys[q - 1] == key) {
      push(lists + DM_V_BND_DUPLICATE * cap, cnt + DM_V_BND_DUPLICATE, cap, b << 32);
      continue;
    }
    // outward check against the owner (ref mesh.cpp:225-242)
    const int32_t* bl = bnd + D * b;
    double nb[3];
    if (D == 2) {
      const double *j = x + 2 * (i64)bl[0], *k = x + 2 * (i64)bl[1];
      nb[0] = k[1] - j[1];
      nb[1] = j[0] - k[0];
      nb[2] = 0.0;
    } else {
      const double *j = x + 3 * (i64)bl[0], *r = x + 3 * (i64)bl[1], *l = x + 3 * (i64)bl[2];
      double c0, c1, c2;
      cross3(r[0] - j[0], r[1] - j[1], r[2] - j[2], l[0] - j[0], l[1] - j[1], l[2] - j[2], c0, c1,
             c2);
      nb[0] = 0.5 * c0;
      nb[1] = 0.5 * c1;
      nb[2] = 0.5 * c2;
    }
    const int32_t* t = el + (D + 1) * owner;
    int opp = -1;
    for (int i = 0; i <= D; ++i) {
      bool on = false;
      for (int s = 0; s < D; ++s) on = on || (t[i] == bl[s]);
      if (!on) opp = t[i];
    }
    const double* xo = x + (i64)D * opp;
    const double* xf = x + (i64)D * bl[0];
    double dot = 0.0;
    for (int d = 0; d < D; ++d) dot += nb[d] * (xo[d] - xf[d]);
    if (!(dot < 0.0))
      push(lists + DM_V_BND_INWARD * cap, cnt + DM_V_BND_INWARD, cap, (b << 32) | owner);
  }
}

// Single-incidence faces with no boundary facet (ref mesh.cpp:245-251).
__global__ void k_exposed(const u64* fkeys, const u32* fptr, const u64* bkeys, const u32* bptr,
                          i64 nv, unsigned long long* exposed) {
  const i64 a = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= nv) return;
  const u32 lo = fptr[a], hi = fptr[a + 1];
  unsigned long long mine = 0;
  for (u32 q = lo; q < hi; ++q) {
    if (q > lo && fkeys[q] == fkeys[q - 1]) continue;
    if (q + 1 < hi && fkeys[q + 1] == fkeys[q]) continue;
    if (find_key(bkeys, bptr[a], bptr[a + 1], fkeys[q]) == bptr[a + 1]) ++mine;
  }
  if (mine) atomicAdd(exposed, mine);
}

// Derived boundary (ref mesh.cpp:287-323): single-incidence faces in the
// owner's outward order, then sorted lexicographically.
template <int D>
__global__ void k_derive_count(const u64* fkeys, const u32* fvals, const u32* fptr,
                               const int32_t* el, i64 nv, u32* cnt) {
  const i64 a = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= nv) return;
  const u32 lo = fptr[a], hi = fptr[a + 1];
  for (u32 q = lo; q < hi; ++q) {
    if ((q > lo && fkeys[q] == fkeys[q - 1]) || (q + 1 < hi && fkeys[q + 1] == fkeys[q])) continue;
    int o[3];
    face_nodes<D>(el, fvals[q] / (D + 1), static_cast<int>(fvals[q] % (D + 1)), o);
    atomicAdd(cnt + o[0], 1u);
  }
}

template <int D>
__global__ void k_derive_scatter(const u64* fkeys, const u32* fvals, const u32* fptr,
                                 const int32_t* el, i64 nv, const u32* start, u32* fill,
                                 u64* out) {
  const i64 a = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= nv) return;
  const u32 lo = fptr[a], hi = fptr[a + 1];
  for (u32 q = lo; q < hi; ++q) {
    if ((q > lo && fkeys[q] == fkeys[q - 1]) || (q + 1 < hi && fkeys[q + 1] == fkeys[q])) continue;
    int o[3];
    face_nodes<D>(el, fvals[q] / (D + 1), static_cast<int>(fvals[q] % (D + 1)), o);
    const u32 p = start[o[0]] + atomicAdd(fill + o[0], 1u);
    out[p] = (static_cast<u64>(static_cast<u32>(o[1])) << 32) | static_cast<u32>(o[2]);
  }
}

template <int D>
__global__ void k_derive_emit(const u64* keys, const u32* start, i64 nv, int32_t* out) {
  const i64 a = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= nv) return;
  for (u32 q = start[a]; q < start[a + 1]; ++q) {
    out[D * static_cast<i64>(q)] = static_cast<int32_t>(a);
    out[D * static_cast<i64>(q) + 1] = static_cast<int32_t>(keys[q] >> 32);
    if (D == 3) out[D * static_cast<i64>(q) + 2] = static_cast<int32_t>(keys[q] & 0xffffffffu);
  }
}

// Bucket-sort the element faces (and optionally the boundary facets).
template <int D>
int build_faces(dm_ctx* c, Faces& F, bool with_boundary) {
  const i64 nv = c->nv, nF = c->nE * (D + 1);
  DM_CK(c, F.fptr.ensure(nv + 1));
  DM_CK(c, F.fkey.ensure(nF));
  DM_CK(c, F.fval.ensure(nF));
  DM_CK(c, c->fill.ensure(nv + 1));
  DM_CK(c, cudaMemsetAsync(F.fptr.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_CK(c, cudaMemsetAsync(c->fill.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_LAUNCH(c, k_face_count<D>, grid_for(nF, 256), 256, 0, c->elems.p, c->nE, F.fptr.p);
  int st = scan_exclusive(c, F.fptr.p, F.fptr.p, nv);
  if (st) return st;
  DM_LAUNCH(c, k_face_scatter<D>, grid_for(nF, 256), 256, 0, c->elems.p, c->nE, F.fptr.p,
            c->fill.p, F.fkey.p, F.fval.p);
  st = segment_sort_kv(c, F.fkey.p, F.fval.p, F.fptr.p, nv);
  if (st) return st;
  if (!with_boundary) return DM_OK;
  const i64 nB = c->nB;
  DM_CK(c, F.bptr.ensure(nv + 1));
  DM_CK(c, F.bkey.ensure(nB));
  DM_CK(c, F.bval.ensure(nB));
  DM_CK(c, cudaMemsetAsync(F.bptr.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_CK(c, cudaMemsetAsync(c->fill.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_LAUNCH(c, k_bnd_count<D>, grid_for(nB, 256), 256, 0, c->bnd.p, nB, F.bptr.p);
  st = scan_exclusive(c, F.bptr.p, F.bptr.p, nv);
  if (st) return st;
  DM_LAUNCH(c, k_bnd_scatter<D>, grid_for(nB, 256), 256, 0, c->bnd.p, nB, F.bptr.p, c->fill.p,
            F.bkey.p, F.bval.p);
  return segment_sort_kv(c, F.bkey.p, F.bval.p, F.bptr.p, nv);
}

template <int D>
int validate_impl(dm_ctx* c, int8_t* signs, int64_t* counts, int64_t* exposed) {
  const i64 nv = c->nv, nE = c->nE, nB = c->nB;
  const i64 cap = std::max<i64>(std::max<i64>(nE * (D + 1), nB), 1);
  DM_CK(c, c->vlist.ensure(static_cast<size_t>(cap * DM_VCOUNT)));
  DevBuf<unsigned long long> cnt;
  DM_CK(c, cnt.ensure(DM_VCOUNT + 1));
  DM_CK(c, cudaMemsetAsync(cnt.p, 0, (DM_VCOUNT + 1) * sizeof(unsigned long long), c->stream));
  c->vlist_cap = cap;
  DM_LAUNCH(c, k_range<D>, grid_for(nE + nB, 256), 256, 0, c->elems.p, nE, c->bnd.p, nB, nv,
            c->vlist.p, cap, cnt.p);
  unsigned long long h[DM_VCOUNT + 1];
  DM_CK(c, cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  if (h[DM_V_OUT_OF_RANGE_ELEM] + h[DM_V_OUT_OF_RANGE_BND] == 0) {
    DevBuf<int8_t> dsig;
    DM_CK(c, dsig.ensure(std::max<i64>(nE, 1)));
    DM_LAUNCH(c, k_signs<D>, grid_for(nE, 256), 256, 0, c->elems.p, c->coords.p, nE, dsig.p,
              c->vlist.p, cap, cnt.p);
    Faces F;
    int st = build_faces<D>(c, F, true);
    if (st) return st;
    DM_LAUNCH(c, k_overshared<D>, grid_for(nv, 256), 256, 0, F.fkey.p, F.fval.p, F.fptr.p, nv,
              c->vlist.p, cap, cnt.p);
    DM_LAUNCH(c, k_bnd_check<D>, grid_for(nv, 256), 256, 0, F.bkey.p, F.bval.p, F.bptr.p,
              F.fkey.p, F.fval.p, F.fptr.p, c->elems.p, c->bnd.p, c->coords.p, nv, c->vlist.p, cap,
              cnt.p);
    DM_LAUNCH(c, k_exposed, grid_for(nv, 256), 256, 0, F.fkey.p, F.fptr.p, F.bkey.p, F.bptr.p, nv,
              cnt.p + DM_VCOUNT);
    if (signs && nE)
      DM_CK(c, cudaMemcpyAsync(signs, dsig.p, nE, cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaMemcpyAsync(h, cnt.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    DM_CK(c, cudaStreamSynchronize(c->stream));
  }
  for (int k = 0; k < DM_VCOUNT; ++k) {
    c->vlist_n[k] = static_cast<i64>(h[k]);
    if (counts) counts[k] = static_cast<int64_t>(h[k]);
  }
  if (exposed) *exposed = static_cast<int64_t>(h[DM_VCOUNT]);
  return DM_OK;
}

template <int D>
int derive_impl(dm_ctx* c) {
  Faces F;
  int st = build_faces<D>(c, F, false);
  if (st) return st;
  const i64 nv = c->nv;
  DevBuf<u32> ptr;
  DM_CK(c, ptr.ensure(nv + 1));
  DM_CK(c, cudaMemsetAsync(ptr.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_CK(c, cudaMemsetAsync(c->fill.p, 0, (nv + 1) * sizeof(u32), c->stream));
  DM_LAUNCH(c, k_derive_count<D>, grid_for(nv, 256), 256, 0, F.fkey.p, F.fval.p, F.fptr.p,
            c->elems.p, nv, ptr.p);
  st = scan_exclusive(c, ptr.p, ptr.p, nv);
  if (st) return st;
  u32 n = 0;
  DM_CK(c, cudaMemcpyAsync(&n, ptr.p + nv, sizeof(u32), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  DevBuf<u64> keys;
  DM_CK(c, keys.ensure(std::max<u32>(n, 1)));
  DM_LAUNCH(c, k_derive_scatter<D>, grid_for(nv, 256), 256, 0, F.fkey.p, F.fval.p, F.fptr.p,
            c->elems.p, nv, ptr.p, c->fill.p, keys.p);
  st = segment_sort_u64(c, keys.p, ptr.p, nv);
  if (st) return st;
  DM_CK(c, c->derived.ensure(std::max<i64>(static_cast<i64>(n) * D, 1)));
  DM_LAUNCH(c, k_derive_emit<D>, grid_for(nv, 256), 256, 0, keys.p, ptr.p, nv, c->derived.p);
  DM_CK(c, cudaStreamSynchronize(c->stream));
  c->n_derived = n;
  return DM_OK;
}

}  // namespace
}  // namespace dm

using namespace dm;

extern "C" int dm_validate(dm_ctx* c, int8_t* volume_signs, int64_t counts[DM_VCOUNT],
                           int64_t* exposed_faces) {
  if (!c) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "no mesh");
  if (c->nv >= (1ll << 31) || c->nE * (c->dim + 1) >= (1ll << 32))
    return fail(c, DM_ERR_UNSUPPORTED, "mesh too large for 32-bit face ids");
  return c->dim == 3 ? validate_impl<3>(c, volume_signs, counts, exposed_faces)
                     : validate_impl<2>(c, volume_signs, counts, exposed_faces);
}

extern "C" int dm_validate_list(dm_ctx* c, int kind, int64_t* ids, int64_t cap, int64_t* n) {
  if (!c || kind < 0 || kind >= DM_VCOUNT || (cap > 0 && !ids)) return DM_ERR_INVALID_ARG;
  const i64 have = std::min(c->vlist_n[kind], c->vlist_cap);
  const i64 take = std::min<i64>(have, cap);
  std::vector<i64> v(static_cast<size_t>(have));
  if (have)
    DM_CK(c, cudaMemcpy(v.data(), c->vlist.p + kind * c->vlist_cap, have * sizeof(i64),
                        cudaMemcpyDeviceToHost));
  std::sort(v.begin(), v.end());  // the reference reports in ascending id order
  for (i64 i = 0; i < take; ++i) ids[i] = v[static_cast<size_t>(i)];
  if (n) *n = take;
  return DM_OK;
}

extern "C" int dm_derive_boundary(dm_ctx* c, int64_t* n_faces) {
  if (!c) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "no mesh");
  int st = c->dim == 3 ? derive_impl<3>(c) : derive_impl<2>(c);
  if (st) return st;
  if (n_faces) *n_faces = c->n_derived;
  return DM_OK;
}

extern "C" int dm_get_derived_boundary(dm_ctx* c, int32_t* faces) {
  if (!c || !faces) return DM_ERR_INVALID_ARG;
  if (c->n_derived)
    DM_CK(c, cudaMemcpy(faces, c->derived.p, c->n_derived * c->dim * sizeof(int32_t),
                        cudaMemcpyDeviceToHost));
  return DM_OK;
}
