// volumes.cu -- median-dual volumes on the GPU.
//
//   K4 edge-based: V_j = (1/(2D)) sum of
//      s_e over the edges touching j, with s_e = (x_k - x_j).n_jk produced by
//      the nav kernel.  One thread per node folds its incoming edges (the
//      transposed CSR, ascending edge id) and then its outgoing row
//      (origin_start), which is the order in which the serial edge loop of
//      the oracle updates V_j -- bitwise identical, no atomics.
//   K6 element-based: V_E per element
//      (coalesced pass), then one thread per node folds V_E over its
//      incident elements in ascending id and scales by 1/(D+1).
#include "geometry.cuh"

namespace dm {
namespace {

// acc += s[idx(q)] for q in [b, e), in order; the loads of each batch of
// kB terms are issued before any add (memory-level parallelism on a
// latency-bound gather; the fold order is unchanged).
constexpr int kB = 6;
template <typename Idx>
__device__ __forceinline__ double fold_terms(double acc, u32 b, u32 e, const Idx& idx,
                                             const double* __restrict__ s) {
  for (u32 q0 = b; q0 < e; q0 += kB) {
    double v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) v[u] = q0 + u < e ? s[idx(q0 + u)] : 0.0;
#pragma unroll
    for (int u = 0; u < kB; ++u)
      if (q0 + u < e) acc += v[u];
  }
  return acc;
}

// One node's fold: incoming terms (ascending edge id, through `in_idx`), then
// the outgoing row -- with the first eight terms of BOTH lists loaded before
// any add (most nodes have <= 8 + 8), so the two lists' gathers overlap
// instead of running back to back (C5 0.345 -> 0.317 ms; same order, same
// bits; in_list loads without L1 allocation measured slower).
template <typename InIdx>
__device__ __forceinline__ double fold_node(u32 ib, u32 ie, u32 ob, u32 oe, const InIdx& in_idx,
                                            const double* __restrict__ s) {
  double vi[8], vo[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    vi[u] = ib + u < ie ? s[in_idx(ib + u)] : 0.0;
    vo[u] = ob + u < oe ? s[ob + u] : 0.0;
  }
  double acc = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (ib + u < ie) acc += vi[u];
  if (ie > ib + 8) acc = fold_terms(acc, ib + 8, ie, in_idx, s);
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (ob + u < oe) acc += vo[u];
  if (oe > ob + 8) acc = fold_terms(acc, ob + 8, oe, [](u32 q) { return q; }, s);
  return acc;
}

template <int D>
__global__ void __launch_bounds__(256, 8)
    k_vol_edge(const u32* __restrict__ in_ptr, const int32_t* __restrict__ in_list,
               const u32* __restrict__ os, const double* __restrict__ svals, i64 nv,
               double* __restrict__ V) {
  const i64 v = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const double acc = fold_node(in_ptr[v], in_ptr[v + 1], os[v], os[v + 1],
                               [&](u32 q) { return __ldg(in_list + q); }, svals);
  V[v] = acc * (1.0 / static_cast<double>(2 * D));
}

// Same fold with the ring path's position-ordered s: one thread per Morton
// rank r (node morder[r]), incoming positions rin_list, outgoing positions
// [rpstart[r], rpstart[r+1]) -- each node's terms in the same order as above.
__global__ void __launch_bounds__(256)
    k_vol_edge_pos(const int32_t* __restrict__ morder, const u32* __restrict__ rin_ptr,
                   const int32_t* __restrict__ rin_list, const u32* __restrict__ rpstart,
                   const double* __restrict__ svals, i64 nv, double* __restrict__ V) {
  const i64 r = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nv) return;
  const double acc = fold_node(rin_ptr[r], rin_ptr[r + 1], rpstart[r], rpstart[r + 1],
                               [&](u32 q) { return __ldg(rin_list + q); }, svals);
  V[morder[r]] = acc * (1.0 / 6.0);
}

template <int D, typename CX>
__global__ void __launch_bounds__(256)
    k_elem_vol(const int32_t* __restrict__ el, CX X, i64 nE, double* __restrict__ ve) {
  const i64 E = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (E >= nE) return;
  if constexpr (D == 3) {
    const int4 t = ld_i4(reinterpret_cast<const int4*>(el) + E);
    ve[E] = evol3(X, t.x, t.y, t.z, t.w);
  } else {
    ve[E] = evol2(X, __ldg(el + 3 * E), __ldg(el + 3 * E + 1), __ldg(el + 3 * E + 2));
  }
}

template <int D>
__global__ void __launch_bounds__(256, 8)
    k_vol_elem(const u32* __restrict__ ptr, const int32_t* __restrict__ n2e,
               const double* __restrict__ ve, i64 nv, double* __restrict__ V) {
  const i64 v = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  const double acc =
      fold_terms(0.0, ptr[v], ptr[v + 1], [&](u32 q) { return __ldg(n2e + q); }, ve);
  V[v] = acc * (1.0 / static_cast<double>(D + 1));
}

}  // namespace

int compute_element_volumes(dm_ctx* c) {
  DM_CK(c, c->velem.ensure(static_cast<size_t>(c->nE)));
  if (c->dim == 3) {  // raw coordinates: no copy carried between calls
    Coords3R X{c->coords.p};
    DM_LAUNCH(c, (k_elem_vol<3, Coords3R>), grid_for(c->nE, 256), 256, 0, c->elems.p, X, c->nE,
              c->velem.p);
  } else {
    Coords<2> X{reinterpret_cast<const double2*>(c->coords.p)};
    DM_LAUNCH(c, (k_elem_vol<2, Coords<2>>), grid_for(c->nE, 256), 256, 0, c->elems.p, X, c->nE,
              c->velem.p);
  }
  return DM_OK;
}

int volumes_impl(dm_ctx* c, int algo) {
  const i64 nv = c->nv;
  DM_CK(c, c->vols.ensure(static_cast<size_t>(nv)));
  if (algo != DM_VOL_EDGE && algo != DM_VOL_ELEMENT)
    return fail(c, DM_ERR_INVALID_ARG, "unknown volume algorithm");
  if (algo == DM_VOL_EDGE && !c->have_navs)
    return fail(c, DM_ERR_STATE, "edge-based volumes need navs first");
  if (c->nE == 0) {  // no elements: every dual volume is an empty sum
    if (nv > 0) DM_CK(c, cudaMemsetAsync(c->vols.p, 0, nv * sizeof(double), c->stream));
    c->have_vols = true;
    return DM_OK;
  }
  if (algo == DM_VOL_EDGE) {
    if (!c->have_navs) return fail(c, DM_ERR_STATE, "edge-based volumes need navs first");
    int st = ensure_incoming(c);
    if (st) return st;
    tmark(c, 2);
    if (c->svals_pos) {
      DM_LAUNCH(c, k_vol_edge_pos, grid_for(nv, 256), 256, 0, c->morder.p, c->rin_ptr.p,
                c->rin_list.p, c->rpstart.p, c->svals.p, nv, c->vols.p);
    } else if (c->dim == 3) {
      DM_LAUNCH(c, k_vol_edge<3>, grid_for(nv, 256), 256, 0, c->in_ptr.p, c->in_list.p, c->os.p,
                c->svals.p, nv, c->vols.p);
    } else {
      DM_LAUNCH(c, k_vol_edge<2>, grid_for(nv, 256), 256, 0, c->in_ptr.p, c->in_list.p, c->os.p,
                c->svals.p, nv, c->vols.p);
    }
    tmark(c, 3);
  } else if (algo == DM_VOL_ELEMENT) {
    int st = ensure_n2e(c);
    if (st) return st;
    tmark(c, 2);
    st = compute_element_volumes(c);
    if (st) return st;
    if (c->dim == 3) {
      DM_LAUNCH(c, k_vol_elem<3>, grid_for(nv, 256), 256, 0, c->n2e_ptr.p, c->n2e.p, c->velem.p,
                nv, c->vols.p);
    } else {
      DM_LAUNCH(c, k_vol_elem<2>, grid_for(nv, 256), 256, 0, c->n2e_ptr.p, c->n2e.p, c->velem.p,
                nv, c->vols.p);
    }
    tmark(c, 3);
  } else {
    return fail(c, DM_ERR_INVALID_ARG, "unknown volume algorithm");
  }
  c->have_vols = true;
  return DM_OK;
}

}  // namespace dm
