// navs.cu -- lumped directed-area vectors (navs) on the GPU.
//
//   K2  element loop     : dual-free or traditional
//                           contributions
//   K3  boundary pass    : n_jk += n_B / (D(D+1))
//   s   edge dot product : s_e = (x_k - x_j) . n_jk, the per-edge term of the
//                          edge-based dual volumes, fused here
//                          so K4 never re-reads navs.
//
// Variants (north_star (b)):
//   GATHER  (default): one CTA per 256 consecutive edges.  The CTA's slice of
//           the edge->element CSR (inc) is contiguous; its incidences are
//           evaluated in parallel into shared memory, then every edge thread
//           folds its own incidences in ascending element id, scales, adds
//           its boundary terms in ascending facet id and writes navs and s
//           once.  This is the serial oracle's summation order, so the result
//           is bitwise identical to it.  No atomics, no memset.
//   SCATTER: one thread per element, fp64 atomics (REDG.E.ADD.F64) through
//           e2l into zeroed navs, then the same per-edge tail.  Faster or
//           not, its summation order varies run to run (<=1e-12 parity).
#include "geometry.cuh"

namespace dm {
namespace {

constexpr int kEB = 256;    // edges per CTA (one per thread)
constexpr int kCH = 1536;   // incidences staged per shared-memory chunk

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

// Per-edge tail shared by both variants: scale pass, boundary pass, write
// navs and s.  acc holds the element-loop sum for edge e (in ascending
// element order for GATHER).  [rb, re) is the CTA's slice of the sorted
// boundary (edge, facet) list.
template <int D, int ALGO>
__device__ __forceinline__ void edge_tail(const Coords<D>& X, i64 e, int j, int k, double* acc,
                                          const u64* __restrict__ bedge, u32 rb, u32 re,
                                          const int32_t* __restrict__ bnd,
                                          double* __restrict__ navs, double* __restrict__ svals) {
  double n[3] = {acc[0], acc[1], D == 3 ? acc[2] : 0.0};
  if constexpr (D == 3) {
    const double f = ALGO == kDualFree ? (1.0 / 12.0) : 0.5;  // SPEC.md:162 / PAPER.md:170
    n[0] *= f;
    n[1] *= f;
    n[2] *= f;
  }
  if constexpr (ALGO == kDualFree) {
    if (rb < re) {
      // lower bound of edge e in the slice
      u32 lo = rb, hi = re;
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
  double s;
  if constexpr (D == 3) {
    const d4 xj = X[j], xk = X[k];
    s = (xk.x - xj.x) * n[0] + (xk.y - xj.y) * n[1];
    s = s + (xk.z - xj.z) * n[2];
    navs[3 * e] = n[0];
    navs[3 * e + 1] = n[1];
    navs[3 * e + 2] = n[2];
  } else {
    const double2 xj = X[j], xk = X[k];
    s = (xk.x - xj.x) * n[0] + (xk.y - xj.y) * n[1];
    navs[2 * e] = n[0];
    navs[2 * e + 1] = n[1];
  }
  svals[e] = s;
}

__device__ __forceinline__ u32 lower_bound_edge(const u64* bedge, u32 n, i64 e) {
  u32 lo = 0, hi = n;
  while (lo < hi) {
    const u32 mid = (lo + hi) >> 1;
    if ((bedge[mid] >> 32) < static_cast<u64>(e)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <int D, int ALGO>
__global__ void __launch_bounds__(kEB)
    k_navs_gather(const int2* __restrict__ edges, const int32_t* __restrict__ inc_ptr,
                  const int32_t* __restrict__ inc, const int32_t* __restrict__ el, Coords<D> X,
                  i64 ne, const u64* __restrict__ bedge, u32 n_bedge,
                  const int32_t* __restrict__ bnd, double* __restrict__ navs,
                  double* __restrict__ svals) {
  __shared__ int s_j[kEB], s_k[kEB];
  __shared__ unsigned char s_le[kCH];
  __shared__ double s_c[kCH * D];
  __shared__ u32 s_br[2];

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
  if (ALGO == kDualFree && t == 0) {
    s_br[0] = lower_bound_edge(bedge, n_bedge, e0);
    s_br[1] = lower_bound_edge(bedge, n_bedge, e1);
  }
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
      for (int d = 0; d < D; ++d) s_c[(q - c0) * D + d] = c[d];
    }
    __syncthreads();
    for (int q = qb; q < qe; ++q) {
#pragma unroll
      for (int d = 0; d < D; ++d) acc[d] += s_c[(q - c0) * D + d];
    }
    __syncthreads();
  }
  if (!valid) return;
  edge_tail<D, ALGO>(X, e, j, k, acc, bedge, ALGO == kDualFree ? s_br[0] : 0u,
                     ALGO == kDualFree ? s_br[1] : 0u, bnd, navs, svals);
}

// -------------------------------------------------------------- SCATTER
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

template <int D, int ALGO>
__global__ void __launch_bounds__(256)
    k_edge_finalize(const int2* __restrict__ edges, Coords<D> X, i64 ne,
                    const u64* __restrict__ bedge, u32 n_bedge, const int32_t* __restrict__ bnd,
                    double* __restrict__ navs, double* __restrict__ svals) {
  __shared__ u32 s_br[2];
  const i64 e0 = static_cast<i64>(blockIdx.x) * blockDim.x;
  const i64 e1 = (e0 + blockDim.x < ne) ? e0 + blockDim.x : ne;
  if (ALGO == kDualFree && threadIdx.x == 0) {
    s_br[0] = lower_bound_edge(bedge, n_bedge, e0);
    s_br[1] = lower_bound_edge(bedge, n_bedge, e1);
  }
  __syncthreads();
  const i64 e = e0 + threadIdx.x;
  if (e >= ne) return;
  const int2 jk = edges[e];
  double acc[3] = {navs[D * e], navs[D * e + 1], D == 3 ? navs[D * e + 2] : 0.0};
  edge_tail<D, ALGO>(X, e, jk.x, jk.y, acc, bedge, ALGO == kDualFree ? s_br[0] : 0u,
                     ALGO == kDualFree ? s_br[1] : 0u, bnd, navs, svals);
}

template <int D, int ALGO>
int launch_navs(dm_ctx* c, int variant) {
  Coords<D> X;
  if constexpr (D == 3) X.p = c->x4.p;
  else X.p = reinterpret_cast<const double2*>(c->coords.p);
  const u32 nb = static_cast<u32>(c->n_bedge);
  const i64 ne = c->ne;
  if (variant == DM_VARIANT_SCATTER) {
    tmark(c, 0);
    DM_CK(c, cudaMemsetAsync(c->navs.p, 0, sizeof(double) * D * ne, c->stream));
    DM_LAUNCH(c, (k_navs_scatter<D, ALGO>), grid_for(c->nE, 256), 256, 0, c->elems.p, X, c->nE,
              c->e2l.p, c->navs.p);
    tmark(c, 1);
    DM_LAUNCH(c, (k_edge_finalize<D, ALGO>), grid_for(ne, 256), 256, 0, c->edges.p, X, ne,
              c->bedge.p, nb, c->bnd.p, c->navs.p, c->svals.p);
    tmark(c, 2);
  } else {
    tmark(c, 0);
    DM_LAUNCH(c, (k_navs_gather<D, ALGO>), grid_for(ne, kEB), kEB, 0, c->edges.p, c->inc_ptr.p,
              c->inc.p, c->elems.p, X, ne, c->bedge.p, nb, c->bnd.p, c->navs.p, c->svals.p);
    tmark(c, 1);
    tmark(c, 2);
  }
  return DM_OK;
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

}  // namespace

int svals_from_navs(dm_ctx* c) {
  if (c->dim == 3) {
    Coords<3> X{c->x4.p};
    DM_LAUNCH(c, k_svals<3>, grid_for(c->ne, 256), 256, 0, c->edges.p, X, c->ne, c->navs.p,
              c->svals.p);
  } else {
    Coords<2> X{reinterpret_cast<const double2*>(c->coords.p)};
    DM_LAUNCH(c, k_svals<2>, grid_for(c->ne, 256), 256, 0, c->edges.p, X, c->ne, c->navs.p,
              c->svals.p);
  }
  return DM_OK;
}

int navs_impl(dm_ctx* c, int algo, int variant) {
  if (!c->have_edges) return fail(c, DM_ERR_STATE, "navs requested before build_edges");
  if (algo != DM_NAV_TRADITIONAL && algo != DM_NAV_DUALFREE)
    return fail(c, DM_ERR_INVALID_ARG, "unknown nav algorithm");
  if (variant != DM_VARIANT_GATHER && variant != DM_VARIANT_SCATTER)
    return fail(c, DM_ERR_INVALID_ARG, "unknown nav variant");
  int st = ensure_bedge(c);
  if (st) return st;
  DM_CK(c, c->navs.ensure(static_cast<size_t>(c->dim * c->ne)));
  DM_CK(c, c->svals.ensure(static_cast<size_t>(c->ne)));
  if (c->dim == 3) {
    st = algo == DM_NAV_DUALFREE ? launch_navs<3, kDualFree>(c, variant)
                                 : launch_navs<3, kTraditional>(c, variant);
  } else {
    st = algo == DM_NAV_DUALFREE ? launch_navs<2, kDualFree>(c, variant)
                                 : launch_navs<2, kTraditional>(c, variant);
  }
  if (st) return st;
  c->have_navs = true;
  c->navs_algo = algo;
  c->have_vols = false;
  return DM_OK;
}

}  // namespace dm
