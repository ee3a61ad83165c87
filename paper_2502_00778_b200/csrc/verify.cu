// verify.cu -- SPEC verify checks and mesh-wide reductions on the GPU.
//
//   closure      SPEC.md:245-253 / PAPER.md:399-424
//   total volume SPEC.md:255-263 / PAPER.md:§4.3, double-double block sums
//   linear exactness SPEC.md:265-274 (affine flux, average edge flux)
//   max_face_area, max_element_volume, total_volume, boundary_node_mask
//                ref mesh.cpp:325-349
#include <cmath>
#include <cstring>

#include <cudaTypedefs.h>

#include "geometry.cuh"

namespace dm {
namespace {

__device__ __forceinline__ void atomic_max_nonneg(u64* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

__global__ void k_pad3(const double* __restrict__ c, i64 nv, d4* __restrict__ x4) {
  const i64 v = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  d4 r;
  r.x = c[3 * v];
  r.y = c[3 * v + 1];
  r.z = c[3 * v + 2];
  r.w = 0.0;
  x4[v] = r;
}

__global__ void k_bmask(const int32_t* __restrict__ bnd, i64 n, uint8_t* __restrict__ mask) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) mask[bnd[i]] = 1;
}

// a_v = sum_out n - sum_in n; interior max before the boundary closure.
template <int D>
__global__ void k_closure_nodes(const u32* __restrict__ in_ptr, const int32_t* __restrict__ in_list,
                                const u32* __restrict__ os, const double* __restrict__ navs,
                                const uint8_t* __restrict__ bmask, i64 nv, double* __restrict__ a,
                                u64* __restrict__ mx) {
  const i64 v = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  double s[3] = {0.0, 0.0, 0.0};
  for (u32 q = os[v]; q < os[v + 1]; ++q)
    for (int d = 0; d < D; ++d) s[d] += navs[D * static_cast<i64>(q) + d];
  for (u32 q = in_ptr[v]; q < in_ptr[v + 1]; ++q) {
    const i64 e = in_list[q];
    for (int d = 0; d < D; ++d) s[d] -= navs[D * e + d];
  }
  for (int d = 0; d < D; ++d) a[D * v + d] = s[d];
  if (!bmask[v]) {
    double r = 0.0;
    for (int d = 0; d < D; ++d) r += s[d] * s[d];
    atomic_max_nonneg(mx + 1, sqrt(r));
  }
}

template <int D>
__global__ void k_closure_bnd(const int32_t* __restrict__ bnd, Coords<D> X, i64 nB,
                              double* __restrict__ a) {
  const i64 b = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nB) return;
  double n[3];
  if constexpr (D == 3) bnormal3(X, bnd + 3 * b, n[0], n[1], n[2]);
  else bnormal2(X, bnd + 2 * b, n[0], n[1]);
  const double f = 1.0 / static_cast<double>(D);
  for (int t = 0; t < D; ++t) {
    const i64 v = bnd[D * b + t];
    for (int d = 0; d < D; ++d) atomicAdd(a + D * v + d, f * n[d]);
  }
}

// ---- linear exactness
struct Affine {
  double A[9], b[3], tr;
  int zero;
};

// phi_e = ((F_j + F_k) * 0.5) . n_e with F(x) = A x + b, in the oracle's
// operation order; max |phi| into mx.
template <int D>
__global__ void k_lin_phi(const int2* __restrict__ edges, Coords<D> X,
                          const double* __restrict__ navs, i64 ne, Affine F,
                          double* __restrict__ phi, u64* __restrict__ mx) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  double ap = 0.0;
  if (e < ne) {
    const int2 jk = edges[e];
    double xj[3], xk[3];
    if constexpr (D == 3) {
      const d4 a = X[jk.x], c = X[jk.y];
      xj[0] = a.x; xj[1] = a.y; xj[2] = a.z;
      xk[0] = c.x; xk[1] = c.y; xk[2] = c.z;
    } else {
      const double2 a = X[jk.x], c = X[jk.y];
      xj[0] = a.x; xj[1] = a.y; xj[2] = 0.0;
      xk[0] = c.x; xk[1] = c.y; xk[2] = 0.0;
    }
    double p = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) {
      double fj = F.b[r], fk = F.b[r];
#pragma unroll
      for (int c = 0; c < D; ++c) {
        fj += F.A[r * D + c] * xj[c];
        fk += F.A[r * D + c] * xk[c];
      }
      p += ((fj + fk) * 0.5) * navs[D * e + r];
    }
    phi[e] = p;
    ap = fabs(p);
  }
  for (int o = 16; o > 0; o >>= 1) ap = fmax(ap, __shfl_xor_sync(0xffffffffu, ap, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(mx, ap);
}

// Res_v = -sum_in phi + sum_out phi (the serial edge loop's order per node);
// affine flux: max over interior nodes of |Res/V - tr| / |tr| into mx[1];
// constant flux: Res kept for the boundary closure.
__global__ void k_lin_nodes(const u32* __restrict__ in_ptr, const int32_t* __restrict__ in_list,
                            const u32* __restrict__ os, const double* __restrict__ phi,
                            const double* __restrict__ V, const uint8_t* __restrict__ bmask,
                            i64 nv, Affine F, double* __restrict__ res, u64* __restrict__ mx) {
  const i64 v = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  double r = 0.0;
  if (v < nv) {
    double acc = 0.0;
    for (u32 q = in_ptr[v]; q < in_ptr[v + 1]; ++q) acc -= phi[in_list[q]];
    for (u32 q = os[v]; q < os[v + 1]; ++q) acc += phi[q];
    if (F.zero) res[v] = acc;
    else if (!bmask[v]) r = fabs(acc / V[v] - F.tr) / fabs(F.tr);
  }
  for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(mx + 1, r);
}

template <int D>
__global__ void k_lin_bnd(const int32_t* __restrict__ bnd, Coords<D> X, i64 nB, Affine F,
                          double* __restrict__ res) {
  const i64 q = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nB) return;
  double n[3] = {0.0, 0.0, 0.0};
  if constexpr (D == 3) bnormal3(X, bnd + 3 * q, n[0], n[1], n[2]);
  else bnormal2(X, bnd + 2 * q, n[0], n[1]);
  double bn = 0.0;
  for (int d = 0; d < D; ++d) bn += F.b[d] * n[d];
  const double f = 1.0 / static_cast<double>(D);
  for (int t = 0; t < D; ++t) atomicAdd(res + bnd[D * q + t], f * bn);
}

__global__ void k_abs_max(const double* __restrict__ x, i64 n, u64* __restrict__ mx) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  double r = i < n ? fabs(x[i]) : 0.0;
  for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(mx, r);
}

template <int D>
__global__ void k_norm_max(const double* __restrict__ x, i64 n, u64* __restrict__ mx) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  double r = 0.0;
  if (i < n) {
    for (int d = 0; d < D; ++d) r += x[D * i + d] * x[D * i + d];
    r = sqrt(r);
  }
  // warp max then one atomic
  for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(mx, r);
}

// Double-double (TwoSum) accumulation: deterministic for a fixed grid.
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ void dd_add(double& hi, double& lo, double v) {
  double s, e;
  two_sum(hi, v, s, e);
  hi = s;
  lo += e;
}
__device__ __forceinline__ void dd_merge(double& hi, double& lo, double ohi, double olo) {
  double s, e;
  two_sum(hi, ohi, s, e);
  hi = s;
  lo = lo + olo + e;
}

constexpr int kSumBlocks = 592;

__global__ void __launch_bounds__(256) k_dd_sum(const double* __restrict__ x, i64 n,
                                                double2* __restrict__ part) {
  __shared__ double sh[256], sl[256];
  double hi = 0.0, lo = 0.0;
  for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    dd_add(hi, lo, x[i]);
  sh[threadIdx.x] = hi;
  sl[threadIdx.x] = lo;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      double h = sh[threadIdx.x], l = sl[threadIdx.x];
      dd_merge(h, l, sh[threadIdx.x + s], sl[threadIdx.x + s]);
      sh[threadIdx.x] = h;
      sl[threadIdx.x] = l;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = make_double2(sh[0], sl[0]);
}

template <int D>
__global__ void k_face_max(const int32_t* __restrict__ el, Coords<D> X, i64 nE, u64* mx) {
  const i64 E = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  double m = 0.0, mv = 0.0;
  if (E < nE) {
    if constexpr (D == 3) {
      const int4 t = ld_i4(reinterpret_cast<const int4*>(el) + E);
      for (int i = 0; i < 4; ++i) {
        double c0, c1, c2;
        df3(X, t.x, t.y, t.z, t.w, i, c0, c1, c2);
        c0 *= 0.5;
        c1 *= 0.5;
        c2 *= 0.5;  // opposite_face_normal = 0.5 * cross (ref mesh.cpp:110)
        m = fmax(m, sqrt(c0 * c0 + c1 * c1 + c2 * c2));
      }
      mv = fabs(evol3(X, t.x, t.y, t.z, t.w));
    } else {
      const int v[3] = {__ldg(el + 3 * E), __ldg(el + 3 * E + 1), __ldg(el + 3 * E + 2)};
      for (int i = 0; i < 3; ++i) {
        const double2 p = X[v[(i + 1) % 3]], q = X[v[(i + 2) % 3]];
        const double n0 = q.y - p.y, n1 = p.x - q.x;
        m = fmax(m, sqrt(n0 * n0 + n1 * n1 + 0.0 * 0.0));
      }
      mv = fabs(evol2(X, v[0], v[1], v[2]));
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    mv = fmax(mv, __shfl_xor_sync(0xffffffffu, mv, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_max_nonneg(mx, m);
    atomic_max_nonneg(mx + 1, mv);
  }
}

__global__ void k_corrupt(double* navs, i64 e, int D, double delta) {
  for (int d = 0; d < D; ++d) navs[D * e + d] += delta;
}

// Neumaier on the host over the block partials.
double finish_sum(const double2* part, int n) {
  double s = 0.0, cc = 0.0;
  auto add = [&](double v) {
    const double t = s + v;
    if (std::fabs(s) >= std::fabs(v)) cc += (s - t) + v;
    else cc += (v - t) + s;
    s = t;
  };
  for (int i = 0; i < n; ++i) {
    add(part[i].x);
    add(part[i].y);
  }
  return s + cc;
}

int device_sum(dm_ctx* c, const double* x, i64 n, double* out) {
  DevBuf<double2> part;
  DM_CK(c, part.ensure(kSumBlocks));
  DM_LAUNCH(c, k_dd_sum, kSumBlocks, 256, 0, x, n, part.p);
  double2 h[kSumBlocks];
  DM_CK(c, cudaMemcpyAsync(h, part.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  *out = finish_sum(h, kSumBlocks);
  return DM_OK;
}

}  // namespace

int coords_changed(dm_ctx* c) {
  c->x4_fresh = false;
  return DM_OK;
}
int pad_x4(dm_ctx* c) {
  if (c->dim != 3) return DM_OK;
  DM_CK(c, c->x4.ensure(static_cast<size_t>(c->nv)));
  DM_LAUNCH(c, k_pad3, grid_for(c->nv, 256), 256, 0, c->coords.p, c->nv, c->x4.p);
  c->x4_fresh = true;
  return DM_OK;
}
int ensure_x4(dm_ctx* c) { return c->x4_fresh ? DM_OK : pad_x4(c); }

int face_stats(dm_ctx* c, double* max_face, double* max_vol) {
  if (int st = ensure_x4(c)) return st;
  DM_CK(c, c->redu.ensure(4));
  DM_CK(c, cudaMemsetAsync(c->redu.p, 0, 4 * sizeof(u64), c->stream));
  if (c->dim == 3) {
    Coords<3> X{c->x4.p};
    DM_LAUNCH(c, k_face_max<3>, grid_for(c->nE, 256), 256, 0, c->elems.p, X, c->nE, c->redu.p);
  } else {
    Coords<2> X{reinterpret_cast<const double2*>(c->coords.p)};
    DM_LAUNCH(c, k_face_max<2>, grid_for(c->nE, 256), 256, 0, c->elems.p, X, c->nE, c->redu.p);
  }
  u64 h[2];
  DM_CK(c, cudaMemcpyAsync(h, c->redu.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  if (max_face) std::memcpy(max_face, &h[0], sizeof(double));
  if (max_vol) std::memcpy(max_vol, &h[1], sizeof(double));
  return DM_OK;
}

}  // namespace dm

// ------------------------------------------------------------------ C-ABI
using namespace dm;

extern "C" int dm_check_closure(dm_ctx* c, double* residual, double* interior_residual) {
  if (!c || !residual) return DM_ERR_INVALID_ARG;
  if (!c->have_navs) return fail(c, DM_ERR_STATE, "closure check needs navs");
  int st = ensure_incoming(c);
  if (!st) st = ensure_x4(c);
  if (st) return st;
  const i64 nv = c->nv;
  DevBuf<uint8_t> mask;
  DM_CK(c, mask.ensure(static_cast<size_t>(nv)));
  DM_CK(c, c->red.ensure(static_cast<size_t>(c->dim * nv)));
  DM_CK(c, c->redu.ensure(4));
  DM_CK(c, cudaMemsetAsync(mask.p, 0, nv, c->stream));
  DM_CK(c, cudaMemsetAsync(c->redu.p, 0, 4 * sizeof(u64), c->stream));
  DM_LAUNCH(c, k_bmask, grid_for(c->nB * c->dim, 256), 256, 0, c->bnd.p, c->nB * c->dim, mask.p);
  if (c->dim == 3) {
    Coords<3> X{c->x4.p};
    DM_LAUNCH(c, k_closure_nodes<3>, grid_for(nv, 256), 256, 0, c->in_ptr.p, c->in_list.p, c->os.p,
              c->navs.p, mask.p, nv, c->red.p, c->redu.p);
    DM_LAUNCH(c, k_closure_bnd<3>, grid_for(c->nB, 256), 256, 0, c->bnd.p, X, c->nB, c->red.p);
    DM_LAUNCH(c, k_norm_max<3>, grid_for(nv, 256), 256, 0, c->red.p, nv, c->redu.p + 2);
    DM_LAUNCH(c, k_norm_max<3>, grid_for(c->ne, 256), 256, 0, c->navs.p, c->ne, c->redu.p);
  } else {
    Coords<2> X{reinterpret_cast<const double2*>(c->coords.p)};
    DM_LAUNCH(c, k_closure_nodes<2>, grid_for(nv, 256), 256, 0, c->in_ptr.p, c->in_list.p, c->os.p,
              c->navs.p, mask.p, nv, c->red.p, c->redu.p);
    DM_LAUNCH(c, k_closure_bnd<2>, grid_for(c->nB, 256), 256, 0, c->bnd.p, X, c->nB, c->red.p);
    DM_LAUNCH(c, k_norm_max<2>, grid_for(nv, 256), 256, 0, c->red.p, nv, c->redu.p + 2);
    DM_LAUNCH(c, k_norm_max<2>, grid_for(c->ne, 256), 256, 0, c->navs.p, c->ne, c->redu.p);
  }
  u64 h[4];
  DM_CK(c, cudaMemcpyAsync(h, c->redu.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  double nmax, rint, rall;
  std::memcpy(&nmax, &h[0], 8);
  std::memcpy(&rint, &h[1], 8);
  std::memcpy(&rall, &h[2], 8);
  *residual = nmax > 0.0 ? rall / nmax : rall;
  if (interior_residual) *interior_residual = nmax > 0.0 ? rint / nmax : rint;
  return DM_OK;
}

extern "C" int dm_check_linear_exactness(dm_ctx* c, const double* A, const double* b,
                                         double* residual) {
  if (!c || !A || !b || !residual) return DM_ERR_INVALID_ARG;
  if (!c->have_navs) return fail(c, DM_ERR_STATE, "exactness check needs navs");
  const int D = c->dim;
  Affine F{};
  F.zero = 1;
  for (int i = 0; i < D * D; ++i) {
    F.A[i] = A[i];
    F.zero &= A[i] == 0.0;
  }
  for (int i = 0; i < D; ++i) {
    F.b[i] = b[i];
    F.tr += A[i * D + i];
  }
  if (!F.zero && F.tr == 0.0)
    return fail(c, DM_ERR_INVALID_ARG, "trace(A) = 0: relative residual undefined");
  if (!F.zero && !c->have_vols) return fail(c, DM_ERR_STATE, "exactness check needs volumes");
  int st = ensure_incoming(c);
  if (st) return st;
  if (int sx = ensure_x4(c)) return sx;
  const i64 nv = c->nv, ne = c->ne;
  DevBuf<uint8_t> mask;
  DevBuf<double> phi;
  DM_CK(c, mask.ensure(static_cast<size_t>(nv)));
  DM_CK(c, phi.ensure(static_cast<size_t>(ne)));
  DM_CK(c, c->red.ensure(static_cast<size_t>(D * nv)));
  DM_CK(c, c->redu.ensure(4));
  DM_CK(c, cudaMemsetAsync(mask.p, 0, nv, c->stream));
  DM_CK(c, cudaMemsetAsync(c->redu.p, 0, 4 * sizeof(u64), c->stream));
  DM_LAUNCH(c, k_bmask, grid_for(c->nB * D, 256), 256, 0, c->bnd.p, c->nB * D, mask.p);
  if (D == 3) {
    Coords<3> X{c->x4.p};
    DM_LAUNCH(c, k_lin_phi<3>, grid_for(ne, 256), 256, 0, c->edges.p, X, c->navs.p, ne, F,
              phi.p, c->redu.p);
  } else {
    Coords<2> X{reinterpret_cast<const double2*>(c->coords.p)};
    DM_LAUNCH(c, k_lin_phi<2>, grid_for(ne, 256), 256, 0, c->edges.p, X, c->navs.p, ne, F,
              phi.p, c->redu.p);
  }
  DM_LAUNCH(c, k_lin_nodes, grid_for(nv, 256), 256, 0, c->in_ptr.p, c->in_list.p, c->os.p, phi.p,
            F.zero ? nullptr : c->vols.p, mask.p, nv, F, c->red.p, c->redu.p);
  if (F.zero) {
    if (D == 3) {
      Coords<3> X{c->x4.p};
      DM_LAUNCH(c, k_lin_bnd<3>, grid_for(c->nB, 256), 256, 0, c->bnd.p, X, c->nB, F, c->red.p);
    } else {
      Coords<2> X{reinterpret_cast<const double2*>(c->coords.p)};
      DM_LAUNCH(c, k_lin_bnd<2>, grid_for(c->nB, 256), 256, 0, c->bnd.p, X, c->nB, F, c->red.p);
    }
    DM_LAUNCH(c, k_abs_max, grid_for(nv, 256), 256, 0, c->red.p, nv, c->redu.p + 1);
  }
  u64 h[2];
  DM_CK(c, cudaMemcpyAsync(h, c->redu.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  double pmax, r;
  std::memcpy(&pmax, &h[0], 8);
  std::memcpy(&r, &h[1], 8);
  *residual = F.zero && pmax > 0.0 ? r / pmax : r;
  return DM_OK;
}

extern "C" int dm_check_total_volume(dm_ctx* c, double* rel, double* sum_v, double* sum_e) {
  if (!c || !rel) return DM_ERR_INVALID_ARG;
  if (!c->have_vols) return fail(c, DM_ERR_STATE, "total-volume check needs volumes");
  double sv = 0.0, se = 0.0;
  int st = device_sum(c, c->vols.p, c->nv, &sv);
  if (st) return st;
  st = compute_element_volumes(c);
  if (st) return st;
  st = device_sum(c, c->velem.p, c->nE, &se);
  if (st) return st;
  *rel = std::fabs(sv - se) / se;
  if (sum_v) *sum_v = sv;
  if (sum_e) *sum_e = se;
  return DM_OK;
}

extern "C" int dm_corrupt_nav(dm_ctx* c, int64_t e, double delta) {
  if (!c) return DM_ERR_INVALID_ARG;
  if (!c->have_navs) return fail(c, DM_ERR_STATE, "no navs to corrupt");
  if (e < 0 || e >= c->ne) return fail(c, DM_ERR_INVALID_ARG, "edge out of range");
  DM_LAUNCH(c, k_corrupt, 1, 1, 0, c->navs.p, e, c->dim, delta);
  return DM_OK;
}

extern "C" int dm_max_face_area(dm_ctx* c, double* out) {
  if (!c || !out) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "no mesh");
  return face_stats(c, out, nullptr);
}

extern "C" int dm_max_element_volume(dm_ctx* c, double* out) {
  if (!c || !out) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "no mesh");
  return face_stats(c, nullptr, out);
}

extern "C" int dm_total_volume(dm_ctx* c, double* out) {
  if (!c || !out) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "no mesh");
  int st = compute_element_volumes(c);
  if (st) return st;
  return device_sum(c, c->velem.p, c->nE, out);
}

extern "C" int dm_boundary_node_mask(dm_ctx* c, uint8_t* mask) {
  if (!c || !mask) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "no mesh");
  DevBuf<uint8_t> m;
  DM_CK(c, m.ensure(static_cast<size_t>(c->nv)));
  DM_CK(c, cudaMemsetAsync(m.p, 0, c->nv, c->stream));
  DM_LAUNCH(c, k_bmask, grid_for(c->nB * c->dim, 256), 256, 0, c->bnd.p, c->nB * c->dim, m.p);
  DM_CK(c, cudaMemcpyAsync(mask, m.p, c->nv, cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}
