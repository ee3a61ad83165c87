// geometry.cuh -- per-(element, edge) contributions evaluated in registers.
//
// Each function reproduces, operation for operation, the serial arithmetic of
// the oracle (oracle/oracle.c) so that with -fmad=false the GPU sums are
// bitwise equal to it when accumulated in the same order.
#pragma once

#include "dm_internal.cuh"

namespace dm {

constexpr int kTraditional = DM_NAV_TRADITIONAL;
constexpr int kDualFree = DM_NAV_DUALFREE;

template <int D>
struct Coords;

template <>
struct Coords<3> {
  const d4* __restrict__ p;
  __device__ __forceinline__ d4 operator[](int v) const { return ld_d4(p + v); }
  __device__ __forceinline__ d4 xyz(int v) const { return ld_d3(p + v); }
};
// Raw 3D coordinates (the caller's x, y, z per node, 24-byte records): read by
// the kernels of the default step, which take no coordinate copy
struct Coords3R {
  const double* __restrict__ p;
  __device__ __forceinline__ d4 operator[](int v) const {
    const double* q = p + 3 * static_cast<i64>(v);
    d4 r;
    r.x = __ldg(q);
    r.y = __ldg(q + 1);
    r.z = __ldg(q + 2);
    r.w = 0.0;
    return r;
  }
};
template <>
struct Coords<2> {
  const double2* __restrict__ p;
  __device__ __forceinline__ double2 operator[](int v) const { return ld_d2(p + v); }
  __device__ __forceinline__ double2 xyz(int v) const { return ld_d2(p + v); }
};

// Dual-free 3D: the
// unscaled cross product 2*n_j^E of the face opposite the origin j, with the
// face vertex order of tet_opposite_face (ref mesh.cpp:15,103-110).
template <typename CX>
__device__ __forceinline__ void df3(const CX& X, int v0, int v1, int v2, int v3, int ij,
                                    double& c0, double& c1, double& c2) {
  const unsigned f = (kOppPacked >> (6 * ij)) & 63u;
  const d4 p0 = X[sel4(v0, v1, v2, v3, f & 3)];
  const d4 p1 = X[sel4(v0, v1, v2, v3, (f >> 2) & 3)];
  const d4 p2 = X[sel4(v0, v1, v2, v3, (f >> 4) & 3)];
  cross3(p1.x - p0.x, p1.y - p0.y, p1.z - p0.z, p2.x - p0.x, p2.y - p0.y, p2.z - p0.z, c0, c1, c2);
}

// Dual-free 2D: (1/3) n_j^E with
// n_i^E = (q_y - p_y, p_x - q_x), p = el[(i+1)%3], q = el[(i+2)%3]
// (ref mesh.cpp:97-101).
__device__ __forceinline__ void df2(const Coords<2>& X, int v0, int v1, int v2, int ij, double& c0,
                                    double& c1) {
  const double2 p = X[sel3(v0, v1, v2, ij == 2 ? 0 : ij + 1)];
  const double2 q = X[sel3(v0, v1, v2, ij == 0 ? 2 : ij - 1)];
  c0 = (1.0 / 3.0) * (q.y - p.y);
  c1 = (1.0 / 3.0) * (p.x - q.x);
}

// Traditional 3D:
// c = (E-m)x(L-m) + (R-m)x(E-m), sign fixed so that c.(x_k-x_j) >= 0.
// x0..x3 in local order (for the centroid sum); xl / xr are the two other
// local nodes in ascending local order.
__device__ __forceinline__ void tr3_core(const d4& x0, const d4& x1, const d4& x2, const d4& x3,
                                         const d4& xj, const d4& xk, const d4& xl, const d4& xr,
                                         double& c0, double& c1, double& c2) {
  const double mx = (xj.x + xk.x) * 0.5, my = (xj.y + xk.y) * 0.5, mz = (xj.z + xk.z) * 0.5;
  const double Ex = (x0.x + x1.x + x2.x + x3.x) * 0.25;
  const double Ey = (x0.y + x1.y + x2.y + x3.y) * 0.25;
  const double Ez = (x0.z + x1.z + x2.z + x3.z) * 0.25;
  const double Lx = (xj.x + xl.x + xk.x) * (1.0 / 3.0);
  const double Ly = (xj.y + xl.y + xk.y) * (1.0 / 3.0);
  const double Lz = (xj.z + xl.z + xk.z) * (1.0 / 3.0);
  const double Rx = (xj.x + xr.x + xk.x) * (1.0 / 3.0);
  const double Ry = (xj.y + xr.y + xk.y) * (1.0 / 3.0);
  const double Rz = (xj.z + xr.z + xk.z) * (1.0 / 3.0);
  const double emx = Ex - mx, emy = Ey - my, emz = Ez - mz;
  double a0, a1, a2, b0, b1, b2;
  cross3(emx, emy, emz, Lx - mx, Ly - my, Lz - mz, a0, a1, a2);
  cross3(Rx - mx, Ry - my, Rz - mz, emx, emy, emz, b0, b1, b2);
  c0 = a0 + b0;
  c1 = a1 + b1;
  c2 = a2 + b2;
  if (c0 * (xk.x - xj.x) + c1 * (xk.y - xj.y) + c2 * (xk.z - xj.z) < 0.0) {
    c0 = -c0;
    c1 = -c1;
    c2 = -c2;
  }
}

template <typename CX>
__device__ __forceinline__ void tr3(const CX& X, int v0, int v1, int v2, int v3, int ij,
                                    int ik, double& c0, double& c1, double& c2) {
  const d4 x0 = X[v0], x1 = X[v1], x2 = X[v2], x3 = X[v3];
  const unsigned rest = 0xFu & ~((1u << ij) | (1u << ik));
  const int il = __ffs(rest) - 1;
  const int ir = __ffs(rest & (rest - 1)) - 1;
  auto pick = [&](int i) -> d4 { return i == 0 ? x0 : (i == 1 ? x1 : (i == 2 ? x2 : x3)); };
  tr3_core(x0, x1, x2, x3, pick(ij), pick(ik), pick(il), pick(ir), c0, c1, c2);
}

// Traditional 2D: rotation of t = x_E - x_m with positive
// dot against x_k - x_j.
__device__ __forceinline__ void tr2_core(const double2& x0, const double2& x1, const double2& x2,
                                         const double2& xj, const double2& xk, double& c0,
                                         double& c1) {
  const double tx = (x0.x + x1.x + x2.x) * (1.0 / 3.0) - (xj.x + xk.x) * 0.5;
  const double ty = (x0.y + x1.y + x2.y) * (1.0 / 3.0) - (xj.y + xk.y) * 0.5;
  c0 = ty;
  c1 = -tx;
  if (c0 * (xk.x - xj.x) + c1 * (xk.y - xj.y) < 0.0) {
    c0 = -c0;
    c1 = -c1;
  }
}

__device__ __forceinline__ void tr2(const Coords<2>& X, int v0, int v1, int v2, int ij, int ik,
                                    double& c0, double& c1) {
  const double2 x0 = X[v0], x1 = X[v1], x2 = X[v2];
  auto pick = [&](int i) -> double2 { return i == 0 ? x0 : (i == 1 ? x1 : x2); };
  tr2_core(x0, x1, x2, pick(ij), pick(ik), c0, c1);
}

// Boundary directed area n_B (ref mesh.cpp:113-127).
template <typename CX>
__device__ __forceinline__ void bnormal3(const CX& X, const int32_t* bl, double& n0, double& n1,
                                         double& n2) {
  const d4 j = X[__ldg(bl)], r = X[__ldg(bl + 1)], l = X[__ldg(bl + 2)];
  double c0, c1, c2;
  cross3(r.x - j.x, r.y - j.y, r.z - j.z, l.x - j.x, l.y - j.y, l.z - j.z, c0, c1, c2);
  n0 = 0.5 * c0;
  n1 = 0.5 * c1;
  n2 = 0.5 * c2;
}
__device__ __forceinline__ void bnormal2(const Coords<2>& X, const int32_t* bl, double& n0,
                                         double& n1) {
  const double2 j = X[__ldg(bl)], k = X[__ldg(bl + 1)];
  n0 = k.y - j.y;
  n1 = j.x - k.x;
}

// Signed element volume (ref mesh.cpp:75-92): 2D 0.5*cross, 3D (uxv).w / 6.0.
template <typename CX>
__device__ __forceinline__ double evol3(const CX& X, int v0, int v1, int v2, int v3) {
  const d4 a = X[v0], b = X[v1], c = X[v2], d = X[v3];
  double uv0, uv1, uv2;
  cross3(b.x - a.x, b.y - a.y, b.z - a.z, c.x - a.x, c.y - a.y, c.z - a.z, uv0, uv1, uv2);
  return (uv0 * (d.x - a.x) + uv1 * (d.y - a.y) + uv2 * (d.z - a.z)) / 6.0;
}
__device__ __forceinline__ double evol2(const Coords<2>& X, int v0, int v1, int v2) {
  const double2 a = X[v0], b = X[v1], c = X[v2];
  return 0.5 * ((b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x));
}

}  // namespace dm
