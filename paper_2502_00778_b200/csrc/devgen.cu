// devgen.cu -- the SPEC meshgen module on the device.
//
// the BASELINE grids are synthesised straight into the
// context's device buffers instead of on the host plus a 2 GB upload at C5.
// Bitwise the same grids as the host generator (csrc/meshgen.cpp,
// include/dm_meshgen.h):
//   * splitmix64 is counter-based -- the n-th draw of a stream seeded with s
//     is mix(s + (n+1) * 0x9E3779B97F4A7C15) -- so every node computes its own
//     draw indices (the host draws in node order, x then y (then z), only for
//     jittered nodes) and the same arithmetic (2u - 1) * a * h;
//   * elements and boundary facets are written per hex / quad at the index
//     the host loops give them;
//   * the random relabelling (Fisher-Yates, j = next() % (i+1)) is inherently
//     sequential: the permutation arrays are drawn on the host (4 B per node
//     / 8 B per element) and applied on the device.
#include <cstring>
#include <utility>
#include <vector>

#include "dm_internal.cuh"

namespace dm {
namespace {

constexpr u64 kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ u64 smix(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// n-th draw (0-based) of splitmix64(seed), as u in [0, 1)
__device__ __forceinline__ double unit_n(u64 seed, u64 n) {
  return static_cast<double>(smix(seed + (n + 1) * kGolden) >> 11) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double jitter_n(u64 seed, u64 n, double a, double h) {
  return (2.0 * unit_n(seed, n) - 1.0) * a * h;
}

__global__ void k_gen_tet_coords(int nx, int ny, int nz, const double* __restrict__ zn, int mode,
                                 double amp, u64 seed, double* __restrict__ x) {
  const i64 v = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 sx = nx + 1, sxy = sx * (ny + 1);
  if (v >= sxy * (nz + 1)) return;
  const int k = static_cast<int>(v / sxy), j = static_cast<int>((v % sxy) / sx),
            i = static_cast<int>(v % sx);
  const double hx = 1.0 / nx, hy = 1.0 / ny, hz = 1.0 / nz;
  double px = (i == nx) ? 1.0 : i * hx;
  double py = (j == ny) ? 1.0 : j * hy;
  double pz = zn ? zn[k] : ((k == nz) ? 1.0 : k * hz);
  const bool in_xy = i > 0 && i < nx && j > 0 && j < ny;
  if (amp != 0.0) {
    if (mode == 0 && in_xy && k > 0 && k < nz) {
      const u64 q = static_cast<u64>((i - 1) + static_cast<i64>(nx - 1) *
                                                   ((j - 1) + static_cast<i64>(ny - 1) * (k - 1)));
      px += jitter_n(seed, 3 * q, amp, hx);
      py += jitter_n(seed, 3 * q + 1, amp, hy);
      pz += jitter_n(seed, 3 * q + 2, amp, hz);
    } else if (mode == 1 && in_xy) {
      const u64 q = static_cast<u64>((i - 1) + static_cast<i64>(nx - 1) *
                                                   ((j - 1) + static_cast<i64>(ny - 1) * k));
      px += jitter_n(seed, 2 * q, amp, hx);
      py += jitter_n(seed, 2 * q + 1, amp, hy);
    }
  }
  x[3 * v] = px;
  x[3 * v + 1] = py;
  x[3 * v + 2] = pz;
}

// corner offsets (di, dj, dk) of the 6 Kuhn tets in output vertex order
struct KuhnPattern {
  int8_t c[6][4][3];
};

__global__ void k_gen_tet_elems(int nx, int ny, int nz, KuhnPattern P, int32_t* __restrict__ el) {
  const i64 h = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h >= static_cast<i64>(nx) * ny * nz) return;
  const i64 sx = nx + 1, sxy = sx * (ny + 1);
  const int i = static_cast<int>(h % nx), j = static_cast<int>((h / nx) % ny),
            k = static_cast<int>(h / (static_cast<i64>(nx) * ny));
  for (int p = 0; p < 6; ++p)
    for (int a = 0; a < 4; ++a)
      el[24 * h + 4 * p + a] = static_cast<int32_t>((i + P.c[p][a][0]) + sx * (j + P.c[p][a][1]) +
                                                    sxy * (k + P.c[p][a][2]));
}

struct BoxFaces {
  i64 base[7];  // first boundary triangle of (axis, side) = 2 * axis + side
  int dims[3];
};

__global__ void k_gen_tet_bnd(int nx, int ny, BoxFaces F, int32_t* __restrict__ bnd) {
  const i64 b = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= F.base[6]) return;
  int f = 0;
  while (b >= F.base[f + 1]) ++f;
  const int axis = f >> 1, side = f & 1;
  const int ua = (axis + 1) % 3, va = (axis + 2) % 3;
  const int u_lo = ua < va ? ua : va, v_hi = ua < va ? va : ua;
  const i64 r = b - F.base[f];
  const int tri = static_cast<int>(r & 1);
  const i64 quad = r >> 1;
  const int uu = static_cast<int>(quad % F.dims[u_lo]), vv = static_cast<int>(quad / F.dims[u_lo]);
  int c[4][3];
  for (int t = 0; t < 4; ++t) {
    c[t][axis] = side ? F.dims[axis] : 0;
    c[t][u_lo] = uu + (t & 1);
    c[t][v_hi] = vv + (t >> 1);
  }
  int o[3] = {0, tri ? 3 : 1, tri ? 2 : 3};  // corners 00,10,01,11; diagonal 00-11
  int d1[3], d2[3];
  for (int t = 0; t < 3; ++t) {
    d1[t] = c[o[1]][t] - c[o[0]][t];
    d2[t] = c[o[2]][t] - c[o[0]][t];
  }
  const long long n_axis = static_cast<long long>(d1[(axis + 1) % 3]) * d2[(axis + 2) % 3] -
                           static_cast<long long>(d1[(axis + 2) % 3]) * d2[(axis + 1) % 3];
  if ((side ? n_axis : -n_axis) < 0) {
    const int s = o[1];
    o[1] = o[2];
    o[2] = s;
  }
  const i64 sx = nx + 1, sxy = sx * (ny + 1);
  for (int t = 0; t < 3; ++t)
    bnd[3 * b + t] = static_cast<int32_t>(c[o[t]][0] + sx * c[o[t]][1] + sxy * c[o[t]][2]);
}

__global__ void k_gen_tri(int n, u64 diag_seed, double amp, u64 seed, double* __restrict__ x,
                          int32_t* __restrict__ el) {
  const i64 v = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 w = n + 1;
  if (v < w * w) {  // node (i, j)
    const int i = static_cast<int>(v % w), j = static_cast<int>(v / w);
    const double h = 1.0 / n;
    double px = (i == n) ? 1.0 : i * h;
    double py = (j == n) ? 1.0 : j * h;
    if (amp != 0.0 && i > 0 && i < n && j > 0 && j < n) {
      const u64 q = static_cast<u64>((i - 1) + static_cast<i64>(n - 1) * (j - 1));
      px += jitter_n(seed, 2 * q, amp, h);
      py += jitter_n(seed, 2 * q + 1, amp, h);
    }
    x[2 * v] = px;
    x[2 * v + 1] = py;
  }
  if (v < static_cast<i64>(n) * n) {  // quad (i, j), two CCW triangles
    const int i = static_cast<int>(v % n), j = static_cast<int>(v / n);
    const int32_t a = static_cast<int32_t>(i + w * j), b = a + 1,
                  c = static_cast<int32_t>(i + w * (j + 1)), d = c + 1;
    const bool main_diag = diag_seed == 0 || unit_n(diag_seed, static_cast<u64>(v)) < 0.5;
    int32_t* t = el + 6 * v;
    if (main_diag) {
      t[0] = a; t[1] = b; t[2] = d;
      t[3] = a; t[4] = d; t[5] = c;
    } else {
      t[0] = a; t[1] = b; t[2] = c;
      t[3] = b; t[4] = d; t[5] = c;
    }
  }
}

__global__ void k_gen_tri_bnd(int n, int32_t* __restrict__ bnd) {
  const i64 q = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= 4ll * n) return;
  const int s = static_cast<int>(q / n), r = static_cast<int>(q % n);
  const int w = n + 1;
  auto id = [w](int i, int j) { return static_cast<int32_t>(i + w * j); };
  int32_t a, b;
  if (s == 0) { a = id(r, 0); b = id(r + 1, 0); }
  else if (s == 1) { a = id(n, r); b = id(n, r + 1); }
  else if (s == 2) { a = id(n - r, n); b = id(n - r - 1, n); }
  else { a = id(0, n - r); b = id(0, n - r - 1); }
  bnd[2 * q] = a;
  bnd[2 * q + 1] = b;
}

// ---- relabelling: perm[old] = new
__global__ void k_perm_coords(const double* __restrict__ in, const int32_t* __restrict__ perm,
                              i64 nv, int D, double* __restrict__ out) {
  const i64 v = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= nv) return;
  for (int d = 0; d < D; ++d) out[D * static_cast<i64>(perm[v]) + d] = in[D * v + d];
}
__global__ void k_perm_ids(int32_t* __restrict__ ids, i64 n, const int32_t* __restrict__ perm) {
  const i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) ids[t] = perm[ids[t]];
}
__global__ void k_perm_rows(const int32_t* __restrict__ in, const int64_t* __restrict__ perm,
                            i64 n, int npe, int32_t* __restrict__ out) {
  const i64 e = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  for (int a = 0; a < npe; ++a) out[npe * perm[e] + a] = in[npe * e + a];
}

// Fisher-Yates as the host generator draws it (j = next() % (i+1), i from n-1 down)
template <typename T>
std::vector<T> fisher_yates(i64 n, u64 seed) {
  std::vector<T> p(static_cast<size_t>(n));
  for (i64 i = 0; i < n; ++i) p[i] = static_cast<T>(i);
  u64 x = seed;
  for (i64 i = n - 1; i > 0; --i) {
    x += kGolden;
    const i64 j = static_cast<i64>(smix(x) % static_cast<u64>(i + 1));
    std::swap(p[i], p[j]);
  }
  return p;
}

long long det3(const int* a, const int* b, const int* c, const int* d) {
  long long u[3], v[3], w[3];
  for (int t = 0; t < 3; ++t) {
    u[t] = b[t] - a[t];
    v[t] = c[t] - a[t];
    w[t] = d[t] - a[t];
  }
  return (u[1] * v[2] - u[2] * v[1]) * w[0] + (u[2] * v[0] - u[0] * v[2]) * w[1] +
         (u[0] * v[1] - u[1] * v[0]) * w[2];
}

int begin_mesh(dm_ctx* c, int dim, i64 nv, i64 nE, i64 nB) {
  if (nv >= (1ll << 31)) return fail(c, DM_ERR_UNSUPPORTED, "node ids are 32-bit");
  c->have_edges = c->have_in = c->have_bedge = c->have_n2e = c->have_ifl = c->have_tables = c->have_rings =
      false;
  c->have_navs = c->have_vols = false;
  c->navs_algo = -1;
  c->ne = c->n_bedge = c->n_derived = 0;
  c->dim = dim;
  c->nv = nv;
  c->nE = nE;
  c->nB = nB;
  DM_CK(c, c->coords.ensure(static_cast<size_t>(dim * (nv + 2))));  // row plan: even-rounded runs
  DM_CK(c, c->elems.ensure(static_cast<size_t>((dim + 1) * nE)));
  DM_CK(c, c->bnd.ensure(static_cast<size_t>(dim * nB)));
  return DM_OK;
}

}  // namespace
}  // namespace dm

using namespace dm;

extern "C" int dm_gen_tri_square(dm_ctx* c, int n, uint64_t diag_seed, double amp,
                                 uint64_t seed) {
  if (!c || !c->stream) return DM_ERR_INVALID_ARG;
  if (n < 1) return fail(c, DM_ERR_INVALID_ARG, "gen_tri_square: n < 1");
  const i64 m = n;
  int st = begin_mesh(c, 2, (m + 1) * (m + 1), 2 * m * m, 4 * m);
  if (st) return st;
  DM_LAUNCH(c, k_gen_tri, grid_for((m + 1) * (m + 1), 256), 256, 0, n, diag_seed, amp, seed,
            c->coords.p, c->elems.p);
  DM_LAUNCH(c, k_gen_tri_bnd, grid_for(4 * m, 256), 256, 0, n, c->bnd.p);
  st = coords_changed(c);
  if (st) return st;
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}

extern "C" int dm_gen_tet_box(dm_ctx* c, int nx, int ny, int nz, const double* z_nodes,
                              int jitter_mode, double amp, uint64_t seed) {
  if (!c || !c->stream) return DM_ERR_INVALID_ARG;
  if (nx < 1 || ny < 1 || nz < 1) return fail(c, DM_ERR_INVALID_ARG, "gen_tet_box: n < 1");
  if (jitter_mode != 0 && jitter_mode != 1)
    return fail(c, DM_ERR_INVALID_ARG, "gen_tet_box: jitter_mode must be 0 or 1");
  const i64 a = nx, b = ny, cz = nz;
  const i64 nv = (a + 1) * (b + 1) * (cz + 1), nE = 6 * a * b * cz,
            nB = 4 * (a * b + b * cz + a * cz);
  int st = begin_mesh(c, 3, nv, nE, nB);
  if (st) return st;
  DevBuf<double> zd;
  if (z_nodes) {
    DM_CK(c, zd.ensure(static_cast<size_t>(nz + 1)));
    DM_CK(c, cudaMemcpyAsync(zd.p, z_nodes, sizeof(double) * (nz + 1), cudaMemcpyHostToDevice,
                             c->stream));
  }
  DM_LAUNCH(c, k_gen_tet_coords, grid_for(nv, 256), 256, 0, nx, ny, nz, z_nodes ? zd.p : nullptr,
            jitter_mode, amp, seed, c->coords.p);
  // the six Kuhn tets: path v000 -> +e_p0 -> +e_p1 -> v111, positively ordered
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  KuhnPattern P{};
  for (int p = 0; p < 6; ++p) {
    int q[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {1, 1, 1}};
    q[1][perms[p][0]] = 1;
    q[2][perms[p][0]] = 1;
    q[2][perms[p][1]] = 1;
    int ord[4] = {0, 1, 2, 3};
    if (det3(q[0], q[1], q[2], q[3]) < 0) std::swap(ord[2], ord[3]);
    for (int v = 0; v < 4; ++v)
      for (int t = 0; t < 3; ++t) P.c[p][v][t] = static_cast<int8_t>(q[ord[v]][t]);
  }
  DM_LAUNCH(c, k_gen_tet_elems, grid_for(a * b * cz, 256), 256, 0, nx, ny, nz, P, c->elems.p);
  BoxFaces F{};
  F.dims[0] = nx;
  F.dims[1] = ny;
  F.dims[2] = nz;
  F.base[0] = 0;
  for (int f = 0; f < 6; ++f) {
    const int axis = f >> 1;
    const i64 quads = static_cast<i64>(F.dims[(axis + 1) % 3]) * F.dims[(axis + 2) % 3];
    F.base[f + 1] = F.base[f] + 2 * quads;
  }
  DM_LAUNCH(c, k_gen_tet_bnd, grid_for(nB, 256), 256, 0, nx, ny, F, c->bnd.p);
  if (z_nodes) DM_CK(c, cudaStreamSynchronize(c->stream));  // zd dies here
  st = coords_changed(c);
  if (st) return st;
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}

extern "C" int dm_gen_permute(dm_ctx* c, uint64_t node_seed, uint64_t elem_seed) {
  if (!c || !c->stream) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "dm_gen_permute before a mesh is set");
  const int D = c->dim, npe = D + 1;
  const i64 nv = c->nv, nE = c->nE, nB = c->nB;
  if (node_seed != 0 && nv > 0) {
    const std::vector<int32_t> p = fisher_yates<int32_t>(nv, node_seed);
    DevBuf<int32_t> dp;
    DevBuf<double> tmp;
    DM_CK(c, dp.ensure(static_cast<size_t>(nv)));
    DM_CK(c, tmp.ensure(static_cast<size_t>(D * nv)));
    DM_CK(c, cudaMemcpyAsync(dp.p, p.data(), sizeof(int32_t) * nv, cudaMemcpyHostToDevice,
                             c->stream));
    DM_CK(c, cudaMemcpyAsync(tmp.p, c->coords.p, sizeof(double) * D * nv,
                             cudaMemcpyDeviceToDevice, c->stream));
    DM_LAUNCH(c, k_perm_coords, grid_for(nv, 256), 256, 0, tmp.p, dp.p, nv, D, c->coords.p);
    DM_LAUNCH(c, k_perm_ids, grid_for(npe * nE, 256), 256, 0, c->elems.p, npe * nE, dp.p);
    DM_LAUNCH(c, k_perm_ids, grid_for(D * nB, 256), 256, 0, c->bnd.p, D * nB, dp.p);
    DM_CK(c, cudaStreamSynchronize(c->stream));
  }
  if (elem_seed != 0 && nE > 0) {
    const std::vector<int64_t> p = fisher_yates<int64_t>(nE, elem_seed);
    DevBuf<int64_t> dp;
    DevBuf<int32_t> tmp;
    DM_CK(c, dp.ensure(static_cast<size_t>(nE)));
    DM_CK(c, tmp.ensure(static_cast<size_t>(npe * nE)));
    DM_CK(c, cudaMemcpyAsync(dp.p, p.data(), sizeof(int64_t) * nE, cudaMemcpyHostToDevice,
                             c->stream));
    DM_CK(c, cudaMemcpyAsync(tmp.p, c->elems.p, sizeof(int32_t) * npe * nE,
                             cudaMemcpyDeviceToDevice, c->stream));
    DM_LAUNCH(c, k_perm_rows, grid_for(nE, 256), 256, 0, tmp.p, dp.p, nE, npe, c->elems.p);
    DM_CK(c, cudaStreamSynchronize(c->stream));
  }
  c->have_edges = c->have_in = c->have_bedge = c->have_n2e = c->have_ifl = c->have_tables = c->have_rings =
      false;
  c->have_navs = c->have_vols = false;
  c->ne = c->n_bedge = c->n_derived = 0;
  return coords_changed(c);
}

extern "C" int dm_get_mesh(dm_ctx* c, double* coords, int32_t* elements, int32_t* boundary) {
  if (!c) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "no mesh");
  const int D = c->dim;
  if (coords && c->nv)
    DM_CK(c, cudaMemcpyAsync(coords, c->coords.p, sizeof(double) * D * c->nv,
                             cudaMemcpyDeviceToHost, c->stream));
  if (elements && c->nE)
    DM_CK(c, cudaMemcpyAsync(elements, c->elems.p, sizeof(int32_t) * (D + 1) * c->nE,
                             cudaMemcpyDeviceToHost, c->stream));
  if (boundary && c->nB)
    DM_CK(c, cudaMemcpyAsync(boundary, c->bnd.p, sizeof(int32_t) * D * c->nB,
                             cudaMemcpyDeviceToHost, c->stream));
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}

extern "C" int dm_mesh_sizes(dm_ctx* c, int* dim, int64_t* n_nodes, int64_t* n_elements,
                             int64_t* n_boundary) {
  if (!c) return DM_ERR_INVALID_ARG;
  if (dim) *dim = c->dim;
  if (n_nodes) *n_nodes = c->nv;
  if (n_elements) *n_elements = c->nE;
  if (n_boundary) *n_boundary = c->nB;
  return DM_OK;
}
