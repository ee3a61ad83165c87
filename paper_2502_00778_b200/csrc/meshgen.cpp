// meshgen.cpp -- SPEC meshgen module as host C++.
//
// Generates the synthetic grids of BASELINE.json / SURVEY.md 8(d).  It is
// input synthesis, not part of the measured path; it is compiled into its own
// libdm_meshgen.so so CPU-only tests can use it without touching CUDA.
#include "dm_meshgen.h"

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

namespace {

struct SplitMix64 {
  std::uint64_t x;
  explicit SplitMix64(std::uint64_t seed) : x(seed) {}
  std::uint64_t next() {
    x += 0x9E3779B97F4A7C15ull;
    std::uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  // u in [0,1) with 53 random bits; jitter = (2u-1)*a*h.
  double unit() { return static_cast<double>(next() >> 11) * (1.0 / 9007199254740992.0); }
  double jitter(double a, double h) { return (2.0 * unit() - 1.0) * a * h; }
};

// Signed volume from integer lattice offsets: decides orientation exactly.
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

}  // namespace

extern "C" {

void dmg_tri_square_sizes(int n, int64_t* n_nodes, int64_t* n_elements, int64_t* n_boundary) {
  const int64_t m = n;
  if (n_nodes) *n_nodes = (m + 1) * (m + 1);
  if (n_elements) *n_elements = 2 * m * m;
  if (n_boundary) *n_boundary = 4 * m;
}

int dmg_tri_square(int n, uint64_t diag_seed, double amp, uint64_t seed, double* coords,
                   int32_t* elements, int32_t* boundary) {
  if (n < 1 || !coords || !elements || !boundary) return -1;
  const int32_t w = n + 1;
  const double h = 1.0 / n;
  auto id = [w](int i, int j) { return static_cast<int32_t>(i + w * j); };
  SplitMix64 rj(seed);
  for (int j = 0; j <= n; ++j)
    for (int i = 0; i <= n; ++i) {
      const std::size_t v = static_cast<std::size_t>(id(i, j));
      double x = (i == n) ? 1.0 : i * h;
      double y = (j == n) ? 1.0 : j * h;
      if (amp != 0.0 && i > 0 && i < n && j > 0 && j < n) {
        x += rj.jitter(amp, h);
        y += rj.jitter(amp, h);
      }
      coords[2 * v] = x;
      coords[2 * v + 1] = y;
    }
  SplitMix64 rd(diag_seed);
  std::size_t e = 0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      const int32_t a = id(i, j), b = id(i + 1, j), c = id(i, j + 1), d = id(i + 1, j + 1);
      bool main_diag = true;  // a-d
      if (diag_seed != 0) main_diag = (rd.unit() < 0.5);
      int32_t* t = elements + 6 * e;
      if (main_diag) {
        t[0] = a; t[1] = b; t[2] = d;
        t[3] = a; t[4] = d; t[5] = c;
      } else {
        t[0] = a; t[1] = b; t[2] = c;
        t[3] = b; t[4] = d; t[5] = c;
      }
      ++e;
    }
  std::size_t k = 0;
  for (int i = 0; i < n; ++i) { boundary[k++] = id(i, 0); boundary[k++] = id(i + 1, 0); }
  for (int j = 0; j < n; ++j) { boundary[k++] = id(n, j); boundary[k++] = id(n, j + 1); }
  for (int i = n; i > 0; --i) { boundary[k++] = id(i, n); boundary[k++] = id(i - 1, n); }
  for (int j = n; j > 0; --j) { boundary[k++] = id(0, j); boundary[k++] = id(0, j - 1); }
  return 0;
}

void dmg_tet_box_sizes(int nx, int ny, int nz, int64_t* n_nodes, int64_t* n_elements,
                       int64_t* n_boundary) {
  const int64_t a = nx, b = ny, c = nz;
  if (n_nodes) *n_nodes = (a + 1) * (b + 1) * (c + 1);
  if (n_elements) *n_elements = 6 * a * b * c;
  if (n_boundary) *n_boundary = 4 * (a * b + b * c + a * c);
}

int dmg_bl_z(int nz, double dz0, double ratio, double* z_nodes) {
  if (nz < 1 || !z_nodes) return -1;
  z_nodes[0] = 0.0;
  double dz = dz0;
  for (int k = 0; k < nz; ++k) {
    z_nodes[k + 1] = z_nodes[k] + dz;
    dz *= ratio;
  }
  return 0;
}

int dmg_tet_box(int nx, int ny, int nz, const double* z_nodes, int jitter_mode, double amp,
                uint64_t seed, double* coords, int32_t* elements, int32_t* boundary) {
  if (nx < 1 || ny < 1 || nz < 1 || !coords || !elements || !boundary) return -1;
  const int64_t sx = nx + 1, sxy = (int64_t)(nx + 1) * (ny + 1);
  auto id = [sx, sxy](int i, int j, int k) {
    return static_cast<int32_t>(i + sx * j + sxy * k);
  };
  const double hx = 1.0 / nx, hy = 1.0 / ny, hz = 1.0 / nz;
  SplitMix64 r(seed);
  for (int k = 0; k <= nz; ++k)
    for (int j = 0; j <= ny; ++j)
      for (int i = 0; i <= nx; ++i) {
        const std::size_t v = static_cast<std::size_t>(id(i, j, k));
        double x = (i == nx) ? 1.0 : i * hx;
        double y = (j == ny) ? 1.0 : j * hy;
        double z = z_nodes ? z_nodes[k] : ((k == nz) ? 1.0 : k * hz);
        const bool in_xy = i > 0 && i < nx && j > 0 && j < ny;
        if (amp != 0.0) {
          if (jitter_mode == 0 && in_xy && k > 0 && k < nz) {
            x += r.jitter(amp, hx);
            y += r.jitter(amp, hy);
            z += r.jitter(amp, hz);
          } else if (jitter_mode == 1 && in_xy) {
            x += r.jitter(amp, hx);
            y += r.jitter(amp, hy);
          }
        }
        coords[3 * v] = x;
        coords[3 * v + 1] = y;
        coords[3 * v + 2] = z;
      }
  // Kuhn split: one tet per axis permutation, path v000 -> +e_p0 -> +e_p1 -> v111.
  static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  std::size_t e = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i)
        for (const auto& p : perms) {
          int q[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {1, 1, 1}};
          q[1][p[0]] = 1;
          q[2][p[0]] = 1;
          q[2][p[1]] = 1;
          int ord[4] = {0, 1, 2, 3};
          if (det3(q[0], q[1], q[2], q[3]) < 0) std::swap(ord[2], ord[3]);
          int32_t* t = elements + 4 * e;
          for (int a = 0; a < 4; ++a)
            t[a] = id(i + q[ord[a]][0], j + q[ord[a]][1], k + q[ord[a]][2]);
          ++e;
        }
  // Boundary: each boundary quad's diagonal joins its lowest and highest
  // corners (the Kuhn faces); orientation fixed against the outward axis.
  std::size_t b = 0;
  const int dims[3] = {nx, ny, nz};
  for (int axis = 0; axis < 3; ++axis)
    for (int side = 0; side < 2; ++side) {
      const int ua = (axis + 1) % 3, va = (axis + 2) % 3;
      const int u_lo = ua < va ? ua : va, v_hi = ua < va ? va : ua;
      for (int vv = 0; vv < dims[v_hi]; ++vv)
        for (int uu = 0; uu < dims[u_lo]; ++uu) {
          int c[4][3];
          for (int t = 0; t < 4; ++t) {
            c[t][axis] = side ? dims[axis] : 0;
            c[t][u_lo] = uu + (t & 1);
            c[t][v_hi] = vv + (t >> 1);
          }
          // corners 00,10,01,11 in (u,v); diagonal 00-11
          const int tri[2][3] = {{0, 1, 3}, {0, 3, 2}};
          for (const auto& tr : tri) {
            int o[3] = {tr[0], tr[1], tr[2]};
            // normal . outward must be > 0; outward = (side ? +1 : -1) e_axis
            int d1[3], d2[3];
            for (int t = 0; t < 3; ++t) {
              d1[t] = c[o[1]][t] - c[o[0]][t];
              d2[t] = c[o[2]][t] - c[o[0]][t];
            }
            const long long n_axis =
                (long long)d1[(axis + 1) % 3] * d2[(axis + 2) % 3] -
                (long long)d1[(axis + 2) % 3] * d2[(axis + 1) % 3];
            if ((side ? n_axis : -n_axis) < 0) std::swap(o[1], o[2]);
            for (int t = 0; t < 3; ++t)
              boundary[3 * b + t] = id(c[o[t]][0], c[o[t]][1], c[o[t]][2]);
            ++b;
          }
        }
    }
  return 0;
}

int dmg_permute(int dim, int64_t n_nodes, int64_t n_elements, int64_t n_boundary,
                uint64_t node_seed, uint64_t elem_seed, double* coords, int32_t* elements,
                int32_t* boundary) {
  if ((dim != 2 && dim != 3) || n_nodes < 0 || n_elements < 0) return -1;
  const int npe = dim + 1;
  if (node_seed != 0) {
    std::vector<int32_t> perm(static_cast<std::size_t>(n_nodes));
    for (int64_t i = 0; i < n_nodes; ++i) perm[i] = static_cast<int32_t>(i);
    SplitMix64 r(node_seed);
    for (int64_t i = n_nodes - 1; i > 0; --i) {
      const int64_t j = static_cast<int64_t>(r.next() % static_cast<std::uint64_t>(i + 1));
      std::swap(perm[i], perm[j]);
    }
    // perm[old] = new id
    std::vector<double> c(coords, coords + dim * n_nodes);
    for (int64_t v = 0; v < n_nodes; ++v)
      for (int d = 0; d < dim; ++d) coords[dim * (int64_t)perm[v] + d] = c[dim * v + d];
    for (int64_t t = 0; t < n_elements * npe; ++t) elements[t] = perm[elements[t]];
    for (int64_t t = 0; t < n_boundary * dim; ++t) boundary[t] = perm[boundary[t]];
  }
  if (elem_seed != 0) {
    std::vector<int64_t> perm(static_cast<std::size_t>(n_elements));
    for (int64_t i = 0; i < n_elements; ++i) perm[i] = i;
    SplitMix64 r(elem_seed);
    for (int64_t i = n_elements - 1; i > 0; --i) {
      const int64_t j = static_cast<int64_t>(r.next() % static_cast<std::uint64_t>(i + 1));
      std::swap(perm[i], perm[j]);
    }
    std::vector<int32_t> el(elements, elements + n_elements * npe);
    for (int64_t e = 0; e < n_elements; ++e)
      for (int a = 0; a < npe; ++a) elements[npe * perm[e] + a] = el[npe * e + a];
  }
  return 0;
}

// Seeded random 2-3 flips: a generator of genuinely unstructured tetrahedral
// topology (ring lengths 3..10+) from any valid tet mesh.  Two tets (a,b,c,d)
// and (a,b,c,e) sharing the interior face abc become (a,b,d,e), (b,c,d,e),
// (c,a,d,e) when the segment d-e pierces abc (the three new volumes have one
// sign); conformity is kept (the union's boundary faces are unchanged).
// Interior faces are visited in a splitmix64(seed) shuffled order and a tet
// takes part in at most one flip; at most max_flips flips.  Writes
// n_elements + flips tets to out_elements (first the originals in place,
// flipped pairs rewritten, then the third tets appended), all positively
// oriented; returns the number of flips.
int64_t dmg_flip23(int64_t n_nodes, const double* x, int64_t n_elements, const int32_t* el,
                   int64_t max_flips, uint64_t seed, int32_t* out) {
  if (n_nodes < 0 || n_elements < 0 || !x || !el || !out || n_nodes >= (int64_t(1) << 31))
    return -1;
  // faces keyed by their sorted node triple (32 bits each)
  using Key = unsigned __int128;
  std::vector<std::pair<Key, int64_t>> f;
  f.reserve(static_cast<std::size_t>(4 * n_elements));
  for (int64_t e = 0; e < n_elements; ++e)
    for (int o = 0; o < 4; ++o) {
      int v[3], q = 0;
      for (int a = 0; a < 4; ++a)
        if (a != o) v[q++] = el[4 * e + a];
      std::sort(v, v + 3);
      const Key key = static_cast<Key>(static_cast<uint32_t>(v[0])) << 64 |
                      static_cast<Key>(static_cast<uint32_t>(v[1])) << 32 |
                      static_cast<Key>(static_cast<uint32_t>(v[2]));
      f.push_back({key, 4 * e + o});
    }
  std::sort(f.begin(), f.end());
  std::vector<std::pair<int64_t, int64_t>> inner;  // (tet*4+opposite local) pairs
  for (std::size_t i = 0; i + 1 < f.size(); ++i)
    if (f[i].first == f[i + 1].first) inner.push_back({f[i].second, f[i + 1].second});
  SplitMix64 r(seed);
  for (std::size_t i = inner.size(); i > 1; --i)
    std::swap(inner[i - 1], inner[static_cast<std::size_t>(r.next() % i)]);
  std::copy(el, el + 4 * n_elements, out);
  std::vector<uint8_t> used(static_cast<std::size_t>(n_elements), 0);
  auto vol = [&](int a, int b, int c, int d) {
    const double* p = x + 3 * static_cast<int64_t>(a);
    const double* q = x + 3 * static_cast<int64_t>(b);
    const double* s = x + 3 * static_cast<int64_t>(c);
    const double* t = x + 3 * static_cast<int64_t>(d);
    const double u0 = q[0] - p[0], u1 = q[1] - p[1], u2 = q[2] - p[2];
    const double v0 = s[0] - p[0], v1 = s[1] - p[1], v2 = s[2] - p[2];
    const double w0 = t[0] - p[0], w1 = t[1] - p[1], w2 = t[2] - p[2];
    return (u1 * v2 - u2 * v1) * w0 + (u2 * v0 - u0 * v2) * w1 + (u0 * v1 - u1 * v0) * w2;
  };
  int64_t flips = 0, next = n_elements;
  for (const auto& [fa, fb] : inner) {
    if (flips >= max_flips) break;
    const int64_t t1 = fa >> 2, t2 = fb >> 2;
    if (used[t1] || used[t2]) continue;
    const int d = el[4 * t1 + (fa & 3)], e = el[4 * t2 + (fb & 3)];
    int abc[3], q = 0;
    for (int a = 0; a < 4; ++a)
      if (a != (fa & 3)) abc[q++] = el[4 * t1 + a];
    const int tri[3][2] = {{abc[0], abc[1]}, {abc[1], abc[2]}, {abc[2], abc[0]}};
    double vs[3];
    for (int k = 0; k < 3; ++k) vs[k] = vol(tri[k][0], tri[k][1], d, e);
    const bool pos = vs[0] > 0 && vs[1] > 0 && vs[2] > 0;
    const bool neg = vs[0] < 0 && vs[1] < 0 && vs[2] < 0;
    if (!pos && !neg) continue;  // d-e misses the face: no valid 2-3 flip
    // reject slivers: each new volume at least 1e-3 of the pair's mean
    const double total = std::abs(vs[0]) + std::abs(vs[1]) + std::abs(vs[2]);
    if (std::min({std::abs(vs[0]), std::abs(vs[1]), std::abs(vs[2])}) < 1e-3 * total / 3) continue;
    used[t1] = used[t2] = 1;
    int32_t* slots[3] = {out + 4 * t1, out + 4 * t2, out + 4 * next};
    for (int k = 0; k < 3; ++k) {
      int32_t* t = slots[k];
      t[0] = tri[k][0];
      t[1] = tri[k][1];
      t[2] = pos ? d : e;
      t[3] = pos ? e : d;
    }
    ++next;
    ++flips;
  }
  return flips;
}

int64_t dmg_first_inverted(int dim, int64_t n_elements, const double* x, const int32_t* el) {
  for (int64_t e = 0; e < n_elements; ++e) {
    double v;
    if (dim == 2) {
      const double* a = x + 2 * (int64_t)el[3 * e];
      const double* b = x + 2 * (int64_t)el[3 * e + 1];
      const double* c = x + 2 * (int64_t)el[3 * e + 2];
      v = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]);
    } else {
      const double* a = x + 3 * (int64_t)el[4 * e];
      const double* b = x + 3 * (int64_t)el[4 * e + 1];
      const double* c = x + 3 * (int64_t)el[4 * e + 2];
      const double* d = x + 3 * (int64_t)el[4 * e + 3];
      const double u0 = b[0] - a[0], u1 = b[1] - a[1], u2 = b[2] - a[2];
      const double v0 = c[0] - a[0], v1 = c[1] - a[1], v2 = c[2] - a[2];
      const double w0 = d[0] - a[0], w1 = d[1] - a[1], w2 = d[2] - a[2];
      v = (u1 * v2 - u2 * v1) * w0 + (u2 * v0 - u0 * v2) * w1 + (u0 * v1 - u1 * v0) * w2;
    }
    if (!(v > 0.0)) return e;
  }
  return -1;
}

}  // extern "C"
