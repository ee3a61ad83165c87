/* oracle.c -- serial CPU restatement of the grid-metric path.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Build with -ffp-contract=off.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ref mesh.cpp:15 -- outward faces of a positive tet, entry i opposite node i */
static const int kOppFace[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};
/* ref mesh.cpp:17 (3D) and mesh.cpp:263-265 (2D) local edge order */
static const int kTetEdge[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
static const int kTriEdge[3][2] = {{0, 1}, {1, 2}, {2, 0}};

static void cross3(const double* u, const double* v, double* c) {
  /* ref mesh.cpp:25-27 */
  c[0] = u[1] * v[2] - u[2] * v[1];
  c[1] = u[2] * v[0] - u[0] * v[2];
  c[2] = u[0] * v[1] - u[1] * v[0];
}

void or_free(void* p) { free(p); }

/* ---- edges ------------------------------------------------------------- */

/* Restates build_edges (mesh.cpp:256-285): the set of (min,max) pairs in
 * lexicographic order plus the origin CSR.  Implemented as a counting sort
 * on the origin followed by a per-row sort + unique, which yields the same
 * sequence as unordered_set + std::sort. */
static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

int64_t or_build_edges(int dim, int64_t n_nodes, const int32_t* el, int64_t n_elements,
                       int32_t** edges_out, uint64_t** os_out) {
  const int npe = dim + 1, L = dim == 2 ? 3 : 6;
  const int(*loc)[2] = dim == 2 ? kTriEdge : kTetEdge;
  uint64_t* cnt = (uint64_t*)calloc((size_t)n_nodes + 1, sizeof(uint64_t));
  if (!cnt) return -1;
  for (int64_t e = 0; e < n_elements; ++e)
    for (int l = 0; l < L; ++l) {
      int32_t a = el[npe * e + loc[l][0]], b = el[npe * e + loc[l][1]];
      cnt[(a < b ? a : b) + 1]++;
    }
  for (int64_t v = 0; v < n_nodes; ++v) cnt[v + 1] += cnt[v];
  const uint64_t m = cnt[n_nodes];
  int32_t* dst = (int32_t*)malloc((m ? m : 1) * sizeof(int32_t));
  uint64_t* fill = (uint64_t*)malloc(((size_t)n_nodes + 1) * sizeof(uint64_t));
  if (!dst || !fill) return -1;
  memcpy(fill, cnt, ((size_t)n_nodes + 1) * sizeof(uint64_t));
  for (int64_t e = 0; e < n_elements; ++e)
    for (int l = 0; l < L; ++l) {
      int32_t a = el[npe * e + loc[l][0]], b = el[npe * e + loc[l][1]];
      int32_t j = a < b ? a : b, k = a < b ? b : a;
      dst[fill[j]++] = k;
    }
  uint64_t* os = (uint64_t*)malloc(((size_t)n_nodes + 1) * sizeof(uint64_t));
  int32_t* edges = (int32_t*)malloc(2 * (m ? m : 1) * sizeof(int32_t));
  if (!os || !edges) return -1;
  uint64_t ne = 0;
  for (int64_t j = 0; j < n_nodes; ++j) {
    os[j] = ne;
    int32_t* row = dst + cnt[j];
    size_t len = (size_t)(cnt[j + 1] - cnt[j]);
    qsort(row, len, sizeof(int32_t), cmp_i32);
    for (size_t t = 0; t < len; ++t)
      if (t == 0 || row[t] != row[t - 1]) {
        edges[2 * ne] = (int32_t)j;
        edges[2 * ne + 1] = row[t];
        ++ne;
      }
  }
  os[n_nodes] = ne;
  free(cnt);
  free(fill);
  free(dst);
  *edges_out = edges;
  *os_out = os;
  return (int64_t)ne;
}

/* ref EdgeList::edge_of, mesh.cpp:58-73 (lower bound in row min(a,b)). */
int32_t or_edge_of(const int32_t* edges, const uint64_t* os, int64_t n_nodes, int32_t a,
                   int32_t b) {
  if (a > b) {
    int32_t t = a;
    a = b;
    b = t;
  }
  if (a < 0 || (int64_t)a + 1 >= n_nodes + 1) return -1;
  uint64_t lo = os[a], hi = os[a + 1];
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (edges[2 * mid + 1] < b)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < os[a + 1] && edges[2 * lo + 1] == b) return (int32_t)lo;
  return -1;
}

int or_edge_maps(int dim, int64_t n_nodes, const int32_t* el, int64_t n_elements,
                 const int32_t* edges, const uint64_t* os, int64_t n_edges, int32_t* e2l,
                 int32_t* inc_ptr, int32_t* inc) {
  const int npe = dim + 1, L = dim == 2 ? 3 : 6;
  const int(*loc)[2] = dim == 2 ? kTriEdge : kTetEdge;
  int32_t* map = e2l ? e2l : (int32_t*)malloc((size_t)(L * n_elements + 1) * sizeof(int32_t));
  if (!map) return -1;
  for (int64_t e = 0; e < n_elements; ++e)
    for (int l = 0; l < L; ++l) {
      int32_t id = or_edge_of(edges, os, n_nodes, el[npe * e + loc[l][0]], el[npe * e + loc[l][1]]);
      if (id < 0) return -2;
      map[L * e + l] = id;
    }
  if (inc_ptr) {
    memset(inc_ptr, 0, (size_t)(n_edges + 1) * sizeof(int32_t));
    for (int64_t t = 0; t < L * n_elements; ++t) inc_ptr[map[t] + 1]++;
    for (int64_t i = 0; i < n_edges; ++i) inc_ptr[i + 1] += inc_ptr[i];
    if (inc) {
      int32_t* fill = (int32_t*)malloc((size_t)(n_edges + 1) * sizeof(int32_t));
      if (!fill) return -1;
      memcpy(fill, inc_ptr, (size_t)(n_edges + 1) * sizeof(int32_t));
      for (int64_t t = 0; t < L * n_elements; ++t) inc[fill[map[t]]++] = (int32_t)(t / L);
      free(fill);
    }
  }
  if (!e2l) free(map);
  return 0;
}

/* ---- geometry ------------------------------------------------------------ */

double or_element_volume(int dim, const double* x, const int32_t* el) {
  /* ref mesh.cpp:75-92 */
  if (dim == 2) {
    const double *a = x + 2 * (int64_t)el[0], *b = x + 2 * (int64_t)el[1],
                 *c = x + 2 * (int64_t)el[2];
    return 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]));
  }
  const double *a = x + 3 * (int64_t)el[0], *b = x + 3 * (int64_t)el[1],
               *c = x + 3 * (int64_t)el[2], *d = x + 3 * (int64_t)el[3];
  double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  double w[3] = {d[0] - a[0], d[1] - a[1], d[2] - a[2]};
  double uv[3];
  cross3(u, v, uv);
  return (uv[0] * w[0] + uv[1] * w[1] + uv[2] * w[2]) / 6.0;
}

void or_opposite_face_normal(int dim, const double* x, const int32_t* el, int i, double* out) {
  /* ref mesh.cpp:94-111 */
  if (dim == 2) {
    const double* p = x + 2 * (int64_t)el[(i + 1) % 3];
    const double* q = x + 2 * (int64_t)el[(i + 2) % 3];
    out[0] = q[1] - p[1];
    out[1] = p[0] - q[0];
    out[2] = 0.0;
    return;
  }
  const int* f = kOppFace[i];
  const double *p0 = x + 3 * (int64_t)el[f[0]], *p1 = x + 3 * (int64_t)el[f[1]],
               *p2 = x + 3 * (int64_t)el[f[2]];
  double d1[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
  double d2[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
  double c[3];
  cross3(d1, d2, c);
  out[0] = 0.5 * c[0];
  out[1] = 0.5 * c[1];
  out[2] = 0.5 * c[2];
}

void or_boundary_normal(int dim, const double* x, const int32_t* bl, double* out) {
  /* ref mesh.cpp:113-127 */
  if (dim == 2) {
    const double *j = x + 2 * (int64_t)bl[0], *k = x + 2 * (int64_t)bl[1];
    out[0] = k[1] - j[1];
    out[1] = j[0] - k[0];
    out[2] = 0.0;
    return;
  }
  const double *j = x + 3 * (int64_t)bl[0], *r = x + 3 * (int64_t)bl[1],
               *l = x + 3 * (int64_t)bl[2];
  double d1[3] = {r[0] - j[0], r[1] - j[1], r[2] - j[2]};
  double d2[3] = {l[0] - j[0], l[1] - j[1], l[2] - j[2]};
  double c[3];
  cross3(d1, d2, c);
  out[0] = 0.5 * c[0];
  out[1] = 0.5 * c[1];
  out[2] = 0.5 * c[2];
}

/* ---- metrics ------------------------------------------------------------- */

static int boundary_pass(int dim, const double* x, int64_t n_nodes, const int32_t* bnd,
                         int64_t n_boundary, const int32_t* edges, const uint64_t* os,
                         double* navs) {
  /* every edge of every
   * boundary facet gets (1/(D(D+1))) n_B, in ascending facet order, facet
   * edges (v0,v1),(v1,v2),(v2,v0). */
  const double f = 1.0 / (double)(dim * (dim + 1));
  const int ne_b = dim == 2 ? 1 : 3;
  for (int64_t b = 0; b < n_boundary; ++b) {
    const int32_t* bl = bnd + dim * b;
    double nb[3];
    or_boundary_normal(dim, x, bl, nb);
    for (int t = 0; t < ne_b; ++t) {
      int32_t id = or_edge_of(edges, os, n_nodes, bl[t], bl[(t + 1) % dim]);
      if (id < 0) return -3;
      for (int d = 0; d < dim; ++d) navs[(int64_t)dim * id + d] += f * nb[d];
    }
  }
  return 0;
}

int or_navs_dualfree(int dim, const double* x, int64_t n_nodes, const int32_t* el,
                     int64_t n_elements, const int32_t* bnd, int64_t n_boundary,
                     const int32_t* edges, const uint64_t* os, int64_t n_edges,
                     const int32_t* e2l, double* navs) {
  /* SPEC.md:157-168. */
  const int npe = dim + 1, L = dim == 2 ? 3 : 6;
  const int(*loc)[2] = dim == 2 ? kTriEdge : kTetEdge;
  memset(navs, 0, (size_t)(dim * n_edges) * sizeof(double));
  for (int64_t e = 0; e < n_elements; ++e) {
    const int32_t* t = el + npe * e;
    for (int l = 0; l < L; ++l) {
      const int la = loc[l][0], lb = loc[l][1];
      const int ij = t[la] < t[lb] ? la : lb;
      int32_t id = e2l ? e2l[L * e + l] : or_edge_of(edges, os, n_nodes, t[la], t[lb]);
      if (id < 0) return -2;
      double* n = navs + (int64_t)dim * id;
      if (dim == 3) {
        /* pass 1: 2 n_j^E as the unscaled cross product */
        const int* f = kOppFace[ij];
        const double *p0 = x + 3 * (int64_t)t[f[0]], *p1 = x + 3 * (int64_t)t[f[1]],
                     *p2 = x + 3 * (int64_t)t[f[2]];
        double d1[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
        double d2[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
        double c[3];
        cross3(d1, d2, c);
        n[0] += c[0];
        n[1] += c[1];
        n[2] += c[2];
      } else {
        double nj[3];
        or_opposite_face_normal(2, x, t, ij, nj);
        n[0] += (1.0 / 3.0) * nj[0];
        n[1] += (1.0 / 3.0) * nj[1];
      }
    }
  }
  if (dim == 3) /* pass 2 */
    for (int64_t i = 0; i < 3 * n_edges; ++i) navs[i] *= (1.0 / 12.0);
  return boundary_pass(dim, x, n_nodes, bnd, n_boundary, edges, os, navs); /* pass 3 */
}

int or_navs_traditional(int dim, const double* x, int64_t n_nodes, const int32_t* el,
                        int64_t n_elements, const int32_t* edges, const uint64_t* os,
                        int64_t n_edges, const int32_t* e2l, double* navs) {
  /* SPEC.md:147-155, SURVEY App. A.9. */
  const int npe = dim + 1, L = dim == 2 ? 3 : 6;
  const int(*loc)[2] = dim == 2 ? kTriEdge : kTetEdge;
  memset(navs, 0, (size_t)(dim * n_edges) * sizeof(double));
  for (int64_t e = 0; e < n_elements; ++e) {
    const int32_t* t = el + npe * e;
    for (int l = 0; l < L; ++l) {
      const int la = loc[l][0], lb = loc[l][1];
      const int ij = t[la] < t[lb] ? la : lb, ik = t[la] < t[lb] ? lb : la;
      int32_t id = e2l ? e2l[L * e + l] : or_edge_of(edges, os, n_nodes, t[la], t[lb]);
      if (id < 0) return -2;
      double* n = navs + (int64_t)dim * id;
      if (dim == 2) {
        const double *xj = x + 2 * (int64_t)t[ij], *xk = x + 2 * (int64_t)t[ik];
        const double *x0 = x + 2 * (int64_t)t[0], *x1 = x + 2 * (int64_t)t[1],
                     *x2 = x + 2 * (int64_t)t[2];
        double c[2];
        double tx = (x0[0] + x1[0] + x2[0]) * (1.0 / 3.0) - (xj[0] + xk[0]) * 0.5;
        double ty = (x0[1] + x1[1] + x2[1]) * (1.0 / 3.0) - (xj[1] + xk[1]) * 0.5;
        c[0] = ty;
        c[1] = -tx;
        if (c[0] * (xk[0] - xj[0]) + c[1] * (xk[1] - xj[1]) < 0.0) {
          c[0] = -c[0];
          c[1] = -c[1];
        }
        n[0] += c[0];
        n[1] += c[1];
      } else {
        int other[2], no = 0;
        for (int q = 0; q < 4; ++q)
          if (q != la && q != lb) other[no++] = q;
        const double *xj = x + 3 * (int64_t)t[ij], *xk = x + 3 * (int64_t)t[ik],
                     *xl = x + 3 * (int64_t)t[other[0]], *xr = x + 3 * (int64_t)t[other[1]];
        const double *x0 = x + 3 * (int64_t)t[0], *x1 = x + 3 * (int64_t)t[1],
                     *x2 = x + 3 * (int64_t)t[2], *x3 = x + 3 * (int64_t)t[3];
        double m[3], E[3], Lc[3], R[3], em[3], lm[3], rm[3], c1[3], c2[3], c[3];
        for (int d = 0; d < 3; ++d) {
          m[d] = (xj[d] + xk[d]) * 0.5;
          E[d] = (x0[d] + x1[d] + x2[d] + x3[d]) * 0.25;
          Lc[d] = (xj[d] + xl[d] + xk[d]) * (1.0 / 3.0);
          R[d] = (xj[d] + xr[d] + xk[d]) * (1.0 / 3.0);
          em[d] = E[d] - m[d];
          lm[d] = Lc[d] - m[d];
          rm[d] = R[d] - m[d];
        }
        cross3(em, lm, c1);
        cross3(rm, em, c2);
        for (int d = 0; d < 3; ++d) c[d] = c1[d] + c2[d];
        if (c[0] * (xk[0] - xj[0]) + c[1] * (xk[1] - xj[1]) + c[2] * (xk[2] - xj[2]) < 0.0) {
          c[0] = -c[0];
          c[1] = -c[1];
          c[2] = -c[2];
        }
        n[0] += c[0];
        n[1] += c[1];
        n[2] += c[2];
      }
    }
  }
  if (dim == 3) /* deferred 1/2 */
    for (int64_t i = 0; i < 3 * n_edges; ++i) navs[i] *= 0.5;
  return 0;
}

int or_volumes_edge(int dim, const double* x, int64_t n_nodes, const int32_t* edges,
                    int64_t n_edges, const double* navs, double* V) {
  /* SPEC.md:170-178 */
  memset(V, 0, (size_t)n_nodes * sizeof(double));
  for (int64_t e = 0; e < n_edges; ++e) {
    const int32_t j = edges[2 * e], k = edges[2 * e + 1];
    const double *xj = x + (int64_t)dim * j, *xk = x + (int64_t)dim * k;
    const double* n = navs + (int64_t)dim * e;
    double s = (xk[0] - xj[0]) * n[0] + (xk[1] - xj[1]) * n[1];
    if (dim == 3) s = s + (xk[2] - xj[2]) * n[2];
    V[j] += s;
    V[k] += s;
  }
  const double f = 1.0 / (double)(2 * dim);
  for (int64_t v = 0; v < n_nodes; ++v) V[v] *= f;
  return 0;
}

int or_volumes_element(int dim, const double* x, int64_t n_nodes, const int32_t* el,
                       int64_t n_elements, double* V) {
  /* SPEC.md:180-188 */
  const int npe = dim + 1;
  memset(V, 0, (size_t)n_nodes * sizeof(double));
  for (int64_t e = 0; e < n_elements; ++e) {
    const double ve = or_element_volume(dim, x, el + npe * e);
    for (int i = 0; i < npe; ++i) V[el[npe * e + i]] += ve;
  }
  const double f = 1.0 / (double)(dim + 1);
  for (int64_t v = 0; v < n_nodes; ++v) V[v] *= f;
  return 0;
}

/* ---- verify -------------------------------------------------------------- */

static double vnorm(const double* a, int dim) {
  double s = 0.0;
  for (int d = 0; d < dim; ++d) s += a[d] * a[d];
  return sqrt(s);
}

int or_check_closure(int dim, const double* x, int64_t n_nodes, const int32_t* bnd,
                     int64_t n_boundary, const int32_t* edges, int64_t n_edges,
                     const double* navs, double* residual, double* interior_residual) {
  /* SPEC.md:245-253 */
  double* a = (double*)calloc((size_t)(dim * n_nodes) + 1, sizeof(double));
  unsigned char* isb = (unsigned char*)calloc((size_t)n_nodes + 1, 1);
  if (!a || !isb) return -1;
  double nmax = 0.0;
  for (int64_t e = 0; e < n_edges; ++e) {
    const int32_t j = edges[2 * e], k = edges[2 * e + 1];
    const double* n = navs + (int64_t)dim * e;
    for (int d = 0; d < dim; ++d) {
      a[(int64_t)dim * j + d] += n[d];
      a[(int64_t)dim * k + d] -= n[d];
    }
    double nn = vnorm(n, dim);
    if (nn > nmax) nmax = nn;
  }
  for (int64_t t = 0; t < dim * n_boundary; ++t) isb[bnd[t]] = 1;
  double ri = 0.0;
  for (int64_t v = 0; v < n_nodes; ++v)
    if (!isb[v]) {
      double r = vnorm(a + (int64_t)dim * v, dim);
      if (r > ri) ri = r;
    }
  const double f = 1.0 / (double)dim;
  for (int64_t b = 0; b < n_boundary; ++b) {
    double nb[3];
    or_boundary_normal(dim, x, bnd + dim * b, nb);
    for (int t = 0; t < dim; ++t)
      for (int d = 0; d < dim; ++d) a[(int64_t)dim * bnd[dim * b + t] + d] += f * nb[d];
  }
  double r = 0.0;
  for (int64_t v = 0; v < n_nodes; ++v) {
    double q = vnorm(a + (int64_t)dim * v, dim);
    if (q > r) r = q;
  }
  *residual = nmax > 0.0 ? r / nmax : r;
  if (interior_residual) *interior_residual = nmax > 0.0 ? ri / nmax : ri;
  free(a);
  free(isb);
  return 0;
}

int or_check_linear_exactness(int dim, const double* x, int64_t n_nodes, const int32_t* bnd,
                              int64_t n_boundary, const int32_t* edges, int64_t n_edges,
                              const double* navs, const double* V, const double* A,
                              const double* b, double* residual) {
  /* SPEC.md:265-274 (check_linear_exactness): F(x) = A x + b, arithmetic-average
   * edge flux phi = ((F_j + F_k) * 0.5) . n_jk; Res_j += phi, Res_k -= phi.
   * trace(A) != 0: max over interior nodes of |Res_j / V_j - tr| / |tr|.
   * A == 0: constant flux, boundary closure b . (1/D) n_B added at every node
   * of every boundary element, max_j |Res_j| / max_e |phi_e|. */
  int zero = 1;
  double tr = 0.0;
  for (int i = 0; i < dim * dim; ++i) zero &= A[i] == 0.0;
  for (int i = 0; i < dim; ++i) tr += A[i * dim + i];
  if (!zero && tr == 0.0) return -1;
  double* res = (double*)calloc((size_t)n_nodes + 1, sizeof(double));
  unsigned char* isb = (unsigned char*)calloc((size_t)n_nodes + 1, 1);
  if (!res || !isb) return -2;
  double pmax = 0.0;
  for (int64_t e = 0; e < n_edges; ++e) {
    const int32_t j = edges[2 * e], k = edges[2 * e + 1];
    const double *xj = x + (int64_t)dim * j, *xk = x + (int64_t)dim * k;
    const double* n = navs + (int64_t)dim * e;
    double phi = 0.0;
    for (int r = 0; r < dim; ++r) {
      double fj = b[r], fk = b[r];
      for (int c = 0; c < dim; ++c) {
        fj += A[r * dim + c] * xj[c];
        fk += A[r * dim + c] * xk[c];
      }
      phi += ((fj + fk) * 0.5) * n[r];
    }
    res[j] += phi;
    res[k] -= phi;
    if (fabs(phi) > pmax) pmax = fabs(phi);
  }
  double out = 0.0;
  if (zero) {
    const double f = 1.0 / (double)dim;
    for (int64_t q = 0; q < n_boundary; ++q) {
      double nb[3];
      or_boundary_normal(dim, x, bnd + dim * q, nb);
      double bn = 0.0;
      for (int d = 0; d < dim; ++d) bn += b[d] * nb[d];
      for (int t = 0; t < dim; ++t) res[bnd[dim * q + t]] += f * bn;
    }
    for (int64_t v = 0; v < n_nodes; ++v)
      if (fabs(res[v]) > out) out = fabs(res[v]);
    out = pmax > 0.0 ? out / pmax : out;
  } else {
    for (int64_t t = 0; t < dim * n_boundary; ++t) isb[bnd[t]] = 1;
    for (int64_t v = 0; v < n_nodes; ++v)
      if (!isb[v]) {
        const double r = fabs(res[v] / V[v] - tr) / fabs(tr);
        if (r > out) out = r;
      }
  }
  *residual = out;
  free(res);
  free(isb);
  return 0;
}

/* Neumaier summation. */
typedef struct {
  double s, c;
} ksum;
static void kadd(ksum* k, double v) {
  double t = k->s + v;
  if (fabs(k->s) >= fabs(v))
    k->c += (k->s - t) + v;
  else
    k->c += (v - t) + k->s;
  k->s = t;
}

int or_check_total_volume(int dim, const double* x, int64_t n_nodes, const int32_t* el,
                          int64_t n_elements, const double* V, double* rel, double* sum_v,
                          double* sum_e) {
  /* SPEC.md:255-263 */
  ksum a = {0.0, 0.0}, b = {0.0, 0.0};
  for (int64_t v = 0; v < n_nodes; ++v) kadd(&a, V[v]);
  for (int64_t e = 0; e < n_elements; ++e) kadd(&b, or_element_volume(dim, x, el + (dim + 1) * e));
  const double sv = a.s + a.c, se = b.s + b.c;
  if (sum_v) *sum_v = sv;
  if (sum_e) *sum_e = se;
  *rel = fabs(sv - se) / se;
  return 0;
}

double or_max_face_area(int dim, const double* x, const int32_t* el, int64_t n_elements) {
  /* ref mesh.cpp:325-330 */
  double m = 0.0;
  for (int64_t e = 0; e < n_elements; ++e)
    for (int i = 0; i <= dim; ++i) {
      double n[3];
      or_opposite_face_normal(dim, x, el + (dim + 1) * e, i, n);
      double a = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
      if (a > m) m = a;
    }
  return m;
}

double or_max_element_volume(int dim, const double* x, const int32_t* el, int64_t n_elements) {
  /* ref mesh.cpp:332-337 */
  double m = 0.0;
  for (int64_t e = 0; e < n_elements; ++e) {
    double v = fabs(or_element_volume(dim, x, el + (dim + 1) * e));
    if (v > m) m = v;
  }
  return m;
}

/* ---- multi-threaded form (bench reference arm) --------------------------- */
/* The serial loops above accumulate, for every edge, its element terms in
 * ascending element id and then its facet terms in ascending facet id, and
 * for every node its edge terms in ascending edge id (incoming edges first,
 * as they precede the node's own row).  The gathers below visit exactly those
 * terms in exactly that order -- one edge (node) per task -- so they produce
 * the same bits on any number of threads. */
#include <pthread.h>

struct or_plan {
  int dim;
  int64_t n_nodes, n_elements, n_edges;
  const int32_t *el, *bnd, *edges;
  int32_t *inc_ptr, *inc;  /* edge -> elements (ascending) */
  int32_t *bptr, *blist;   /* edge -> boundary facets (ascending) */
  int32_t *in_ptr, *in_list; /* node -> incoming edges (ascending) */
  uint64_t* os;
};

or_plan* or_plan_create(int dim, int64_t n_nodes, const int32_t* el, int64_t n_elements,
                        const int32_t* bnd, int64_t n_boundary, const int32_t* edges,
                        const uint64_t* os, int64_t n_edges) {
  or_plan* p = (or_plan*)calloc(1, sizeof(or_plan));
  if (!p) return NULL;
  const int L = dim == 2 ? 3 : 6, nbe = dim == 2 ? 1 : 3;
  p->dim = dim;
  p->n_nodes = n_nodes;
  p->n_elements = n_elements;
  p->n_edges = n_edges;
  p->el = el;
  p->bnd = bnd;
  p->edges = edges;
  p->inc_ptr = (int32_t*)malloc((size_t)(n_edges + 1) * sizeof(int32_t));
  p->inc = (int32_t*)malloc((size_t)(L * n_elements + 1) * sizeof(int32_t));
  p->bptr = (int32_t*)calloc((size_t)(n_edges + 1), sizeof(int32_t));
  p->blist = (int32_t*)malloc((size_t)(nbe * n_boundary + 1) * sizeof(int32_t));
  p->in_ptr = (int32_t*)calloc((size_t)(n_nodes + 1), sizeof(int32_t));
  p->in_list = (int32_t*)malloc((size_t)(n_edges + 1) * sizeof(int32_t));
  p->os = (uint64_t*)malloc((size_t)(n_nodes + 1) * sizeof(uint64_t));
  int32_t* fill = (int32_t*)malloc((size_t)(n_nodes + n_edges + 2) * sizeof(int32_t));
  if (!p->inc_ptr || !p->inc || !p->bptr || !p->blist || !p->in_ptr || !p->in_list || !p->os ||
      !fill || or_edge_maps(dim, n_nodes, el, n_elements, edges, os, n_edges, NULL, p->inc_ptr,
                            p->inc)) {
    free(fill);
    or_plan_free(p);
    return NULL;
  }
  memcpy(p->os, os, (size_t)(n_nodes + 1) * sizeof(uint64_t));
  for (int64_t b = 0; b < n_boundary; ++b)
    for (int t = 0; t < nbe; ++t) {
      const int32_t* bl = bnd + dim * b;
      int32_t id = or_edge_of(edges, os, n_nodes, bl[t], bl[(t + 1) % dim]);
      if (id < 0) {
        free(fill);
        or_plan_free(p);
        return NULL;
      }
      p->bptr[id + 1]++;
    }
  for (int64_t e = 0; e < n_edges; ++e) p->bptr[e + 1] += p->bptr[e];
  memcpy(fill, p->bptr, (size_t)(n_edges + 1) * sizeof(int32_t));
  for (int64_t b = 0; b < n_boundary; ++b)
    for (int t = 0; t < nbe; ++t) {
      const int32_t* bl = bnd + dim * b;
      int32_t id = or_edge_of(edges, os, n_nodes, bl[t], bl[(t + 1) % dim]);
      p->blist[fill[id]++] = (int32_t)b;
    }
  for (int64_t e = 0; e < n_edges; ++e) p->in_ptr[edges[2 * e + 1] + 1]++;
  for (int64_t v = 0; v < n_nodes; ++v) p->in_ptr[v + 1] += p->in_ptr[v];
  memcpy(fill, p->in_ptr, (size_t)(n_nodes + 1) * sizeof(int32_t));
  for (int64_t e = 0; e < n_edges; ++e) p->in_list[fill[edges[2 * e + 1]]++] = (int32_t)e;
  free(fill);
  return p;
}

void or_plan_free(or_plan* p) {
  if (!p) return;
  free(p->inc_ptr);
  free(p->inc);
  free(p->bptr);
  free(p->blist);
  free(p->in_ptr);
  free(p->in_list);
  free(p->os);
  free(p);
}

typedef struct {
  const or_plan* p;
  const double* x;
  double *navs, *s, *V;
  int64_t lo, hi;
  int phase;
} mt_task;

static void mt_edges(const or_plan* p, const double* x, double* navs, double* sv, int64_t lo,
                     int64_t hi) {
  const int dim = p->dim, npe = dim + 1;
  const double fb = 1.0 / (double)(dim * (dim + 1));
  for (int64_t e = lo; e < hi; ++e) {
    const int32_t j = p->edges[2 * e], k = p->edges[2 * e + 1];
    double n[3] = {0.0, 0.0, 0.0};
    for (int32_t q = p->inc_ptr[e]; q < p->inc_ptr[e + 1]; ++q) {
      const int32_t* t = p->el + (int64_t)npe * p->inc[q];
      int ij = 0;
      while (t[ij] != j) ++ij;
      if (dim == 3) {
        const int* f = kOppFace[ij];
        const double *p0 = x + 3 * (int64_t)t[f[0]], *p1 = x + 3 * (int64_t)t[f[1]],
                     *p2 = x + 3 * (int64_t)t[f[2]];
        double d1[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
        double d2[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
        double c[3];
        cross3(d1, d2, c);
        n[0] += c[0];
        n[1] += c[1];
        n[2] += c[2];
      } else {
        double nj[3];
        or_opposite_face_normal(2, x, t, ij, nj);
        n[0] += (1.0 / 3.0) * nj[0];
        n[1] += (1.0 / 3.0) * nj[1];
      }
    }
    if (dim == 3) {
      n[0] *= (1.0 / 12.0);
      n[1] *= (1.0 / 12.0);
      n[2] *= (1.0 / 12.0);
    }
    for (int32_t q = p->bptr[e]; q < p->bptr[e + 1]; ++q) {
      double nb[3];
      or_boundary_normal(dim, x, p->bnd + (int64_t)dim * p->blist[q], nb);
      for (int d = 0; d < dim; ++d) n[d] += fb * nb[d];
    }
    for (int d = 0; d < dim; ++d) navs[(int64_t)dim * e + d] = n[d];
    const double *xj = x + (int64_t)dim * j, *xk = x + (int64_t)dim * k;
    double s = (xk[0] - xj[0]) * n[0] + (xk[1] - xj[1]) * n[1];
    if (dim == 3) s = s + (xk[2] - xj[2]) * n[2];
    sv[e] = s;
  }
}

static void mt_nodes(const or_plan* p, const double* sv, double* V, int64_t lo, int64_t hi) {
  const double f = 1.0 / (double)(2 * p->dim);
  for (int64_t v = lo; v < hi; ++v) {
    double acc = 0.0;
    for (int32_t q = p->in_ptr[v]; q < p->in_ptr[v + 1]; ++q) acc += sv[p->in_list[q]];
    for (uint64_t e = p->os[v]; e < p->os[v + 1]; ++e) acc += sv[e];
    V[v] = acc * f;
  }
}

static void* mt_run(void* arg) {
  mt_task* t = (mt_task*)arg;
  if (t->phase == 0) mt_edges(t->p, t->x, t->navs, t->s, t->lo, t->hi);
  else mt_nodes(t->p, t->s, t->V, t->lo, t->hi);
  return NULL;
}

int or_metrics_mt(const or_plan* p, const double* x, int nthreads, double* navs, double* s,
                  double* V) {
  if (!p || nthreads < 1) return -1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  mt_task tk[256];
  for (int phase = 0; phase < 2; ++phase) {
    const int64_t n = phase == 0 ? p->n_edges : p->n_nodes;
    for (int i = 0; i < nthreads; ++i) {
      tk[i] = (mt_task){p, x, navs, s, V, n * i / nthreads, n * (i + 1) / nthreads, phase};
      if (i > 0 && pthread_create(&th[i], NULL, mt_run, &tk[i])) return -2;
    }
    mt_run(&tk[0]);
    for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
  }
  return 0;
}

/* ---- input synthesis for the CPU legs ------------------ */
/* gen_tet_cube(n) + perturb_interior(amp, seed): the oracle's own generator,
 * so the bench's CPU arm never loads the product's meshgen library.  Node
 * (i,j,k) -> i + (n+1)j + (n+1)^2 k; each hex is cut into the 6 Kuhn tets
 * that share its v000-v111 diagonal (one per axis order), positively
 * oriented; each boundary quad into 2 triangles along its lowest-highest
 * corner diagonal, outward.  Jitter: splitmix64, three draws
 * per interior node in node order, d = (2u - 1) amp h, u = (r >> 11) 2^-53.
 * tests/test_oracle.py pins it against the product generator bit for bit. */
static uint64_t sm64(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static double sm64_jit(uint64_t* s, double amp, double h) {
  const double u = (double)(sm64(s) >> 11) * (1.0 / 9007199254740992.0);
  return (2.0 * u - 1.0) * amp * h;
}

int or_gen_tet_cube(int n, double amp, uint64_t seed, double* x, int32_t* el, int32_t* bnd) {
  if (n < 1 || !x || !el || !bnd) return -1;
  const int64_t w = n + 1, w2 = w * w;
  const double h = 1.0 / n;
  uint64_t st = seed;
  for (int64_t k = 0; k <= n; ++k)
    for (int64_t j = 0; j <= n; ++j)
      for (int64_t i = 0; i <= n; ++i) {
        double* p = x + 3 * (i + w * j + w2 * k);
        const int64_t ijk[3] = {i, j, k};
        for (int a = 0; a < 3; ++a) p[a] = ijk[a] == n ? 1.0 : (double)ijk[a] * h;
        if (amp != 0.0 && i > 0 && i < n && j > 0 && j < n && k > 0 && k < n)
          for (int a = 0; a < 3; ++a) p[a] += sm64_jit(&st, amp, h);
      }
  /* axis orders of the 6 Kuhn paths; the tet (v000, v000+e_a, v000+e_a+e_b,
   * v111) is positive when (a, b, c) is an even permutation, else its last
   * two nodes are swapped */
  static const int ord[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  static const int even[6] = {1, 0, 0, 1, 1, 0};
  const int64_t step[3] = {1, w, w2};
  int32_t* t = el;
  for (int64_t k = 0; k < n; ++k)
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) {
        const int64_t v0 = i + w * j + w2 * k, v7 = v0 + 1 + w + w2;
        for (int p = 0; p < 6; ++p) {
          const int64_t v1 = v0 + step[ord[p][0]], v2 = v1 + step[ord[p][1]];
          t[0] = (int32_t)v0;
          t[1] = (int32_t)v1;
          t[2] = (int32_t)(even[p] ? v2 : v7);
          t[3] = (int32_t)(even[p] ? v7 : v2);
          t += 4;
        }
      }
  /* boundary: for each axis, low side then high side; the quad's in-plane
   * axes u < v, corners c(du, dv); triangles (c00, c10, c11), (c00, c11, c01)
   * as seen with the outward normal along +axis, reversed on the low side */
  int32_t* b = bnd;
  for (int ax = 0; ax < 3; ++ax) {
    const int u = ax == 0 ? 1 : 0, v = ax == 2 ? 1 : 2;
    /* (e_u x e_v) . e_ax > 0 for ax = 0, 2 and < 0 for ax = 1 */
    const int uv_out = ax != 1;
    for (int side = 0; side < 2; ++side) {
      const int flip = (side == 1) != uv_out; /* reverse (c10 <-> c11 order) */
      const int64_t base = side ? (int64_t)n * step[ax] : 0;
      for (int64_t qv = 0; qv < n; ++qv)
        for (int64_t qu = 0; qu < n; ++qu) {
          const int64_t c00 = base + qu * step[u] + qv * step[v];
          const int64_t c10 = c00 + step[u], c01 = c00 + step[v], c11 = c10 + step[v];
          const int64_t tri[2][3] = {{c00, c10, c11}, {c00, c11, c01}};
          for (int q = 0; q < 2; ++q) {
            b[0] = (int32_t)tri[q][0];
            b[1] = (int32_t)(flip ? tri[q][2] : tri[q][1]);
            b[2] = (int32_t)(flip ? tri[q][1] : tri[q][2]);
            b += 3;
          }
        }
    }
  }
  return 0;
}
