// host_api.cpp -- the reference C++ API (include/dualmesh/mesh.hpp, ref
// proj/include/dualmesh/mesh.hpp) and the SPEC metrics API
// (include/dualmesh/metrics.hpp) implemented over the C-ABI.
//
// Each host thread owns one dm_ctx (C-ABI threading rule).  The functions
// are pure functions of their arguments, like the reference: every call
// takes the mesh it is given -- uploading it in full when its connectivity
// differs from the resident one, only its coordinates otherwise (the edge
// list, plan and derived CSRs stay on the device).  Status codes become
// exceptions here and only here: DM_ERR_INVALID_ARG / MESH_EDGE_MISMATCH /
// EDGE_ABSENT -> std::invalid_argument, everything else -> std::runtime_error.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <sys/mman.h>
#include <initializer_list>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "dm_capi.h"
#include "dualmesh/mesh.hpp"
#include "dualmesh/metrics.hpp"

namespace dualmesh {
namespace {

// Per-thread context plus the topology it holds.  The functions are pure
// functions of their arguments, like the reference, but consecutive calls on
// one mesh (time stepping, a deforming grid, verify after metrics) share its
// topology: a call whose connectivity fingerprint (dim, sizes, elements,
// boundary) matches the resident one only refreshes the coordinates, keeping
// the edge list, the ring plan and the derived CSRs on the device.  The
// fingerprint is a full hash of the arrays (multi-threaded, ~10 ms for C5's
// 1.6 GB), so a changed element is always seen.
struct Topology {
  bool valid = false;
  int dim = 0;
  std::size_t nv = 0, nE = 0, nB = 0;
  std::uint64_t fp = 0;
  bool edges_built = false;
  std::uint64_t fp_edges = 0;  // fingerprint of an EdgeList verified equal to the device's
};

struct ThreadCtx {
  dm_ctx* c = nullptr;
  Topology topo;
  ~ThreadCtx() { dm_destroy(c); }
};

ThreadCtx& tctx() {
  thread_local ThreadCtx t;
  return t;
}

void check(dm_ctx* c, int st, const char* what) {
  if (st == DM_OK) return;
  std::string msg = std::string(what) + ": " + dm_status_string(st) + " (" + dm_last_error(c) + ")";
  if (st == DM_ERR_INVALID_ARG || st == DM_ERR_MESH_EDGE_MISMATCH || st == DM_ERR_EDGE_ABSENT)
    throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

dm_ctx* ctx() {
  ThreadCtx& t = tctx();
  if (!t.c) {
    const char* dev = std::getenv("DUALMESH_DEVICE");
    int st = dm_create(&t.c, dev ? std::atoi(dev) : 0);
    if (st != DM_OK) {
      std::string msg = std::string("dualmesh: no usable sm_100a device: ") + dm_last_error(t.c);
      dm_destroy(t.c);
      t.c = nullptr;
      throw std::runtime_error(msg);
    }
  }
  return t.c;
}

// env DUALMESH_API_TRACE=1: wall time of each phase of a call on stderr
struct ApiTrace {
  bool on;
  std::chrono::steady_clock::time_point t;
  ApiTrace() {
    const char* e = std::getenv("DUALMESH_API_TRACE");
    on = e && e[0] == '1';
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[api] %-28s %9.2f ms\n", what,
                 std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};

// Sizes a result vector for n elements with its pages faulted in by all
// cores first (transparent huge pages requested): resize() alone would fault
// and zero ~3 GB of navs at C5 page by page on one thread (about 1 s).
template <typename T>
void sized(std::vector<T>& v, std::size_t n) {
  v.clear();
  v.reserve(n);
  const std::size_t bytes = n * sizeof(T);
  if (bytes >= (std::size_t(64) << 20)) {
    auto* p = reinterpret_cast<unsigned char*>(v.data());
    const std::size_t page = 4096;
    const auto a = reinterpret_cast<std::uintptr_t>(p);
    const std::uintptr_t lo = (a + (std::size_t(2) << 20) - 1) & ~((std::size_t(2) << 20) - 1);
    if (lo < a + bytes) madvise(reinterpret_cast<void*>(lo), a + bytes - lo, MADV_HUGEPAGE);
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const std::size_t nt = std::min<std::size_t>(16, hw);
    std::vector<std::thread> th;
    for (std::size_t i = 0; i < nt; ++i)
      th.emplace_back([=] {
        const std::size_t b0 = bytes * i / nt, b1 = bytes * (i + 1) / nt;
        for (std::size_t o = b0 & ~(page - 1); o < b1; o += page)
          reinterpret_cast<volatile unsigned char*>(p)[o] = 0;
      });
    for (auto& t : th) t.join();
  }
  v.resize(n);
}

// 64-bit fingerprint of byte ranges: per-slice multiply-xorshift chains over
// 8-byte words on up to 16 threads, combined in slice order.
std::uint64_t fingerprint(std::initializer_list<std::pair<const void*, std::size_t>> parts) {
  std::uint64_t h = 0x9E3779B97F4A7C15ull;
  for (const auto& [ptr, bytes] : parts) {
    const auto* p = static_cast<const unsigned char*>(ptr);
    const std::size_t nw = bytes / 8;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const std::size_t nt = bytes < (std::size_t(8) << 20) ? 1 : std::min<std::size_t>(16, hw);
    std::vector<std::uint64_t> part(nt, 0);
    auto run = [&](std::size_t i) {
      const std::size_t a = nw * i / nt, b = nw * (i + 1) / nt;
      std::uint64_t x = 0xD6E8FEB86659FD93ull ^ i;
      for (std::size_t w = a; w < b; ++w) {
        std::uint64_t v;
        std::memcpy(&v, p + 8 * w, 8);
        x = (x ^ v) * 0x9E3779B97F4A7C15ull;
        x ^= x >> 29;
      }
      part[i] = x;
    };
    std::vector<std::thread> th;
    for (std::size_t i = 1; i < nt; ++i) th.emplace_back(run, i);
    run(0);
    for (auto& t : th) t.join();
    for (std::size_t i = 0; i < nt; ++i) h = (h ^ part[i]) * 0xC2B2AE3D27D4EB4Full;
    std::uint64_t tail = bytes;
    for (std::size_t k = 8 * nw; k < bytes; ++k) tail = tail * 131 + p[k];
    h = (h ^ tail) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 31;
  }
  return h;
}

dm_ctx* upload(const Mesh& m) {
  dm_ctx* c = ctx();
  if (m.dim != 2 && m.dim != 3) throw std::invalid_argument("dim must be 2 or 3");
  Topology& T = tctx().topo;
  ApiTrace tr;
  const std::size_t nv = m.num_nodes(), nE = m.num_elements(), nB = m.num_boundary();
  const std::uint64_t fp =
      fingerprint({{&m.dim, sizeof(m.dim)},
                   {m.elements.data(), m.elements.size() * sizeof(Index)},
                   {m.boundary.data(), m.boundary.size() * sizeof(Index)}});
  tr.mark("upload: fingerprint");
  if (T.valid && T.dim == m.dim && T.nv == nv && T.nE == nE && T.nB == nB && T.fp == fp) {
    check(c, dm_set_coords(c, m.coords.data()), "dm_set_coords");  // same topology
    tr.mark("upload: coordinates");
    return c;
  }
  T.valid = false;
  check(c,
        dm_set_mesh(c, m.dim, m.coords.data(), static_cast<int64_t>(nv), m.elements.data(),
                    static_cast<int64_t>(nE), m.boundary.data(), static_cast<int64_t>(nB)),
        "dm_set_mesh");
  T = Topology{true, m.dim, nv, nE, nB, fp, false, 0};
  tr.mark("upload: mesh");
  return c;
}

// The resident topology's edge list (built once per topology).
int64_t ensure_edges(dm_ctx* c) {
  Topology& T = tctx().topo;
  int64_t ne = 0;
  if (!T.edges_built) {
    check(c, dm_build_edges(c, &ne), "dm_build_edges");
    T.edges_built = true;
    T.fp_edges = 0;
  } else {
    dm_device_view v;
    check(c, dm_device_views(c, &v), "dm_device_views");
    ne = v.n_edges;
  }
  return ne;
}

std::uint64_t edgelist_fp(const EdgeList& l) {
  return fingerprint({{l.edges.data(), l.edges.size() * sizeof(l.edges[0])},
                      {l.origin_start.data(), l.origin_start.size() * sizeof(std::size_t)}});
}

// Upload (or refresh) + the resident edge list, then confirm the caller's
// EdgeList is the one this mesh produces ("mesh/edge
// mismatch"): compared element by element the first time a list is seen for
// this topology, by fingerprint afterwards.
dm_ctx* upload_with_edges(const Mesh& m, const EdgeList& given) {
  dm_ctx* c = upload(m);
  const int64_t ne = ensure_edges(c);
  if (static_cast<std::size_t>(ne) != given.size() ||
      given.origin_start.size() != m.num_nodes() + 1)
    throw std::invalid_argument("mesh/edge mismatch");
  Topology& T = tctx().topo;
  const std::uint64_t fp = edgelist_fp(given);
  if (T.fp_edges != 0 && fp == T.fp_edges) return c;
  std::vector<int32_t> e(2 * static_cast<std::size_t>(ne));
  std::vector<uint64_t> os(m.num_nodes() + 1);
  check(c, dm_get_edges(c, e.data(), os.data()), "dm_get_edges");
  for (std::size_t i = 0; i < given.size(); ++i)
    if (e[2 * i] != given.edges[i][0] || e[2 * i + 1] != given.edges[i][1])
      throw std::invalid_argument("mesh/edge mismatch");
  for (std::size_t v = 0; v < os.size(); ++v)
    if (os[v] != given.origin_start[v]) throw std::invalid_argument("mesh/edge mismatch");
  T.fp_edges = fp;
  return c;
}

const int kOpp[4][3] = {{1, 2, 3}, {0, 3, 2}, {0, 1, 3}, {0, 2, 1}};  // ref mesh.cpp:15

Vec cross(const double* u, const double* v) {
  return {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
}

}  // namespace

// ---------------------------------------------------------------- mesh.hpp
Index EdgeList::edge_of(Index a, Index b) const {
  // Host lookup on the host-resident list (same contract as ref
  // mesh.cpp:58-73); batched device lookups go through dm_edge_of.
  if (a > b) std::swap(a, b);
  if (a < 0 || static_cast<std::size_t>(a) + 1 >= origin_start.size()) return -1;
  std::size_t lo = origin_start[static_cast<std::size_t>(a)];
  const std::size_t end = origin_start[static_cast<std::size_t>(a) + 1];
  std::size_t hi = end;
  while (lo < hi) {
    const std::size_t mid = lo + (hi - lo) / 2;
    if (edges[mid][1] < b) lo = mid + 1;
    else hi = mid;
  }
  return (lo < end && edges[lo][1] == b) ? static_cast<Index>(lo) : -1;
}

EdgeList build_edges(const Mesh& mesh) {
  dm_ctx* c = upload(mesh);
  ApiTrace tr;
  const int64_t ne = ensure_edges(c);
  tr.mark("build_edges: K1");
  EdgeList out;
  sized(out.edges, static_cast<std::size_t>(ne));
  sized(out.origin_start, mesh.num_nodes() + 1);
  tr.mark("build_edges: allocate");
  static_assert(sizeof(std::size_t) == sizeof(uint64_t), "origin_start is 64-bit");
  check(c, dm_get_edges(c, reinterpret_cast<int32_t*>(out.edges.data()),
                        reinterpret_cast<uint64_t*>(out.origin_start.data())),
        "dm_get_edges");
  tr.mark("build_edges: copy out");
  tctx().topo.fp_edges = edgelist_fp(out);  // this exact list needs no re-verification
  tr.mark("build_edges: fingerprint");
  return out;
}

double element_volume(const Mesh& mesh, std::size_t e) {
  const Index* el = mesh.element(e);
  if (mesh.dim == 2) {
    const double *a = mesh.node(el[0]), *b = mesh.node(el[1]), *c = mesh.node(el[2]);
    return 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]));
  }
  const double *a = mesh.node(el[0]), *b = mesh.node(el[1]), *c = mesh.node(el[2]),
               *d = mesh.node(el[3]);
  const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
  const double v[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
  const Vec uv = cross(u, v);
  return (uv[0] * (d[0] - a[0]) + uv[1] * (d[1] - a[1]) + uv[2] * (d[2] - a[2])) / 6.0;
}

Vec opposite_face_normal(const Mesh& mesh, std::size_t e, int i) {
  const Index* el = mesh.element(e);
  if (mesh.dim == 2) {
    const double *p = mesh.node(el[(i + 1) % 3]), *q = mesh.node(el[(i + 2) % 3]);
    return {q[1] - p[1], p[0] - q[0], 0.0};
  }
  const double *p0 = mesh.node(el[kOpp[i][0]]), *p1 = mesh.node(el[kOpp[i][1]]),
               *p2 = mesh.node(el[kOpp[i][2]]);
  const double d1[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
  const double d2[3] = {p2[0] - p0[0], p2[1] - p0[1], p2[2] - p0[2]};
  const Vec c = cross(d1, d2);
  return {0.5 * c[0], 0.5 * c[1], 0.5 * c[2]};
}

Vec boundary_normal(const Mesh& mesh, std::size_t b) {
  const Index* bl = mesh.boundary_element(b);
  if (mesh.dim == 2) {
    const double *j = mesh.node(bl[0]), *k = mesh.node(bl[1]);
    return {k[1] - j[1], j[0] - k[0], 0.0};
  }
  const double *j = mesh.node(bl[0]), *r = mesh.node(bl[1]), *l = mesh.node(bl[2]);
  const double d1[3] = {r[0] - j[0], r[1] - j[1], r[2] - j[2]};
  const double d2[3] = {l[0] - j[0], l[1] - j[1], l[2] - j[2]};
  const Vec c = cross(d1, d2);
  return {0.5 * c[0], 0.5 * c[1], 0.5 * c[2]};
}

ValidationOutcome validate_mesh(const Mesh& mesh) {
  ValidationOutcome out;
  if (mesh.dim != 2 && mesh.dim != 3) {
    out.violations.push_back("dim must be 2 or 3, got " + std::to_string(mesh.dim));
    return out;
  }
  if (mesh.coords.size() % static_cast<std::size_t>(mesh.dim) != 0)
    out.violations.push_back("coordinate array length is not a multiple of dim");
  if (mesh.elements.size() % static_cast<std::size_t>(mesh.dim + 1) != 0)
    out.violations.push_back("element array length is not a multiple of dim+1");
  if (mesh.boundary.size() % static_cast<std::size_t>(mesh.dim) != 0)
    out.violations.push_back("boundary array length is not a multiple of dim");
  if (!out.violations.empty()) return out;
  dm_ctx* c = upload(mesh);
  std::vector<int8_t> signs(mesh.num_elements());
  int64_t counts[DM_VCOUNT] = {0};
  int64_t exposed = 0;
  check(c, dm_validate(c, signs.data(), counts, &exposed), "dm_validate");
  auto ids = [&](int kind) {
    std::vector<int64_t> v(static_cast<std::size_t>(counts[kind]));
    int64_t n = 0;
    if (!v.empty()) check(c, dm_validate_list(c, kind, v.data(), counts[kind], &n), "dm_validate_list");
    return v;
  };
  const bool range_bad = counts[DM_V_OUT_OF_RANGE_ELEM] + counts[DM_V_OUT_OF_RANGE_BND] > 0;
  for (int64_t e : ids(DM_V_OUT_OF_RANGE_ELEM))
    out.violations.push_back("out-of-range node index in element " + std::to_string(e + 1));
  for (int64_t b : ids(DM_V_OUT_OF_RANGE_BND))
    out.violations.push_back("out-of-range node index in boundary element " + std::to_string(b + 1));
  if (range_bad) return out;
  out.volume_signs.assign(signs.begin(), signs.end());
  for (int64_t e : ids(DM_V_NONPOSITIVE))
    out.violations.push_back("nonpositive volume, element " + std::to_string(e + 1));
  for (int64_t f : ids(DM_V_FACE_OVERSHARED))  // f = element * (dim+1) + local face
    out.violations.push_back("face shared by more than two elements, element " +
                             std::to_string(f / (mesh.dim + 1) + 1));
  // Boundary classes are reported in facet order, interleaved as in the
  // reference loop: merge the per-class lists (payload: b << 32 | aux).
  std::vector<std::pair<int64_t, std::string>> bmsgs;
  for (int64_t q : ids(DM_V_BND_NOT_FACE))
    bmsgs.push_back({q >> 32, "boundary element " + std::to_string((q >> 32) + 1) +
                                  " is not a face of any element"});
  for (int64_t q : ids(DM_V_BND_INTERIOR))
    bmsgs.push_back({q >> 32, "boundary element " + std::to_string((q >> 32) + 1) +
                                  " matches an interior face of element " +
                                  std::to_string((q & 0xffffffff) + 1)});
  for (int64_t q : ids(DM_V_BND_DUPLICATE))
    bmsgs.push_back({q >> 32, "duplicate boundary element " + std::to_string((q >> 32) + 1)});
  for (int64_t q : ids(DM_V_BND_INWARD))
    bmsgs.push_back({q >> 32, "boundary element " + std::to_string((q >> 32) + 1) +
                                  " has inward orientation (element " +
                                  std::to_string((q & 0xffffffff) + 1) + ")"});
  std::stable_sort(bmsgs.begin(), bmsgs.end(),
                   [](const auto& x, const auto& y) { return x.first < y.first; });
  for (auto& m : bmsgs) out.violations.push_back(std::move(m.second));
  if (exposed > 0)
    out.violations.push_back(std::to_string(exposed) +
                             " mesh-boundary face(s) missing from the boundary list");
  return out;
}

std::vector<Index> derive_boundary_faces(const Mesh& mesh) {
  dm_ctx* c = upload(mesh);
  int64_t n = 0;
  check(c, dm_derive_boundary(c, &n), "dm_derive_boundary");
  std::vector<Index> out(static_cast<std::size_t>(n) * static_cast<std::size_t>(mesh.dim));
  if (n) check(c, dm_get_derived_boundary(c, out.data()), "dm_get_derived_boundary");
  return out;
}

double max_face_area(const Mesh& mesh) {
  double v = 0.0;
  dm_ctx* c = upload(mesh);
  check(c, dm_max_face_area(c, &v), "dm_max_face_area");
  return v;
}

double max_element_volume(const Mesh& mesh) {
  double v = 0.0;
  dm_ctx* c = upload(mesh);
  check(c, dm_max_element_volume(c, &v), "dm_max_element_volume");
  return v;
}

double total_volume(const Mesh& mesh) {
  double v = 0.0;
  dm_ctx* c = upload(mesh);
  check(c, dm_total_volume(c, &v), "dm_total_volume");
  return v;
}

std::vector<bool> boundary_node_mask(const Mesh& mesh) {
  dm_ctx* c = upload(mesh);
  std::vector<uint8_t> m(mesh.num_nodes());
  check(c, dm_boundary_node_mask(c, m.data()), "dm_boundary_node_mask");
  return std::vector<bool>(m.begin(), m.end());
}

// ---------------------------------------------------------------- metrics.hpp
namespace {
LumpedNavField fetch_navs(dm_ctx* c, const Mesh& mesh, std::size_t ne) {
  ApiTrace tr;
  LumpedNavField f;
  f.dim = mesh.dim;
  sized(f.navs, ne * static_cast<std::size_t>(mesh.dim));
  tr.mark("navs: allocate");
  check(c, dm_get_navs(c, f.navs.data()), "dm_get_navs");
  tr.mark("navs: compute + copy out");
  return f;
}
DualVolumeField fetch_vols(dm_ctx* c, const Mesh& mesh) {
  ApiTrace tr;
  DualVolumeField v;
  sized(v.volumes, mesh.num_nodes());
  check(c, dm_get_volumes(c, v.volumes.data()), "dm_get_volumes");
  tr.mark("volumes: allocate + copy out");
  return v;
}
void put_navs(dm_ctx* c, const Mesh& mesh, const EdgeList& edges, const LumpedNavField& navs) {
  if (navs.dim != mesh.dim || navs.size() != edges.size())
    throw std::invalid_argument("field/edge-list mismatch");
  check(c, dm_put_navs(c, navs.navs.data()), "dm_put_navs");
}
}  // namespace

LumpedNavField lumped_navs_traditional(const Mesh& mesh, const EdgeList& edges) {
  dm_ctx* c = upload_with_edges(mesh, edges);
  check(c, dm_navs(c, DM_NAV_TRADITIONAL, DM_VARIANT_GATHER), "dm_navs");
  return fetch_navs(c, mesh, edges.size());
}

LumpedNavField lumped_navs_dualfree(const Mesh& mesh, const EdgeList& edges) {
  dm_ctx* c = upload_with_edges(mesh, edges);
  check(c, dm_navs(c, DM_NAV_DUALFREE, DM_VARIANT_GATHER), "dm_navs");
  return fetch_navs(c, mesh, edges.size());
}

DualVolumeField dual_volumes_edge_based(const Mesh& mesh, const EdgeList& edges,
                                        const LumpedNavField& navs) {
  dm_ctx* c = upload_with_edges(mesh, edges);
  put_navs(c, mesh, edges, navs);
  check(c, dm_volumes(c, DM_VOL_EDGE), "dm_volumes");
  return fetch_vols(c, mesh);
}

DualVolumeField dual_volumes_element_based(const Mesh& mesh) {
  dm_ctx* c = upload(mesh);
  check(c, dm_volumes(c, DM_VOL_ELEMENT), "dm_volumes");
  return fetch_vols(c, mesh);
}

// The three result vectors of compute_metrics are sized concurrently: most of
// a repeated call is std::vector value-initialisation (a single-threaded
// memset per vector, ~250 ms for C5's 2.8 GB of navs), which the returned-
// by-value API types require.  The kernels run meanwhile (asynchronous on
// the context stream); the copies follow once each vector exists.
MetricsResult compute_metrics(const Mesh& mesh, NavAlgo nav_algo, VolAlgo vol_algo) {
  MetricsResult r;
  dm_ctx* c = upload(mesh);
  ApiTrace tr;
  const int64_t ne = ensure_edges(c);
  tr.mark("compute_metrics: K1");
  check(c, dm_navs(c, static_cast<int>(nav_algo), DM_VARIANT_GATHER), "dm_navs");
  check(c, dm_volumes(c, static_cast<int>(vol_algo)), "dm_volumes");
  tr.mark("compute_metrics: kernels queued");
  const std::size_t D = static_cast<std::size_t>(mesh.dim), nv = mesh.num_nodes();
  r.navs.dim = mesh.dim;
  std::exception_ptr err[2];
  std::thread tn([&] {
    try {
      sized(r.navs.navs, static_cast<std::size_t>(ne) * D);
    } catch (...) {
      err[0] = std::current_exception();
    }
  });
  std::thread tv([&] {
    try {
      sized(r.volumes.volumes, nv);
      sized(r.edges.origin_start, nv + 1);
    } catch (...) {
      err[1] = std::current_exception();
    }
  });
  try {
    sized(r.edges.edges, static_cast<std::size_t>(ne));
  } catch (...) {
    tn.join();
    tv.join();
    throw;
  }
  tv.join();
  if (err[1]) {
    tn.join();
    std::rethrow_exception(err[1]);
  }
  tr.mark("compute_metrics: edge vectors");
  check(c, dm_get_edges(c, reinterpret_cast<int32_t*>(r.edges.edges.data()),
                        reinterpret_cast<uint64_t*>(r.edges.origin_start.data())),
        "dm_get_edges");
  tctx().topo.fp_edges = edgelist_fp(r.edges);  // this exact list needs no re-verification
  tr.mark("compute_metrics: edges out");
  tn.join();
  if (err[0]) std::rethrow_exception(err[0]);
  tr.mark("compute_metrics: navs vector");
  check(c, dm_get_navs(c, r.navs.navs.data()), "dm_get_navs");
  check(c, dm_get_volumes(c, r.volumes.volumes.data()), "dm_get_volumes");
  tr.mark("compute_metrics: navs + volumes out");
  return r;
}

double check_closure(const Mesh& mesh, const EdgeList& edges, const LumpedNavField& navs) {
  dm_ctx* c = upload_with_edges(mesh, edges);
  put_navs(c, mesh, edges, navs);
  double r = 0.0, ri = 0.0;
  check(c, dm_check_closure(c, &r, &ri), "dm_check_closure");
  return r;
}

double check_linear_exactness(const Mesh& mesh, const EdgeList& edges,
                              const LumpedNavField& navs, const DualVolumeField& volumes,
                              const std::vector<double>& A, const std::vector<double>& b) {
  const size_t D = static_cast<size_t>(mesh.dim);
  if (A.size() != D * D || b.size() != D) throw std::invalid_argument("flux/mesh mismatch");
  if (volumes.size() != mesh.num_nodes()) throw std::invalid_argument("field/mesh mismatch");
  dm_ctx* c = upload_with_edges(mesh, edges);
  put_navs(c, mesh, edges, navs);
  check(c, dm_put_volumes(c, volumes.volumes.data()), "dm_put_volumes");
  double r = 0.0;
  check(c, dm_check_linear_exactness(c, A.data(), b.data(), &r), "dm_check_linear_exactness");
  return r;
}

double check_total_volume(const Mesh& mesh, const DualVolumeField& volumes) {
  if (volumes.size() != mesh.num_nodes()) throw std::invalid_argument("field/mesh mismatch");
  dm_ctx* c = upload(mesh);
  check(c, dm_put_volumes(c, volumes.volumes.data()), "dm_put_volumes");
  double rel = 0.0;
  check(c, dm_check_total_volume(c, &rel, nullptr, nullptr), "dm_check_total_volume");
  return rel;
}

}  // namespace dualmesh
