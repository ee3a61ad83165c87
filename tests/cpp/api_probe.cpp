// api_probe.cpp -- TEST INFRASTRUCTURE: extern "C" wrappers that call the
// C++ drop-in API (include/dualmesh/*.hpp, implemented by libdualmesh.so) so
// the Python tests can compare it with the reference's own mesh.cpp
// (oracle/_ref).  Built by the top-level Makefile into build/libapi_probe.so.
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "dualmesh/mesh.hpp"
#include "dualmesh/io.hpp"
#include "dualmesh/metrics.hpp"

namespace {
dualmesh::Mesh make(int dim, const double* x, int64_t nv, const int32_t* el, int64_t ne,
                    const int32_t* b, int64_t nb) {
  dualmesh::Mesh m;
  m.dim = dim;
  m.coords.assign(x, x + dim * nv);
  m.elements.assign(el, el + (dim + 1) * ne);
  if (nb) m.boundary.assign(b, b + dim * nb);
  return m;
}
}  // namespace

extern "C" {

// Returns the number of violations (or -1 on exception, message in buf).
int64_t probe_validate(int dim, const double* x, int64_t nv, const int32_t* el, int64_t ne,
                       const int32_t* b, int64_t nb, char* buf, int64_t cap, int8_t* signs) {
  try {
    auto out = dualmesh::validate_mesh(make(dim, x, nv, el, ne, b, nb));
    std::string j;
    for (const auto& v : out.violations) j += v + "\n";
    std::strncpy(buf, j.c_str(), static_cast<size_t>(cap - 1));
    buf[cap - 1] = '\0';
    if (signs)
      for (size_t e = 0; e < out.volume_signs.size(); ++e) signs[e] = out.volume_signs[e];
    return static_cast<int64_t>(out.violations.size());
  } catch (const std::exception& ex) {
    std::strncpy(buf, ex.what(), static_cast<size_t>(cap - 1));
    buf[cap - 1] = '\0';
    return -1;
  }
}

int64_t probe_derive(int dim, const double* x, int64_t nv, const int32_t* el, int64_t ne,
                     int32_t* out, int64_t cap) {
  auto f = dualmesh::derive_boundary_faces(make(dim, x, nv, el, ne, nullptr, 0));
  for (size_t i = 0; i < f.size() && static_cast<int64_t>(i) < cap; ++i) out[i] = f[i];
  return static_cast<int64_t>(f.size());
}

int64_t probe_build_edges(int dim, const double* x, int64_t nv, const int32_t* el, int64_t ne,
                          int32_t* edges, uint64_t* os, int64_t cap) {
  auto l = dualmesh::build_edges(make(dim, x, nv, el, ne, nullptr, 0));
  for (size_t i = 0; i < l.size() && static_cast<int64_t>(i) < cap; ++i) {
    edges[2 * i] = l.edges[i][0];
    edges[2 * i + 1] = l.edges[i][1];
  }
  for (size_t v = 0; v < l.origin_start.size(); ++v) os[v] = l.origin_start[v];
  return static_cast<int64_t>(l.size());
}

// compute_metrics + the checks; returns 0, or -1 / -2 on invalid_argument / runtime_error.
int probe_compute_metrics(int dim, const double* x, int64_t nv, const int32_t* el, int64_t ne,
                          const int32_t* b, int64_t nb, int nav_algo, int vol_algo, double* navs,
                          double* vols, double* closure, double* total_rel) {
  try {
    auto m = make(dim, x, nv, el, ne, b, nb);
    auto r = dualmesh::compute_metrics(m, static_cast<dualmesh::NavAlgo>(nav_algo),
                                       static_cast<dualmesh::VolAlgo>(vol_algo));
    std::memcpy(navs, r.navs.navs.data(), r.navs.navs.size() * sizeof(double));
    std::memcpy(vols, r.volumes.volumes.data(), r.volumes.volumes.size() * sizeof(double));
    *closure = dualmesh::check_closure(m, r.edges, r.navs);
    *total_rel = dualmesh::check_total_volume(m, r.volumes);
    // the stand-alone SPEC ops must agree with the facade
    auto n2 = dualmesh::lumped_navs_dualfree(m, r.edges);
    auto v2 = dualmesh::dual_volumes_edge_based(m, r.edges, n2);
    if (nav_algo == 1 && vol_algo == 0 &&
        (n2.navs != r.navs.navs || v2.volumes != r.volumes.volumes))
      return -3;
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  } catch (const std::exception&) {
    return -2;
  }
}

// SPEC.md:265-274 through the C++ API: dual-free navs + edge volumes, then
// check_linear_exactness with A (row-major) and b; -1 on invalid_argument.
int probe_linear_exactness(int dim, const double* x, int64_t nv, const int32_t* el, int64_t ne,
                           const int32_t* b, int64_t nb, const double* A, const double* f,
                           double* residual) {
  try {
    auto m = make(dim, x, nv, el, ne, b, nb);
    auto r = dualmesh::compute_metrics(m, dualmesh::NavAlgo::dualfree, dualmesh::VolAlgo::edge);
    std::vector<double> AA(A, A + dim * dim), ff(f, f + dim);
    *residual = dualmesh::check_linear_exactness(m, r.edges, r.navs, r.volumes, AA, ff);
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  } catch (const std::exception&) {
    return -2;
  }
}

// dualmesh::read_mesh -> write_mesh, and compute_metrics -> write_metrics, through
// the C++ API (io.hpp).  Returns the boundary count read (derived when the file
// has no boundary section), -1 on a parse error, -2 on other errors.
int64_t probe_io(const char* in_path, const char* mesh_out, const char* metrics_out) {
  try {
    auto m = dualmesh::read_mesh(in_path);
    dualmesh::write_mesh(m, mesh_out);
    auto r = dualmesh::compute_metrics(m, dualmesh::NavAlgo::dualfree, dualmesh::VolAlgo::edge);
    dualmesh::write_metrics(metrics_out, m, r.edges, r.navs, r.volumes,
                            dualmesh::NavAlgo::dualfree, dualmesh::VolAlgo::edge);
    return static_cast<int64_t>(m.num_boundary());
  } catch (const std::runtime_error&) {
    return -1;
  } catch (const std::exception&) {
    return -2;
  }
}

// mesh/edge mismatch must raise std::invalid_argument.
// A foreign EdgeList must throw std::invalid_argument ("mesh/edge mismatch"),
// whether it differs in size or, with the same size, in one entry (the
// topology and its own list resident, so only the content check can see it).
int probe_mismatch(int dim, const double* x, int64_t nv, const int32_t* el, int64_t ne) {
  auto m = make(dim, x, nv, el, ne, nullptr, 0);
  auto l = dualmesh::build_edges(m);
  (void)dualmesh::lumped_navs_dualfree(m, l);  // the genuine list is accepted
  auto shorter = l;
  shorter.edges.pop_back();
  auto altered = l;
  altered.edges[altered.size() / 2][1] = altered.edges[altered.size() / 2][1] + 1;
  int thrown = 0;
  for (const auto* bad : {&shorter, &altered}) {
    try {
      dualmesh::lumped_navs_dualfree(m, *bad);
    } catch (const std::invalid_argument&) {
      ++thrown;
      continue;
    } catch (...) {
      return 2;
    }
  }
  return thrown == 2 ? 1 : 0;
}

double probe_element_volume(int dim, const double* x, int64_t nv, const int32_t* el, int64_t ne,
                            int64_t e) {
  return dualmesh::element_volume(make(dim, x, nv, el, ne, nullptr, 0), static_cast<size_t>(e));
}

}  // extern "C"
