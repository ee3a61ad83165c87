// ref_shim.cpp -- extern "C" handle API over the reference's own mesh module.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// UNMODIFIED reference source /root/reference/proj/src/mesh.cpp (read in
// place, never copied) into oracle/_ref/libref_mesh.so.  It lets the tests
// and the bench's reference arm call the reference build_edges / edge_of /
// geometry / validate_mesh / derive_boundary_faces directly.  Include path
// must point at /root/reference/proj/include, not at this repo's include/.
#include <cstdlib>
#include <cstring>
#include <string>

#include "dualmesh/mesh.hpp"

namespace {
struct RefHandle {
  dualmesh::Mesh mesh;
  dualmesh::EdgeList edges;
};
}  // namespace

extern "C" {

void* ref_mesh_new(int dim, const double* coords, int64_t n_nodes, const int32_t* el,
                   int64_t n_elements, const int32_t* bnd, int64_t n_boundary) {
  auto* h = new RefHandle;
  h->mesh.dim = dim;
  h->mesh.coords.assign(coords, coords + dim * n_nodes);
  h->mesh.elements.assign(el, el + (dim + 1) * n_elements);
  if (bnd && n_boundary > 0) h->mesh.boundary.assign(bnd, bnd + dim * n_boundary);
  return h;
}

void ref_mesh_free(void* p) { delete static_cast<RefHandle*>(p); }

// ref build_edges, mesh.cpp:256-285.  Returns the edge count.
int64_t ref_build_edges(void* p) {
  auto* h = static_cast<RefHandle*>(p);
  h->edges = dualmesh::build_edges(h->mesh);
  return static_cast<int64_t>(h->edges.size());
}

void ref_get_edges(void* p, int32_t* edges, uint64_t* origin_start) {
  auto* h = static_cast<RefHandle*>(p);
  if (edges)
    for (std::size_t e = 0; e < h->edges.edges.size(); ++e) {
      edges[2 * e] = h->edges.edges[e][0];
      edges[2 * e + 1] = h->edges.edges[e][1];
    }
  if (origin_start)
    for (std::size_t v = 0; v < h->edges.origin_start.size(); ++v)
      origin_start[v] = h->edges.origin_start[v];
}

int32_t ref_edge_of(void* p, int32_t a, int32_t b) {
  return static_cast<RefHandle*>(p)->edges.edge_of(a, b);
}

double ref_element_volume(void* p, int64_t e) {
  return dualmesh::element_volume(static_cast<RefHandle*>(p)->mesh, static_cast<std::size_t>(e));
}

void ref_opposite_face_normal(void* p, int64_t e, int i, double* out) {
  auto v = dualmesh::opposite_face_normal(static_cast<RefHandle*>(p)->mesh,
                                          static_cast<std::size_t>(e), i);
  out[0] = v[0];
  out[1] = v[1];
  out[2] = v[2];
}

void ref_boundary_normal(void* p, int64_t b, double* out) {
  auto v = dualmesh::boundary_normal(static_cast<RefHandle*>(p)->mesh, static_cast<std::size_t>(b));
  out[0] = v[0];
  out[1] = v[1];
  out[2] = v[2];
}

// ref validate_mesh, mesh.cpp:129-254.  Writes the violations joined by
// '\n' into buf (truncated to cap) and the volume signs; returns the count.
int64_t ref_validate(void* p, char* buf, int64_t cap, int8_t* signs) {
  auto out = dualmesh::validate_mesh(static_cast<RefHandle*>(p)->mesh);
  std::string joined;
  for (const auto& v : out.violations) {
    joined += v;
    joined += '\n';
  }
  if (buf && cap > 0) {
    std::size_t n = joined.size() < static_cast<std::size_t>(cap - 1) ? joined.size()
                                                                       : static_cast<std::size_t>(cap - 1);
    std::memcpy(buf, joined.data(), n);
    buf[n] = '\0';
  }
  if (signs)
    for (std::size_t e = 0; e < out.volume_signs.size(); ++e) signs[e] = out.volume_signs[e];
  return static_cast<int64_t>(out.violations.size());
}

// ref derive_boundary_faces, mesh.cpp:287-323.  malloc'd; free with ref_free.
int64_t ref_derive_boundary(void* p, int32_t** faces) {
  auto f = dualmesh::derive_boundary_faces(static_cast<RefHandle*>(p)->mesh);
  *faces = static_cast<int32_t*>(std::malloc((f.size() + 1) * sizeof(int32_t)));
  std::memcpy(*faces, f.data(), f.size() * sizeof(int32_t));
  return static_cast<int64_t>(f.size());
}

void ref_free(void* q) { std::free(q); }

double ref_max_face_area(void* p) { return dualmesh::max_face_area(static_cast<RefHandle*>(p)->mesh); }
double ref_max_element_volume(void* p) {
  return dualmesh::max_element_volume(static_cast<RefHandle*>(p)->mesh);
}
double ref_total_volume(void* p) { return dualmesh::total_volume(static_cast<RefHandle*>(p)->mesh); }

void ref_boundary_node_mask(void* p, uint8_t* mask) {
  auto m = dualmesh::boundary_node_mask(static_cast<RefHandle*>(p)->mesh);
  for (std::size_t v = 0; v < m.size(); ++v) mask[v] = m[v] ? 1 : 0;
}

}  // extern "C"
