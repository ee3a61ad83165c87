// dualmesh/metrics.hpp -- the SPEC "metrics" and "verify" modules as a C++
// API beside the reference mesh module.
//
// The reference ships no code for these operations; their contract is
// SPEC.md:127-227 (metrics) and SPEC.md:229-306 (verify).  Every function is
// computed on the GPU through include/dm_capi.h; none has a CPU fallback.
#ifndef DUALMESH_METRICS_HPP
#define DUALMESH_METRICS_HPP

#include <cstddef>
#include <vector>

#include "dualmesh/mesh.hpp"

namespace dualmesh {

// one D-vector per edge in EdgeList order, stored flat
// (dim doubles per edge, like Mesh::coords).
struct LumpedNavField {
  int dim = 2;
  std::vector<double> navs;
  std::size_t size() const { return navs.size() / static_cast<std::size_t>(dim); }
  const double* nav(std::size_t e) const { return navs.data() + static_cast<std::size_t>(dim) * e; }
};

// one positive scalar per node.
struct DualVolumeField {
  std::vector<double> volumes;
  std::size_t size() const { return volumes.size(); }
};

enum class NavAlgo { traditional = 0, dualfree = 1 };
enum class VolAlgo { edge = 0, element = 1 };

// median-dual faces per element edge.
LumpedNavField lumped_navs_traditional(const Mesh& mesh, const EdgeList& edges);

// dual-free three-pass form.
LumpedNavField lumped_navs_dualfree(const Mesh& mesh, const EdgeList& edges);

// SPEC.md:170-178.
DualVolumeField dual_volumes_edge_based(const Mesh& mesh, const EdgeList& edges,
                                        const LumpedNavField& navs);

// SPEC.md:180-188.
DualVolumeField dual_volumes_element_based(const Mesh& mesh);

struct MetricsResult {
  EdgeList edges;
  LumpedNavField navs;
  DualVolumeField volumes;
};

// SPEC.md:190-198.
MetricsResult compute_metrics(const Mesh& mesh, NavAlgo nav_algo, VolAlgo vol_algo);

// max_j |a_j| / max_e |n_e| after the 1/D boundary closure.
double check_closure(const Mesh& mesh, const EdgeList& edges, const LumpedNavField& navs);

// |sum V_j - sum V_E| / sum V_E, compensated sums.
double check_total_volume(const Mesh& mesh, const DualVolumeField& volumes);

// affine flux F(x) = A x + b (A row-major D x D).  Relative
// interior residual of Res_j / V_j against trace(A); constant flux (A == 0)
// checks the balance with the boundary closure.  trace(A) == 0 with A != 0
// throws std::invalid_argument.
double check_linear_exactness(const Mesh& mesh, const EdgeList& edges,
                              const LumpedNavField& navs, const DualVolumeField& volumes,
                              const std::vector<double>& A, const std::vector<double>& b);

}  // namespace dualmesh

#endif  // DUALMESH_METRICS_HPP
