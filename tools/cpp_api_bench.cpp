// cpp_api_bench.cpp -- times the reference-facing C++ API (include/dualmesh/
// mesh.hpp + metrics.hpp, the drop-in surface) on a BASELINE grid, the way a
// reference user calls it: std::vector in, std::vector out.
//
//   cpp_api_bench [n = 256]      (n^3 Kuhn cube, +-0.15h, seed 42: C5 at 256)
//
// Prints one JSON object (ms):
//   compute_metrics_first   fresh topology: upload, K1, plan, step, results back
//   compute_metrics_repeat  same mesh again (topology resident: coordinates only)
//   compute_metrics_moved   same topology, moved interior nodes
//   navs_dualfree_repeat    lumped_navs_dualfree(mesh, edges) on the resident topology
//   volumes_edge_repeat     dual_volumes_edge_based(mesh, edges, navs)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dm_meshgen.h"
#include "dualmesh/mesh.hpp"
#include "dualmesh/metrics.hpp"

using namespace dualmesh;

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 256;
  int64_t nv = 0, ne = 0, nb = 0;
  dmg_tet_box_sizes(n, n, n, &nv, &ne, &nb);
  Mesh m;
  m.dim = 3;
  m.coords.resize(3 * nv);
  m.elements.resize(4 * ne);
  m.boundary.resize(3 * nb);
  if (dmg_tet_box(n, n, n, nullptr, 0, 0.15, 42, m.coords.data(), m.elements.data(),
                  m.boundary.data()))
    return 1;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  // warm the device context (driver init is not part of any call)
  (void)max_element_volume(Mesh{3, {0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1}, {0, 1, 2, 3}, {}});
  auto t0 = now();
  MetricsResult r = compute_metrics(m, NavAlgo::dualfree, VolAlgo::edge);
  auto t1 = now();
  MetricsResult r2 = compute_metrics(m, NavAlgo::dualfree, VolAlgo::edge);
  auto t2 = now();
  for (std::size_t i = 0; i < m.coords.size(); ++i) {  // a small interior displacement
    const double x = m.coords[i];
    if (x > 0.0 && x < 1.0) m.coords[i] = x + 1e-4 * ((i % 7) - 3.0) / 3.0 / n;
  }
  auto t3 = now();
  MetricsResult r3 = compute_metrics(m, NavAlgo::dualfree, VolAlgo::edge);
  auto t4 = now();
  LumpedNavField f = lumped_navs_dualfree(m, r3.edges);
  auto t5 = now();
  DualVolumeField v = dual_volumes_edge_based(m, r3.edges, f);
  auto t6 = now();
  const bool c1 = r.navs.navs == r2.navs.navs, c2 = r.volumes.volumes == r2.volumes.volumes,
             c3 = f.navs == r3.navs.navs, c4 = v.volumes == r3.volumes.volumes,
             c5 = r.edges.edges == r3.edges.edges;
  const bool same = c1 && c2 && c3 && c4 && c5;
  if (!same) std::fprintf(stderr, "consistency: %d %d %d %d %d\n", c1, c2, c3, c4, c5);
  std::printf("{\"n\": %d, \"n_elements\": %lld, \"n_edges\": %zu, "
              "\"compute_metrics_first_ms\": %.3f, \"compute_metrics_repeat_ms\": %.3f, "
              "\"compute_metrics_moved_ms\": %.3f, \"navs_dualfree_repeat_ms\": %.3f, "
              "\"volumes_edge_repeat_ms\": %.3f, \"consistent\": %s}\n",
              n, static_cast<long long>(ne), r.edges.size(), ms(t0, t1), ms(t1, t2), ms(t3, t4),
              ms(t4, t5), ms(t5, t6), same ? "true" : "false");
  return same ? 0 : 2;
}
