/* oracle.h -- CPU oracle for the dual-free grid-metric path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker or the timed CPU baseline -- never as the product
 * path.  The product (libdualmesh.so) never links or calls it.
 *
 * What it restates, serially and deterministically:
 *  - build_edges / edge_of: reference proj/src/mesh.cpp:256-285, 58-73
 *    (also pinned against the reference's own mesh.cpp compiled into
 *    oracle/_ref/ by oracle/Makefile);
 *  - geometry: mesh.cpp:25-27 (cross), 75-92 (element_volume), 94-111
 *    (opposite_face_normal), 113-127 (boundary_normal);
 *  - metrics: SPEC.md:147-188, with the floating-point contract of
 *    SURVEY.md Appendix A (no FMA: built with -ffp-contract=off; constants
 *    1.0/3.0, 1.0/12.0, 1.0/(D*(D+1)), 1.0/(2D), 1.0/(D+1) as rounded
 *    multipliers; per-edge sums in ascending element id then ascending
 *    boundary id);
 *  - verify: SPEC.md:245-263 (closure, compensated total volume).
 * Parity pins: tests/golden/ (reference outputs + SPEC examples).
 */
#ifndef DM_ORACLE_H
#define DM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Edge extraction.  Returns n_edges or -1.  *edges (2 per edge) and
 * *origin_start (n_nodes+1) are malloc'd; free with or_free. */
int64_t or_build_edges(int dim, int64_t n_nodes, const int32_t* elements, int64_t n_elements,
                       int32_t** edges, uint64_t** origin_start);
int32_t or_edge_of(const int32_t* edges, const uint64_t* origin_start, int64_t n_nodes,
                   int32_t a, int32_t b);
/* e2l[e*L+l] (local order mesh.cpp:17,263-265); inc_ptr[n_edges+1], inc[L*nE]. */
int or_edge_maps(int dim, int64_t n_nodes, const int32_t* elements, int64_t n_elements,
                 const int32_t* edges, const uint64_t* origin_start, int64_t n_edges,
                 int32_t* e2l, int32_t* inc_ptr, int32_t* inc);
void or_free(void* p);

/* Geometry (out: 3 doubles, z = 0 in 2D). */
double or_element_volume(int dim, const double* x, const int32_t* el);
void or_opposite_face_normal(int dim, const double* x, const int32_t* el, int i, double* out);
void or_boundary_normal(int dim, const double* x, const int32_t* bl, double* out);

/* Metrics.  e2l may be NULL (then edge_of is used per element edge). */
int or_navs_dualfree(int dim, const double* x, int64_t n_nodes, const int32_t* elements,
                     int64_t n_elements, const int32_t* boundary, int64_t n_boundary,
                     const int32_t* edges, const uint64_t* origin_start, int64_t n_edges,
                     const int32_t* e2l, double* navs);
int or_navs_traditional(int dim, const double* x, int64_t n_nodes, const int32_t* elements,
                        int64_t n_elements, const int32_t* edges, const uint64_t* origin_start,
                        int64_t n_edges, const int32_t* e2l, double* navs);
int or_volumes_edge(int dim, const double* x, int64_t n_nodes, const int32_t* edges,
                    int64_t n_edges, const double* navs, double* volumes);
int or_volumes_element(int dim, const double* x, int64_t n_nodes, const int32_t* elements,
                       int64_t n_elements, double* volumes);

/* Verify.  closure: max_j |a_j| / max_e |n_e| over all nodes after the 1/D
 * boundary closure; interior: same over non-boundary nodes before it. */
int or_check_closure(int dim, const double* x, int64_t n_nodes, const int32_t* boundary,
                     int64_t n_boundary, const int32_t* edges, int64_t n_edges,
                     const double* navs, double* residual, double* interior_residual);
/* affine flux F(x) = A x + b (A row-major D x D).  Returns -1
 * if trace(A) == 0 with A != 0.  See oracle.c for the residual definition. */
int or_check_linear_exactness(int dim, const double* x, int64_t n_nodes, const int32_t* boundary,
                              int64_t n_boundary, const int32_t* edges, int64_t n_edges,
                              const double* navs, const double* volumes, const double* A,
                              const double* b, double* residual);
/* Neumaier-compensated sums; returns |sV - sE| / sE in *rel. */
int or_check_total_volume(int dim, const double* x, int64_t n_nodes, const int32_t* elements,
                          int64_t n_elements, const double* volumes, double* rel,
                          double* sum_v, double* sum_e);
double or_max_face_area(int dim, const double* x, const int32_t* elements, int64_t n_elements);
double or_max_element_volume(int dim, const double* x, const int32_t* elements,
                             int64_t n_elements);

/* Multi-threaded dual-free navs + edge volumes (bench reference arm): per-edge
 * and per-node gathers in the serial loops' summation order (same bits on any
 * thread count).  The plan holds the incidence / boundary / incoming lists
 * (topology only); s receives the per-edge volume terms. */
typedef struct or_plan or_plan;
or_plan* or_plan_create(int dim, int64_t n_nodes, const int32_t* elements, int64_t n_elements,
                        const int32_t* boundary, int64_t n_boundary, const int32_t* edges,
                        const uint64_t* origin_start, int64_t n_edges);
void or_plan_free(or_plan* plan);
int or_metrics_mt(const or_plan* plan, const double* x, int nthreads, double* navs, double* s,
                  double* volumes);

/* Input synthesis: Kuhn cube n^3 x 6 tets, interior
 * jitter amp*h per axis from splitmix64(seed).  x: 3(n+1)^3, el: 24 n^3,
 * bnd: 36 n^2 entries. */
int or_gen_tet_cube(int n, double amp, uint64_t seed, double* x, int32_t* el, int32_t* bnd);

#ifdef __cplusplus
}
#endif

#endif
