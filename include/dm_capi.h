/* dm_capi.h -- C-ABI of libdualmesh.so, the B200 (sm_100a) grid-metric engine.
 *
 * Plain C: opaque context handle, plain pointers and sizes, int status codes.
 * No C++ exception and no torch type crosses this boundary.  Every entry
 * point names the reference interface it replaces (file:line under
 * /root/reference).  Ids are 0-based, as in the reference Mesh
 * (proj/include/dualmesh/mesh.hpp:17-18).
 *
 * Ownership: host inputs are borrowed for the duration of a call and copied
 * to the device; device buffers belong to the context; host outputs are
 * caller-allocated.  Threading: one context per host thread; all work is
 * ordered on the context's CUDA stream and every dm_get_* synchronises it.
 * There is no CPU fallback: without a usable sm_100 device, dm_create fails
 * with DM_ERR_CUDA.
 */
#ifndef DM_CAPI_H
#define DM_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define DM_OK 0
#define DM_ERR_INVALID_ARG (-1)
#define DM_ERR_MESH_EDGE_MISMATCH (-2) /* SPEC.md:151,174 "mesh/edge mismatch" */
#define DM_ERR_EDGE_ABSENT (-3)        /* SPEC.md:164 boundary edge not in EdgeList */
#define DM_ERR_CUDA (-4)
#define DM_ERR_OOM (-5)
#define DM_ERR_STATE (-6)       /* call order, e.g. navs before edges */
#define DM_ERR_UNSUPPORTED (-7) /* size limits of the device layout */

/* ---- algorithm selectors ----------------------------------------------- */
#define DM_NAV_TRADITIONAL 0
#define DM_NAV_DUALFREE 1
#define DM_VOL_EDGE 0
#define DM_VOL_ELEMENT 1
/* Element-loop variants (north_star (b)). */
#define DM_VARIANT_GATHER 0       /* ring-walk gather (default): deterministic, <=1e-12 */
#define DM_VARIANT_SCATTER 1      /* fp64 atomics (REDG.F64), order nondeterministic */
#define DM_VARIANT_GATHER_ELEM 2  /* element-id CSR gather + conn lookup, bitwise */
#define DM_VARIANT_GATHER_FACES 3 /* face-list CSR gather, bitwise */
#define DM_VARIANT_GATHER_EXACT 4 /* row-table CSR gather, bitwise = serial oracle */

typedef struct dm_ctx dm_ctx;

/* Device-resident views, for device-side timing without PCIe. */
typedef struct dm_device_view {
  int dim;
  int64_t n_nodes, n_elements, n_boundary, n_edges;
  const double* coords;       /* dim doubles per node (caller layout) */
  const int32_t* elements;    /* dim+1 per element */
  const int32_t* boundary;    /* dim per boundary facet */
  const int32_t* edges;       /* 2 per edge (min, max) */
  const uint32_t* origin_start; /* n_nodes+1 (32-bit on device) */
  const int32_t* e2l;         /* L per element */
  const int32_t* inc_ptr;     /* n_edges+1 */
  const int32_t* inc;         /* L*n_elements, ascending element per edge */
  double* navs;               /* dim doubles per edge */
  double* volumes;            /* n_nodes */
} dm_device_view;

int dm_version(void);
const char* dm_status_string(int status);

/* Context lifetime.  device: CUDA ordinal. */
int dm_create(dm_ctx** out, int device);
void dm_destroy(dm_ctx* ctx);
const char* dm_last_error(const dm_ctx* ctx);

/* Mesh upload (replaces constructing dualmesh::Mesh, ref mesh.hpp:23-44).
 * coords: dim*n_nodes doubles; elements: (dim+1)*n_elements ids;
 * boundary: dim*n_boundary ids (may be NULL when n_boundary == 0).
 * Drops every derived structure. */
int dm_set_mesh(dm_ctx* ctx, int dim, const double* coords, int64_t n_nodes,
                const int32_t* elements, int64_t n_elements, const int32_t* boundary,
                int64_t n_boundary);
/* New coordinates for the same topology (deforming-grid step input);
 * edge structures are kept.  Host pointer / device pointer forms. */
int dm_set_coords(dm_ctx* ctx, const double* coords);
int dm_set_coords_device(dm_ctx* ctx, const double* d_coords);

/* Device-side SPEC meshgen: the grids of
 * include/dm_meshgen.h generated straight into the context (bitwise the same
 * coordinates, elements and boundary as the host generator), replacing the
 * current mesh like dm_set_mesh.  z_nodes: host array of nz+1 values or NULL.
 * dm_gen_permute relabels the context's mesh as dmg_permute does. */
int dm_gen_tri_square(dm_ctx* ctx, int n, uint64_t diag_seed, double amp, uint64_t seed);
int dm_gen_tet_box(dm_ctx* ctx, int nx, int ny, int nz, const double* z_nodes, int jitter_mode,
                   double amp, uint64_t seed);
int dm_gen_permute(dm_ctx* ctx, uint64_t node_seed, uint64_t elem_seed);
/* The context's mesh back to the host (any pointer may be NULL), and its sizes. */
int dm_get_mesh(dm_ctx* ctx, double* coords, int32_t* elements, int32_t* boundary);
int dm_mesh_sizes(dm_ctx* ctx, int* dim, int64_t* n_nodes, int64_t* n_elements,
                  int64_t* n_boundary);

/* Edge extraction: ref build_edges, proj/src/mesh.cpp:256-285.  Also builds
 * the element-to-local-edge map e2l[e*L+l] (local order mesh.cpp:17,263-265)
 * and the edge-to-element CSR incidence (ascending element ids per edge).
 * DM_ERR_INVALID_ARG if an element references a node id outside
 * [0, n_nodes) (the reference's behaviour there is undefined). */
int dm_build_edges(dm_ctx* ctx, int64_t* n_edges);
/* edges: 2*n_edges ids; origin_start: n_nodes+1 (size_t in the reference,
 * mesh.hpp:50).  Either pointer may be NULL. */
int dm_get_edges(dm_ctx* ctx, int32_t* edges, uint64_t* origin_start);
int dm_get_e2l(dm_ctx* ctx, int32_t* e2l);
int dm_get_incidence(dm_ctx* ctx, int32_t* inc_ptr, int32_t* inc);
/* Batched ref EdgeList::edge_of, proj/src/mesh.cpp:58-73 (-1 if absent). */
int dm_edge_of(dm_ctx* ctx, const int32_t* a, const int32_t* b, int64_t n, int32_t* out);

/* Metrics.  Results stay on the device until fetched. */
int dm_navs(dm_ctx* ctx, int nav_algo, int variant);
int dm_volumes(dm_ctx* ctx, int vol_algo);
int dm_get_navs(dm_ctx* ctx, double* navs);       /* dim*n_edges */
int dm_get_volumes(dm_ctx* ctx, double* volumes); /* n_nodes */
/* Overwrite device navs / volumes from the host (volumes or verification on
 * externally supplied fields).  dm_put_navs also refreshes the per-edge
 * s_e = (x_k - x_j).n_jk consumed by the edge-based volume kernel. */
int dm_put_navs(dm_ctx* ctx, const double* navs);
int dm_put_volumes(dm_ctx* ctx, const double* volumes);

/* One end-to-end metrics step through host memory (the compute_metrics
 * facade, with the edge list prebuilt as in the SPEC bench
 * region SPEC.md:385): coords host->device, navs + volumes, results
 * device->host.  coords may be NULL to keep the resident coordinates. */
int dm_metrics_host(dm_ctx* ctx, const double* coords, int nav_algo, int variant,
                    int vol_algo, double* navs, double* volumes);

/* The same step, enqueued and returned from at once (a pipelined loop of
 * metrics over a moving or changing set of coordinates): coords arrive on a
 * host->device copy stream, the kernels run once they landed and the
 * previous step's kernels ended, navs / volumes leave on a device->host copy
 * stream.  navs / volumes alternate between two device buffers, so step i+1
 * computes while step i is still being copied out (PCIe is full duplex; the
 * step costs max(copy-out, copy-in + kernels) instead of their sum).  Host
 * buffers must stay valid and untouched until dm_sync(); pinned buffers
 * (dm_host_alloc) are needed for the copies to overlap.  Device views
 * (dm_device_views) are valid until the next metrics call. */
int dm_metrics_host_async(dm_ctx* ctx, const double* coords, int nav_algo, int variant,
                          int vol_algo, double* navs, double* volumes);

/* Verification on the resident navs / volumes. */
int dm_check_closure(dm_ctx* ctx, double* residual, double* interior_residual);
/* SPEC.md:265-274 check_linear_exactness: affine flux F(x) = A x + b (A row-major
 * dim x dim, host).  trace(A) != 0: max over interior nodes of
 * |Res_j / V_j - trace(A)| / |trace(A)| (needs navs and volumes); A == 0:
 * constant flux, max_j |Res_j| / max_e |phi_e| after the boundary closure.
 * trace(A) == 0 with A != 0 -> DM_ERR_INVALID_ARG. */
int dm_check_linear_exactness(dm_ctx* ctx, const double* A, const double* b, double* residual);
int dm_check_total_volume(dm_ctx* ctx, double* rel_err, double* sum_volumes,
                          double* sum_elements);
/* SPEC.md:455,482 hidden test hook: add delta to every component of one nav. */
int dm_corrupt_nav(dm_ctx* ctx, int64_t edge, double delta);

/* Mesh-wide helpers (ref mesh.hpp:92-98, mesh.cpp:325-349). */
int dm_max_face_area(dm_ctx* ctx, double* out);
int dm_max_element_volume(dm_ctx* ctx, double* out);
int dm_total_volume(dm_ctx* ctx, double* out); /* compensated sum */
int dm_boundary_node_mask(dm_ctx* ctx, uint8_t* mask);

/* Validation and boundary derivation (ref mesh.cpp:129-254, 287-323).
 * dm_validate fills per-element volume signs (n_elements, may be NULL) and
 * counts of each violation class into counts[DM_VCOUNT]; detail strings are
 * produced by the C++ layer from the first offending ids in first_ids. */
#define DM_VCOUNT 8
#define DM_V_OUT_OF_RANGE_ELEM 0
#define DM_V_OUT_OF_RANGE_BND 1
#define DM_V_NONPOSITIVE 2
#define DM_V_FACE_OVERSHARED 3
#define DM_V_BND_NOT_FACE 4
#define DM_V_BND_INTERIOR 5
#define DM_V_BND_DUPLICATE 6
#define DM_V_BND_INWARD 7
int dm_validate(dm_ctx* ctx, int8_t* volume_signs, int64_t counts[DM_VCOUNT],
                int64_t* exposed_faces);
int dm_validate_list(dm_ctx* ctx, int kind, int64_t* ids, int64_t cap, int64_t* n);
int dm_derive_boundary(dm_ctx* ctx, int64_t* n_faces);
int dm_get_derived_boundary(dm_ctx* ctx, int32_t* faces);

/* Plumbing: stream, device views, per-phase timing, launch counter. */
int dm_stream(dm_ctx* ctx, void** stream);
int dm_device_views(dm_ctx* ctx, dm_device_view* view);
int dm_sync(dm_ctx* ctx); /* waits for the ctx stream and the pipelined copies */
/* When enabled, dm_navs / dm_volumes record CUDA events around each kernel
 * phase on the context stream; dm_get_timings returns the last values (ms):
 * [0] element loop, [1] boundary pass, [2] edge-volume loop, [3] total. */
int dm_set_timing(dm_ctx* ctx, int enable);
int dm_get_timings(dm_ctx* ctx, float* ms, int n);
/* enable > 1 keeps the phase events of the last `enable` steps (a step = one
 * dm_navs + dm_volumes pair), so a caller can time a run of back-to-back
 * steps without synchronising inside it: dm_get_step_timings waits for the
 * last recorded step and returns up to max_steps rows of the four values
 * above, oldest first (ms[4 * s + i]); *n_steps = rows written. */
int dm_get_step_timings(dm_ctx* ctx, float* ms, int max_steps, int* n_steps);
int64_t dm_kernel_launches(const dm_ctx* ctx);
/* Which element-loop kernels the plan enables: info[0] ring path built (1: Morton
 * tiles, rings.cu; 2: row tiles, rowplan.cu),
 * [1] ring path usable, [2] row tables built, [3] row tables usable,
 * [4] max tile node count (ring path), [5] ring-build bits (2: a Morton tile
 * touches > 1536 nodes and 32: ring codes beyond 64 GB disable the ring path;
 * 4: an edge has > 24 incident elements, 8: a non-manifold fan, 16: an
 * inconsistently oriented fan, 64: a table slot beyond 255 in one of a few Morton
 * tiles over 256 nodes send those edges to the side list),
 * [6] edge-volume pass walks nodes in Morton order (1) or id order (0),
 * [7] tile tables recoloured against bank conflicts (env DUALMESH_PLAN_COLOR=1). */
int dm_plan_info(dm_ctx* ctx, int64_t info[8]);
/* Edges of the ring path's side list (*n): those the ring codes cannot
 * describe -- more than 24 incident elements, a non-manifold or inconsistently
 * oriented fan -- evaluated from their element list inside the same dm_navs
 * call (0 when the ring path is not in use).  [5] of dm_plan_info gives the
 * reasons (4 / 8 / 16 / 64). */
int dm_plan_side_edges(dm_ctx* ctx, int64_t* n);
/* Per-step streams of the row-tile element loop (zeros for other plans):
 * out[0] ring-code bytes, [1] node-table fill bytes (24 B per table slot, from
 * L2 or HBM), [2] tile metadata + run descriptor bytes, [3] tiles.  With the
 * navs / s rows written and the coordinates read once, these are the bytes
 * the kernel's design moves (bench.py design_roofline). */
int dm_plan_bytes(dm_ctx* ctx, int64_t out[4]);
/* SPEC cli_io file formats, host only (no device needed).
 * MeshFile: dm_mesh_file_read parses `path` (call with NULL arrays for the
 * sizes first); ids come back 0-based; *has_boundary = 0 when the file has no
 * boundary section (derive it with dm_derive_boundary).  Parse errors return
 * DM_ERR_INVALID_ARG with "path:line: what" in err (syntax, count mismatch,
 * invalid index).  dm_mesh_file_write writes 1-based ids and 17-significant-
 * digit coordinates (lossless).  MetricsFile: JSON with 1-based edges, navs,
 * volumes and provenance (algorithm names, dm_mesh_checksum = FNV-1a 64 of the
 * mesh arrays); deterministic bytes. */
int dm_mesh_file_read(const char* path, int* dim, int64_t* n_nodes, int64_t* n_elements,
                      int64_t* n_boundary, int* has_boundary, double* coords, int32_t* elements,
                      int32_t* boundary, char* err, int64_t err_len);
int dm_mesh_file_write(const char* path, int dim, const double* coords, int64_t n_nodes,
                       const int32_t* elements, int64_t n_elements, const int32_t* boundary,
                       int64_t n_boundary);
uint64_t dm_mesh_checksum(int dim, const double* coords, int64_t n_nodes, const int32_t* elements,
                          int64_t n_elements, const int32_t* boundary, int64_t n_boundary);
int dm_metrics_file_write(const char* path, int dim, const int32_t* edges, int64_t n_edges,
                          const double* navs, const double* volumes, int64_t n_nodes,
                          int nav_algo, int vol_algo, uint64_t mesh_checksum);

/* Pinned host memory for end-to-end transfers. */
int dm_host_alloc(size_t bytes, void** ptr);
int dm_host_free(void* ptr);

#ifdef __cplusplus
}
#endif

#endif /* DM_CAPI_H */
