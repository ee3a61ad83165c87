/* dm_meshgen.h -- C-ABI of libdm_meshgen.so: the SPEC meshgen module
 * (SPEC.md:308-364), used to synthesise the BASELINE.json grids.
 *
 * The reference ships no generator code; the contract is SPEC.md:313-341
 * plus the concrete grids of SURVEY.md 8(d).  Randomness comes from
 * splitmix64 (a named portable generator):
 *   x += 0x9E3779B97F4A7C15; z = x;
 *   z = (z ^ z>>30) * 0xBF58476D1CE4E5B9; z = (z ^ z>>27) * 0x94D049BB133111EB;
 *   return z ^ z>>31;
 * u = (x >> 11) * 2^-53, jitter = (2u - 1) * amplitude * h.
 * All outputs are caller-allocated; *_sizes gives the counts first.
 */
#ifndef DM_MESHGEN_H
#define DM_MESHGEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Unit square, n x n quads, two CCW triangles each.  diag_seed == 0 picks
 * the uniform lower-left -> upper-right diagonal; otherwise
 * each quad's diagonal is drawn from splitmix64(diag_seed), p = 1/2.
 * Interior nodes get x,y += U(-amp h, amp h) from splitmix64(seed), drawn
 * in node order, x then y.  Boundary edges run CCW around the square. */
void dmg_tri_square_sizes(int n, int64_t* n_nodes, int64_t* n_elements, int64_t* n_boundary);
int dmg_tri_square(int n, uint64_t diag_seed, double amp, uint64_t seed, double* coords,
                   int32_t* elements, int32_t* boundary);

/* nx*ny*nz hexes of a box, each split into the 6 Kuhn tetrahedra sharing
 * the (0,0,0)-(1,1,1) diagonal, positively oriented.
 * x,y nodes are uniform on [0,1]; z nodes are uniform on [0,1] when
 * z_nodes is NULL, else z_nodes[0..nz].  Node (i,j,k) has id
 * i + (nx+1)*(j + (ny+1)*k).  Boundary triangles are outward, two per
 * boundary quad, faces in order x=0,x=1,y=0,y=1,z=0,z=1.
 * jitter_mode 0: nodes interior in all three axes move by U(+-amp h) per
 *   axis (x,y,z order); jitter_mode 1 (boundary layer): nodes interior in
 *   x and y move in x,y only, every layer, no z jitter. */
void dmg_tet_box_sizes(int nx, int ny, int nz, int64_t* n_nodes, int64_t* n_elements,
                       int64_t* n_boundary);
int dmg_tet_box(int nx, int ny, int nz, const double* z_nodes, int jitter_mode, double amp,
                uint64_t seed, double* coords, int32_t* elements, int32_t* boundary);

/* Geometric boundary-layer z distribution: z_0 = 0, z_{k+1} = z_k + dz0*ratio^k. */
int dmg_bl_z(int nz, double dz0, double ratio, double* z_nodes);

/* Random relabelling (Fisher-Yates with splitmix64; j = next() % (i+1)):
 * node ids by node_seed, element order by elem_seed (0 = keep).  Local node
 * order inside each element is kept, so orientation is kept. */
int dmg_permute(int dim, int64_t n_nodes, int64_t n_elements, int64_t n_boundary,
                uint64_t node_seed, uint64_t elem_seed, double* coords, int32_t* elements,
                int32_t* boundary);

/* Returns the index of the first non-positive element (signed volume on the
 * generated coordinates) or -1: the post-hoc inversion check of SPEC.md:336. */
/* Seeded random 2-3 flips of a valid tet mesh (n_nodes < 2^31): interior
 * faces abc shared by (a,b,c,d) and (a,b,c,e) whose segment d-e pierces abc
 * become (a,b,d,e), (b,c,d,e), (c,a,d,e); visited in splitmix64(seed)
 * shuffled order, each tet in at most one flip, slivers (< 1e-3 of the mean
 * new volume) skipped, at most max_flips flips.  out_elements (4 *
 * (n_elements + max_flips) ids) gets the flipped mesh, positively oriented;
 * returns the number of flips (elements: n_elements + flips), or -1. */
int64_t dmg_flip23(int64_t n_nodes, const double* coords, int64_t n_elements,
                   const int32_t* elements, int64_t max_flips, uint64_t seed,
                   int32_t* out_elements);
int64_t dmg_first_inverted(int dim, int64_t n_elements, const double* coords,
                           const int32_t* elements);

#ifdef __cplusplus
}
#endif

#endif /* DM_MESHGEN_H */
