// capi.cu -- the extern "C" surface of libdualmesh.so (include/dm_capi.h):
// context lifetime, mesh upload, result download, timing and plumbing.
#include <cstdlib>
#include <cstring>
#include <vector>

#include "dm_internal.cuh"

using namespace dm;

namespace {

// origin CSR widened to the reference's size_t (mesh.hpp:50) on the device
__global__ void k_widen_u32(const u32* __restrict__ in, i64 n, u64* __restrict__ out) {
  const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

const char* kStatus[] = {"ok",           "invalid argument", "mesh/edge mismatch",
                         "boundary edge absent from EdgeList", "CUDA error", "out of device memory",
                         "call order",   "unsupported size"};

int check_device(dm_ctx* c) {
  int n = 0;
  cudaError_t st = cudaGetDeviceCount(&n);
  if (st != cudaSuccess || n == 0)
    return fail(c, DM_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(st));
  if (c->device < 0 || c->device >= n) return fail(c, DM_ERR_INVALID_ARG, "bad device ordinal");
  cudaDeviceProp prop;
  DM_CK(c, cudaGetDeviceProperties(&prop, c->device));
  if (prop.major != 10 || prop.minor != 0)
    return fail(c, DM_ERR_CUDA, std::string("libdualmesh is built for sm_100a only; device is ") +
                                    prop.name);
  return DM_OK;
}

void drop_derived(dm_ctx* c) {
  c->have_edges = c->have_in = c->have_bedge = c->have_n2e = c->have_ifl = c->have_tables =
      c->have_rings = false;
  c->have_navs = c->have_vols = false;
  c->navs_algo = -1;
  c->ne = 0;
  c->n_bedge = 0;
  c->n_derived = 0;
  c->n_side = 0;
}

// Writers of navs / volumes on the compute stream wait for the pipelined
// copies still reading them (no-op without dm_metrics_host_async).
int wait_out_copies(dm_ctx* c) {
  for (cudaEvent_t e : c->ev_out)
    if (e) DM_CK(c, cudaStreamWaitEvent(c->stream, e, 0));
  return DM_OK;
}
int sync_all(dm_ctx* c) {
  DM_CK(c, cudaStreamSynchronize(c->stream));
  for (cudaStream_t s : {c->s_h2d, c->s_d2h})
    if (s) DM_CK(c, cudaStreamSynchronize(s));
  return DM_OK;
}

float ev_ms(dm_ctx* c, int a, int b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]) != cudaSuccess) ms = -1.f;
  return ms;
}

}  // namespace

extern "C" {

int dm_version(void) { return 1; }

const char* dm_status_string(int status) {
  if (status > 0 || status < -7) return "unknown status";
  return kStatus[-status];
}

int dm_create(dm_ctx** out, int device) {
  if (!out) return DM_ERR_INVALID_ARG;
  *out = nullptr;
  auto* c = new dm_ctx;
  c->device = device;
  // test hook (tests/test_gpu_parity.py): 41 sends every Morton tile down the
  // ring kernel's global-memory path
  if (const char* g = std::getenv("DUALMESH_GATHER_CFG")) c->gather_cfg = std::atoi(g);
  int st = check_device(c);
  if (st == DM_OK) {
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    for (int i = 0; i < 8 && e == cudaSuccess; ++i) e = cudaEventCreate(&c->ev[i]);
    if (e != cudaSuccess) st = fail(c, DM_ERR_CUDA, cudaGetErrorString(e));
  }
  if (st != DM_OK) {
    // keep the context so dm_last_error can explain the failure
    *out = c;
    return st;
  }
  *out = c;
  return DM_OK;
}

void dm_destroy(dm_ctx* c) {
  if (!c) return;
  if (c->stream) {
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (cudaStream_t s : {c->s_h2d, c->s_d2h})
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    for (auto& e : c->ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : c->ev_ring)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : {c->ev_h2d, c->ev_comp, c->ev_out[0], c->ev_out[1]})
      if (e) cudaEventDestroy(e);
    cudaStreamDestroy(c->stream);
  }
  release_stage(c);
  delete c;
}



const char* dm_last_error(const dm_ctx* c) { return c ? c->err.c_str() : "null context"; }

int dm_set_mesh(dm_ctx* c, int dim, const double* coords, int64_t n_nodes, const int32_t* elements,
                int64_t n_elements, const int32_t* boundary, int64_t n_boundary) {
  if (!c || !c->stream) return DM_ERR_INVALID_ARG;
  if ((dim != 2 && dim != 3) || n_nodes < 0 || n_elements < 0 || n_boundary < 0)
    return fail(c, DM_ERR_INVALID_ARG, "dim must be 2 or 3 and counts non-negative");
  if ((n_nodes && !coords) || (n_elements && !elements) || (n_boundary && !boundary))
    return fail(c, DM_ERR_INVALID_ARG, "null array with non-zero count");
  if (n_nodes >= (1ll << 31)) return fail(c, DM_ERR_UNSUPPORTED, "node ids are 32-bit");
  if (int w = sync_all(c)) return w;  // pipelined copies may still read the old buffers
  c->navs_alt.release();
  c->vols_alt.release();
  drop_derived(c);
  c->dim = dim;
  c->nv = n_nodes;
  c->nE = n_elements;
  c->nB = n_boundary;
  // two spare records: the row plan's TMA copies round node runs up to even ids
  DM_CK(c, c->coords.ensure(static_cast<size_t>(dim * (n_nodes + 2))));
  DM_CK(c, c->elems.ensure(static_cast<size_t>((dim + 1) * n_elements)));
  DM_CK(c, c->bnd.ensure(static_cast<size_t>(dim * n_boundary)));
  if (int st = copy_h2d(c, c->coords.p, coords, sizeof(double) * dim * n_nodes)) return st;
  if (int st = copy_h2d(c, c->elems.p, elements, sizeof(int32_t) * (dim + 1) * n_elements))
    return st;
  if (int st = copy_h2d(c, c->bnd.p, boundary, sizeof(int32_t) * dim * n_boundary)) return st;
  int st = coords_changed(c);
  if (st) return st;
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}

int dm_set_coords(dm_ctx* c, const double* coords) {
  if (!c || !coords) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "dm_set_coords before dm_set_mesh");
  if (int st = copy_h2d(c, c->coords.p, coords, sizeof(double) * c->dim * c->nv)) return st;
  c->have_navs = c->have_vols = false;
  return coords_changed(c);
}

int dm_set_coords_device(dm_ctx* c, const double* d_coords) {
  if (!c || !d_coords) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "dm_set_coords_device before dm_set_mesh");
  DM_CK(c, cudaMemcpyAsync(c->coords.p, d_coords, sizeof(double) * c->dim * c->nv,
                           cudaMemcpyDeviceToDevice, c->stream));
  c->have_navs = c->have_vols = false;
  return coords_changed(c);
}

int dm_build_edges(dm_ctx* c, int64_t* n_edges) {
  if (!c) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "dm_build_edges before dm_set_mesh");
  int st = build_edges_impl(c);
  if (st) return st;
  if (n_edges) *n_edges = c->ne;
  return DM_OK;
}

int dm_get_edges(dm_ctx* c, int32_t* edges, uint64_t* origin_start) {
  if (!c) return DM_ERR_INVALID_ARG;
  if (!c->have_edges) return fail(c, DM_ERR_STATE, "edges not built");
  if (edges && c->ne)
    if (int st = copy_d2h(c, edges, c->edges.p, sizeof(int2) * c->ne)) return st;
  if (origin_start) {
    // widen the 32-bit device CSR to the reference's size_t (mesh.hpp:50)
    DevBuf<u64> wide;
    DM_CK(c, wide.ensure(static_cast<size_t>(c->nv + 1)));
    DM_LAUNCH(c, k_widen_u32, grid_for(c->nv + 1, 256), 256, 0, c->os.p, c->nv + 1, wide.p);
    if (int st = copy_d2h(c, origin_start, wide.p, sizeof(u64) * (c->nv + 1))) return st;
    DM_CK(c, cudaStreamSynchronize(c->stream));  // before the scratch is freed
  }
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}

int dm_get_e2l(dm_ctx* c, int32_t* e2l) {
  if (!c || !e2l) return DM_ERR_INVALID_ARG;
  if (!c->have_edges) return fail(c, DM_ERR_STATE, "edges not built");
  const int L = c->dim == 3 ? 6 : 3;
  if (int st = copy_d2h(c, e2l, c->e2l.p, sizeof(int32_t) * L * c->nE)) return st;
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}

int dm_get_incidence(dm_ctx* c, int32_t* inc_ptr, int32_t* inc) {
  if (!c) return DM_ERR_INVALID_ARG;
  if (!c->have_edges) return fail(c, DM_ERR_STATE, "edges not built");
  const int L = c->dim == 3 ? 6 : 3;
  if (inc_ptr)
    if (int st = copy_d2h(c, inc_ptr, c->inc_ptr.p, sizeof(int32_t) * (c->ne + 1))) return st;
  if (inc && c->nE)
    if (int st = copy_d2h(c, inc, c->inc.p, sizeof(int32_t) * L * c->nE)) return st;
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}

int dm_navs(dm_ctx* c, int nav_algo, int variant) {
  if (!c) return DM_ERR_INVALID_ARG;
  int st = wait_out_copies(c);
  return st ? st : navs_impl(c, nav_algo, variant);
}

int dm_volumes(dm_ctx* c, int vol_algo) {
  if (!c) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "no mesh");
  int st = wait_out_copies(c);
  return st ? st : volumes_impl(c, vol_algo);
}

int dm_get_navs(dm_ctx* c, double* navs) {
  if (!c || !navs) return DM_ERR_INVALID_ARG;
  if (!c->have_navs) return fail(c, DM_ERR_STATE, "navs not computed");
  if (int st = copy_d2h(c, navs, c->navs.p, sizeof(double) * c->dim * c->ne)) return st;
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}

int dm_put_navs(dm_ctx* c, const double* navs) {
  if (!c || !navs) return DM_ERR_INVALID_ARG;
  if (!c->have_edges) return fail(c, DM_ERR_STATE, "edges not built");
  if (int w = wait_out_copies(c)) return w;
  DM_CK(c, c->navs.ensure(static_cast<size_t>(c->dim * c->ne)));
  if (int st = copy_h2d(c, c->navs.p, navs, sizeof(double) * c->dim * c->ne)) return st;
  DM_CK(c, c->svals.ensure(static_cast<size_t>(c->ne)));
  int st = svals_from_navs(c);
  c->svals_pos = false;
  if (st) return st;
  c->have_navs = true;
  c->have_vols = false;
  c->navs_algo = -1;
  return DM_OK;
}

int dm_put_volumes(dm_ctx* c, const double* volumes) {
  if (!c || !volumes) return DM_ERR_INVALID_ARG;
  if (c->dim == 0) return fail(c, DM_ERR_STATE, "no mesh");
  if (int w = wait_out_copies(c)) return w;
  DM_CK(c, c->vols.ensure(static_cast<size_t>(c->nv)));
  if (int st = copy_h2d(c, c->vols.p, volumes, sizeof(double) * c->nv)) return st;
  c->have_vols = true;
  return DM_OK;
}

int dm_get_volumes(dm_ctx* c, double* volumes) {
  if (!c || !volumes) return DM_ERR_INVALID_ARG;
  if (!c->have_vols) return fail(c, DM_ERR_STATE, "volumes not computed");
  if (int st = copy_d2h(c, volumes, c->vols.p, sizeof(double) * c->nv)) return st;
  DM_CK(c, cudaStreamSynchronize(c->stream));
  return DM_OK;
}

int dm_metrics_host_async(dm_ctx* c, const double* coords, int nav_algo, int variant,
                          int vol_algo, double* navs, double* volumes) {
  if (!c) return DM_ERR_INVALID_ARG;
  if (!c->have_edges) return fail(c, DM_ERR_STATE, "build the edge list first");
  if (!c->s_h2d) {
    DM_CK(c, cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    DM_CK(c, cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&c->ev_h2d, &c->ev_comp, &c->ev_out[0], &c->ev_out[1]})
      DM_CK(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  }
  int st = DM_OK;
  if (coords) {
    // every kernel or copy already queued on the compute stream (earlier
    // steps, dm_navs / dm_volumes / verify calls, dm_set_coords copies) may
    // still read the resident coordinates: the copy-in waits for all of it
    DM_CK(c, cudaEventRecord(c->ev_comp, c->stream));
    DM_CK(c, cudaStreamWaitEvent(c->s_h2d, c->ev_comp, 0));
    DM_CK(c, cudaMemcpyAsync(c->coords.p, coords, sizeof(double) * c->dim * c->nv,
                             cudaMemcpyHostToDevice, c->s_h2d));
    DM_CK(c, cudaEventRecord(c->ev_h2d, c->s_h2d));
    DM_CK(c, cudaStreamWaitEvent(c->stream, c->ev_h2d, 0));
    c->have_navs = c->have_vols = false;
    st = coords_changed(c);
    if (st) return st;
  }
  // this step writes the other navs / vols buffer once its last copy-out ended
  const int slot = c->out_slot ^ 1;
  c->navs.swap(c->navs_alt);
  c->vols.swap(c->vols_alt);
  c->out_slot = slot;
  c->have_navs = c->have_vols = false;
  DM_CK(c, cudaStreamWaitEvent(c->stream, c->ev_out[slot], 0));
  st = navs_impl(c, nav_algo, variant);
  if (st) return st;
  st = volumes_impl(c, vol_algo);
  if (st) return st;
  DM_CK(c, cudaEventRecord(c->ev_comp, c->stream));
  DM_CK(c, cudaStreamWaitEvent(c->s_d2h, c->ev_comp, 0));
  if (navs)
    DM_CK(c, cudaMemcpyAsync(navs, c->navs.p, sizeof(double) * c->dim * c->ne,
                             cudaMemcpyDeviceToHost, c->s_d2h));
  if (volumes)
    DM_CK(c, cudaMemcpyAsync(volumes, c->vols.p, sizeof(double) * c->nv, cudaMemcpyDeviceToHost,
                             c->s_d2h));
  DM_CK(c, cudaEventRecord(c->ev_out[slot], c->s_d2h));
  return DM_OK;
}

int dm_metrics_host(dm_ctx* c, const double* coords, int nav_algo, int variant, int vol_algo,
                    double* navs, double* volumes) {
  int st = dm_metrics_host_async(c, coords, nav_algo, variant, vol_algo, navs, volumes);
  return st ? st : sync_all(c);
}

int dm_stream(dm_ctx* c, void** stream) {
  if (!c || !stream) return DM_ERR_INVALID_ARG;
  *stream = c->stream;
  return DM_OK;
}

int dm_device_views(dm_ctx* c, dm_device_view* v) {
  if (!c || !v) return DM_ERR_INVALID_ARG;
  std::memset(v, 0, sizeof(*v));
  v->dim = c->dim;
  v->n_nodes = c->nv;
  v->n_elements = c->nE;
  v->n_boundary = c->nB;
  v->n_edges = c->ne;
  v->coords = c->coords.p;
  v->elements = c->elems.p;
  v->boundary = c->bnd.p;
  if (c->have_edges) {
    v->edges = reinterpret_cast<const int32_t*>(c->edges.p);
    v->origin_start = c->os.p;
    v->e2l = c->e2l.p;
    v->inc_ptr = c->inc_ptr.p;
    v->inc = c->inc.p;
  }
  v->navs = c->have_navs ? c->navs.p : nullptr;
  v->volumes = c->have_vols ? c->vols.p : nullptr;
  return DM_OK;
}

int dm_sync(dm_ctx* c) {
  if (!c) return DM_ERR_INVALID_ARG;
  return sync_all(c);
}

int dm_set_timing(dm_ctx* c, int enable) {
  if (!c) return DM_ERR_INVALID_ARG;
  c->timing = enable != 0;
  // enable > 1: a ring of per-step phase events (dm_get_step_timings)
  const int steps = enable > 1 ? enable : 0;
  if (steps != c->ring_steps) {
    DM_CK(c, cudaStreamSynchronize(c->stream));
    for (cudaEvent_t e : c->ev_ring) cudaEventDestroy(e);
    c->ev_ring.clear();
    c->ring_steps = 0;
    if (steps > 0) {
      c->ev_ring.resize(static_cast<size_t>(4 * steps), nullptr);
      for (cudaEvent_t& e : c->ev_ring) DM_CK(c, cudaEventCreate(&e));
      c->ring_steps = steps;
    }
  }
  c->ring_pos = 0;
  return DM_OK;
}

int dm_get_step_timings(dm_ctx* c, float* ms, int max_steps, int* n_steps) {
  if (!c || !ms || !n_steps || max_steps < 0) return DM_ERR_INVALID_ARG;
  if (!c->timing || c->ring_steps == 0) return fail(c, DM_ERR_STATE, "step timing ring disabled");
  const long long have = c->ring_pos < c->ring_steps ? c->ring_pos : c->ring_steps;
  const long long n = have < max_steps ? have : max_steps;
  *n_steps = static_cast<int>(n);
  if (n == 0) return DM_OK;
  DM_CK(c, cudaStreamSynchronize(c->stream));
  for (long long s = 0; s < n; ++s) {  // the newest n steps, oldest first
    const size_t slot = static_cast<size_t>((c->ring_pos - n + s) % c->ring_steps);
    const cudaEvent_t* e = c->ev_ring.data() + 4 * slot;
    auto el = [&](int a, int b) {
      float v = 0.f;
      return cudaEventElapsedTime(&v, e[a], e[b]) == cudaSuccess ? v : -1.f;
    };
    ms[4 * s] = el(0, 1);
    ms[4 * s + 1] = el(1, 2);
    ms[4 * s + 2] = el(2, 3);
    ms[4 * s + 3] = el(0, 3);
  }
  return DM_OK;
}

int dm_get_timings(dm_ctx* c, float* ms, int n) {
  if (!c || !ms) return DM_ERR_INVALID_ARG;
  if (!c->timing) return fail(c, DM_ERR_STATE, "timing disabled");
  DM_CK(c, cudaEventSynchronize(c->ev[3]));
  c->last_ms[0] = ev_ms(c, 0, 1);
  c->last_ms[1] = ev_ms(c, 1, 2);
  c->last_ms[2] = ev_ms(c, 2, 3);
  c->last_ms[3] = ev_ms(c, 0, 3);
  for (int i = 0; i < n && i < 4; ++i) ms[i] = c->last_ms[i];
  return DM_OK;
}

int64_t dm_kernel_launches(const dm_ctx* c) { return c ? c->launches : -1; }

int dm_plan_info(dm_ctx* c, int64_t info[8]) {
  if (!c || !info) return DM_ERR_INVALID_ARG;
  for (int i = 0; i < 8; ++i) info[i] = 0;
  info[0] = c->have_rings ? (c->row_plan ? 2 : 1) : 0;
  info[1] = c->ring_ok;
  info[2] = c->have_tables;
  info[3] = c->table_ok;
  info[4] = c->ring_max_nodes;
  info[5] = c->ring_fail;
  info[6] = c->vol_by_rank;
  info[7] = c->plan_colored;
  return DM_OK;
}

int dm_plan_bytes(dm_ctx* c, int64_t out[4]) {
  if (!c || !out) return DM_ERR_INVALID_ARG;
  for (int i = 0; i < 4; ++i) out[i] = 0;
  if (!(c->have_rings && c->ring_ok && c->row_plan)) return DM_OK;
  out[0] = static_cast<int64_t>(c->rt_bytes[0]);
  out[1] = static_cast<int64_t>(c->rt_bytes[1]);
  out[2] = static_cast<int64_t>(c->rt_bytes[2]);
  out[3] = c->rt_ntiles;
  return DM_OK;
}

int dm_plan_side_edges(dm_ctx* c, int64_t* n) {
  if (!c || !n) return DM_ERR_INVALID_ARG;
  *n = c->have_rings && c->ring_ok ? c->n_side : 0;
  return DM_OK;
}

int dm_host_alloc(size_t bytes, void** ptr) {
  if (!ptr) return DM_ERR_INVALID_ARG;
  return cudaMallocHost(ptr, bytes) == cudaSuccess ? DM_OK : DM_ERR_OOM;
}

int dm_host_free(void* ptr) { return cudaFreeHost(ptr) == cudaSuccess ? DM_OK : DM_ERR_CUDA; }

}  // extern "C"
