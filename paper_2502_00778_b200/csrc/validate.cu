// validate.cu -- validate_mesh / derive_boundary_faces on the GPU
// (ref mesh.cpp:129-254, 287-323).  Filled in by the face-key bucket sort.
#include "dm_internal.cuh"

using namespace dm;

extern "C" int dm_validate(dm_ctx* c, int8_t*, int64_t*, int64_t*) {
  if (!c) return DM_ERR_INVALID_ARG;
  return fail(c, DM_ERR_UNSUPPORTED, "dm_validate not built yet");
}

extern "C" int dm_validate_list(dm_ctx* c, int, int64_t*, int64_t, int64_t*) {
  if (!c) return DM_ERR_INVALID_ARG;
  return fail(c, DM_ERR_UNSUPPORTED, "dm_validate_list not built yet");
}

extern "C" int dm_derive_boundary(dm_ctx* c, int64_t*) {
  if (!c) return DM_ERR_INVALID_ARG;
  return fail(c, DM_ERR_UNSUPPORTED, "dm_derive_boundary not built yet");
}

extern "C" int dm_get_derived_boundary(dm_ctx* c, int32_t*) {
  if (!c) return DM_ERR_INVALID_ARG;
  return fail(c, DM_ERR_UNSUPPORTED, "dm_get_derived_boundary not built yet");
}
