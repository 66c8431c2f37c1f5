// Wan2.1-shaped DiT runtime (placeholder, filled in next).
#include "bc_common.h"
extern "C" int64_t bc_wan_workspace_bytes(const bc_wan_dims*) { return 0; }
extern "C" int bc_wan_create(const bc_wan_dims*, const bc_wan_params*, void*, void*, int64_t, bc_wan_ctx**) { return bc_fail(BC_ERR_CUDA, "not implemented"); }
extern "C" int bc_wan_destroy(bc_wan_ctx*) { return 0; }
extern "C" int bc_wan_set_text(bc_wan_ctx*, const float*, void*) { return bc_fail(BC_ERR_CUDA, "not implemented"); }
extern "C" int bc_wan_step(bc_wan_ctx*, const bc_batch*, const bc_wan_update*, int32_t*, void*) { return bc_fail(BC_ERR_CUDA, "not implemented"); }
