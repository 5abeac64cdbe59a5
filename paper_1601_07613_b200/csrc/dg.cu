// placeholder, replaced by the DG kernels
#include "mc_internal.h"
extern "C" {
MC_API int mc_dg_create(const mc_dg_desc*, mc_dg**) { return mc_fail(MC_EUNSUPPORTED, "todo"); }
MC_API int mc_dg_destroy(mc_dg*) { return 0; }
MC_API int64_t mc_dg_block_stride(const mc_dg*) { return 0; }
MC_API int64_t mc_dg_buffer_bytes(const mc_dg*) { return 0; }
MC_API int mc_dg_rhs(mc_dg*, const double*, double*, int, void*) { return 9; }
MC_API int mc_dg_rk_stage(mc_dg*, double*, const double*, double*, double, double, double, void*) { return 9; }
MC_API int mc_dg_ssprk3(mc_dg*, double*, double*, double, int, void*) { return 9; }
MC_API int mc_dg_ssprk3_host(mc_dg*, double*, double, int) { return 9; }
}
