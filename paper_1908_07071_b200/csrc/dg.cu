// SIPG DG operator and B_DG (rows a3, a9) — implemented in the next milestone.
#include "device.cuh"

namespace lorpc {
int dg_apply(const lorpc_mesh*, const double*, double*, cudaStream_t) { return fail(LORPC_ERR_SIZE, "dg: not built"); }
int dg_diag_setup(lorpc_mesh*, cudaStream_t) { return fail(LORPC_ERR_SIZE, "dg: not built"); }
int dg_restrict_cg(const lorpc_mesh*, const double*, double*, cudaStream_t) { return fail(LORPC_ERR_SIZE, "dg: not built"); }
int dg_combine(const lorpc_mesh*, const double*, const double*, double*, cudaStream_t) { return fail(LORPC_ERR_SIZE, "dg: not built"); }
int dg_bface_points(const lorpc_mesh*, double*, cudaStream_t) { return fail(LORPC_ERR_SIZE, "dg: not built"); }
int dg_rhs_bc(const lorpc_mesh*, const double*, double*, cudaStream_t) { return fail(LORPC_ERR_SIZE, "dg: not built"); }
}  // namespace lorpc
