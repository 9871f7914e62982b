// tcgen05 int8 contraction (placeholder until the tensor path lands).
#include "fc_internal.cuh"

namespace fcb {

int level_prepare_tc(Ctx* c, Level& L) {
  (void)L;
  return set_error(c, FC_ERR_STATE, "tensor path not available");
}

int scan_tc(Ctx* c, Level& L, int64_t M, uint64_t* d_keys) {
  (void)L; (void)M; (void)d_keys;
  return set_error(c, FC_ERR_STATE, "tensor path not available");
}

}  // namespace fcb
