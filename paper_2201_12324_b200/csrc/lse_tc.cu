// K2 placeholder (replaced by the tcgen05 kernel).
#include "otk_common.cuh"
namespace otk {
bool tc_available() { return false; }
int lse_tc_launch(const uint16_t *, const uint16_t *, int64_t, const uint16_t *, const uint16_t *,
                  int64_t, int, float, const float *, int, float *, cudaStream_t) {
  set_error("tcgen05 path not built");
  return OTK_ENOTSUP;
}
}  // namespace otk
