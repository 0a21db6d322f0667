#include "opflow/device.hpp"
namespace opflow {
int gemm_splitk_splits(int64_t, int64_t, int64_t, int) { return 1; }
size_t gemm_splitk_workspace(int64_t, int64_t, int64_t, int) { return 0; }
}  // namespace opflow
