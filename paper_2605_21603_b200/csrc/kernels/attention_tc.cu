// Tensor-core causal prefill attention (placeholder until the tensor-core
// kernel lands): returning false routes attn_prefill to the SIMT kernel.
#include <cuda_bf16.h>

#include "opflow/device.hpp"

namespace opflow {

bool prefill_bf16_tc(const __nv_bfloat16*, __nv_bfloat16*, int64_t, int, int, int, int, float,
                     cudaStream_t) {
  return false;
}

}  // namespace opflow
