// attn_sm100.cu -- tcgen05 / TMEM path of Step 2 (placeholder until the kernel lands).
#include "internal.h"

namespace s2o {
bool tc_supported(const PassArgs&) { return false; }
cudaError_t launch_tc_pass(const PassArgs&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace s2o
