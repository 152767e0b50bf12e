// conv_tc.cu -- tcgen05/TMEM TF32 implicit-GEMM 3x3 conv (placeholder until implemented).
#include "common.cuh"

namespace ld {
bool tc_conv_available() { return false; }
cudaError_t tc_conv_prepare() { return cudaSuccess; }
size_t tc_weight_floats(int ci, int co_pad) { return (size_t)9 * ci * co_pad; }
void tc_pack_weights(const float* Wt, int ci, int co_pad, float* dst) {
  for (size_t i = 0; i < (size_t)9 * ci * co_pad; ++i) dst[i] = Wt[i];
}
cudaError_t launch_conv_tc(const float*, int, int, const float*, const float*, int, int, int, int, float*, float*,
                           cudaStream_t) {
  return cudaErrorNotSupported;
}
}  // namespace ld
