// FFT causal convolution (fft.py:128-145) fused with the LI gates — placeholder
// until the sm_100a FFT kernels land; reports HY_ERR_UNSUPPORTED.
#include "common.cuh"

using namespace hy;

extern "C" size_t hy_fft_conv_workspace_size(int B, int C, int L, int lh, int gs, int dtype) {
  (void)B, (void)C, (void)L, (void)lh, (void)gs, (void)dtype;
  return 0;
}

extern "C" int hy_fft_conv_fwd(const void* q, const void* k, const void* v, void* y, const void* taps, int B,
                               int C, int L, int lh, int gs, int dtype, void* ws, size_t ws_bytes,
                               void* stream) {
  (void)q, (void)k, (void)v, (void)y, (void)taps, (void)B, (void)C, (void)L, (void)lh, (void)gs, (void)dtype;
  (void)ws, (void)ws_bytes, (void)stream;
  return fail(HY_ERR_UNSUPPORTED, "hy_fft_conv_fwd: not built yet");
}
