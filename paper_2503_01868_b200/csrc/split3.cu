// fp32 activations -> the K-concatenated bf16 operand of the split-bf16 fp32 GEMM (blas.py).
//
// Every fp32 x is exactly x0 + x1 + x2 with x0 = bf16(x), x1 = bf16(x - x0), x2 = bf16(x - x0 - x1)
// (the subtractions are exact in fp32). The fp32 projection A @ X runs as bf16 tensor-core GEMMs
// over these parts; the five small products share ONE GEMM whose B operand is the row
// concatenation [X1; X2; X0; X1; X0] (K' = 5K, the order of blas._PAIRS), and the leading
// product A0 @ X0 reads the last K rows of the same buffer. One HBM pass: 4 bytes in, 10 out per
// element (the eager version made eight elementwise / copy passes).
#include "common.cuh"
#include "internal.h"

namespace hy {
namespace {

__device__ __forceinline__ void split1(float x, __nv_bfloat16& a0, __nv_bfloat16& a1, __nv_bfloat16& a2) {
  a0 = __float2bfloat16_rn(x);
  const float r = x - __bfloat162float(a0);
  a1 = __float2bfloat16_rn(r);
  a2 = __float2bfloat16_rn(r - __bfloat162float(a1));
}

// x: (batch, K, N) fp32 rows; out: (batch, 5K, N) bf16. One thread per 8 consecutive elements
// of a row (two 16-byte loads, five 16-byte stores), grid-stride over all of them.
__global__ void split3_cat_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ out, long long batch,
                                  long long K, long long N) {
  const long long per_row = N / 8;
  const long long total = batch * K * per_row;
  const long long KN = K * N;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long row = i / per_row, c8 = (i - row * per_row) * 8;
    const long long b = row / K, k = row - b * K;
    const float4* src = reinterpret_cast<const float4*>(x + row * N + c8);
    const float4 v0 = __ldcs(src), v1 = __ldcs(src + 1);
    const float in[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
    __align__(16) __nv_bfloat16 p0[8], p1[8], p2[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) split1(in[e], p0[e], p1[e], p2[e]);
    __nv_bfloat16* o = out + b * 5 * KN + k * N + c8;
    const int4 w0 = *reinterpret_cast<const int4*>(p0), w1 = *reinterpret_cast<const int4*>(p1),
               w2 = *reinterpret_cast<const int4*>(p2);
    // [X1; X2; X0; X1; X0]
    __stcs(reinterpret_cast<int4*>(o), w1);
    __stcs(reinterpret_cast<int4*>(o + KN), w2);
    __stcs(reinterpret_cast<int4*>(o + 2 * KN), w0);
    __stcs(reinterpret_cast<int4*>(o + 3 * KN), w1);
    __stcs(reinterpret_cast<int4*>(o + 4 * KN), w0);
  }
}

// Unaligned / ragged N: one element per thread.
__global__ void split3_cat_scalar_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ out,
                                         long long batch, long long K, long long N) {
  const long long total = batch * K * N, KN = K * N;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = i / KN, r = i - b * KN;
    __nv_bfloat16 a0, a1, a2;
    split1(x[i], a0, a1, a2);
    __nv_bfloat16* o = out + b * 5 * KN + r;
    o[0] = a1;
    o[KN] = a2;
    o[2 * KN] = a0;
    o[3 * KN] = a1;
    o[4 * KN] = a0;
  }
}

}  // namespace
}  // namespace hy

using namespace hy;

extern "C" HY_API int hy_split3_cat(const float* x, void* out, long long batch, long long K, long long N,
                                    void* stream) {
  if (!x || !out) return fail(HY_ERR_INVALID, "null pointer argument");
  if (batch < 1 || K < 1 || N < 1) return fail(HY_ERR_INVALID, "sizes must be >= 1");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long grid_cap = static_cast<long long>(sms) * 8;  // 8 x 256-thread CTAs resident per SM
  auto* o = static_cast<__nv_bfloat16*>(out);
  if (N % 8 == 0 && aligned16(x) && aligned16(out)) {
    const long long work = batch * K * (N / 8);
    const long long grid = (work + 255) / 256 < grid_cap ? (work + 255) / 256 : grid_cap;
    split3_cat_kernel<<<static_cast<int>(grid), 256, 0, st>>>(x, o, batch, K, N);
  } else {
    const long long work = batch * K * N;
    const long long grid = (work + 255) / 256 < grid_cap ? (work + 255) / 256 : grid_cap;
    split3_cat_scalar_kernel<<<static_cast<int>(grid), 256, 0, st>>>(x, o, batch, K, N);
  }
  return check_launch("split3_cat_kernel");
}
