// Gate multiply out = a * b over contiguous rows (the LI context-parallel layer's q gate on the
// all-to-all's returned slab, hyena.py:186 `q * conv_out` / cpsim.py:336-375 after the return
// round): one streaming pass, 16-byte vectors, fp32 arithmetic, bf16 / fp32 storage.
#include "common.cuh"

namespace hy {
namespace {

template <typename T>
__global__ void gate_mul_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out, long long n) {
  using A = typename Elem<T>::A;
  constexpr int V = Elem<T>::VEC;
  const long long nv = n / V;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    A x[V], y[V];
    unpack16<T>(ld_stream16(a + i * V), x);
    unpack16<T>(ld_stream16(b + i * V), y);
#pragma unroll
    for (int e = 0; e < V; ++e) x[e] *= y[e];
    st_stream16(out + i * V, pack16<T>(x));
  }
  // ragged tail (n % V elements) by the first threads
  const long long t = nv * V + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (blockIdx.x == 0 && t < n) out[t] = Elem<T>::from_a(Elem<T>::to_a(a[t]) * Elem<T>::to_a(b[t]));
}

template <typename T>
int launch(const void* a, const void* b, void* out, long long n, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long work = n / Elem<T>::VEC + 1;
  const long long cap = 8LL * sms;
  const long long grid = (work + 255) / 256 < cap ? (work + 255) / 256 : cap;
  gate_mul_kernel<T><<<static_cast<int>(grid), 256, 0, st>>>(static_cast<const T*>(a), static_cast<const T*>(b),
                                                             static_cast<T*>(out), n);
  return check_launch("gate_mul_kernel");
}

}  // namespace
}  // namespace hy

using namespace hy;

extern "C" HY_API int hy_gate_mul(const void* a, const void* b, void* out, long long n, int dtype, void* stream) {
  if (!a || !b || !out) return fail(HY_ERR_INVALID, "null pointer argument");
  if (n < 0) return fail(HY_ERR_INVALID, "negative length");
  if (n == 0) return HY_OK;
  if (!aligned16(a) || !aligned16(b) || !aligned16(out))
    return fail(HY_ERR_UNSUPPORTED, "hy_gate_mul needs 16-byte aligned tensors");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == HY_BF16) return launch<__nv_bfloat16>(a, b, out, n, st);
  if (dtype == HY_F32) return launch<float>(a, b, out, n, st);
  if (dtype == HY_F64) return launch<double>(a, b, out, n, st);
  return fail(HY_ERR_UNSUPPORTED, "hy_gate_mul: unknown dtype %d", dtype);
}
