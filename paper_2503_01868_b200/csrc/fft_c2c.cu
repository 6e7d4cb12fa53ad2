// Batched complex FFT (power-of-two length, natural order in and out), fp32 / fp64 complex.
//
// The local transform of the distributed FFT (cpsim.py:596-615: after the cross-rank DiF stages
// each rank transforms its slice) and the device form of the reference's fft / ifft helpers
// (fft.py:55-125; forward unnormalised, the 1/N of the inverse applied by the caller as fft.py).
// Radix-2 Stockham auto-sort stages (no bit reversal pass):
//     v0 = x[j], v1 = x[j + N/2] * exp(sign 2 pi i (j mod Ns) / (2 Ns))
//     y[(j / Ns) 2 Ns + j mod Ns] = v0 + v1,   y[... + Ns] = v0 - v1,     Ns = 1, 2, 4, ..., N/2
// Rows of up to SMALL_N points run all stages in one CTA in shared memory; longer rows run one
// stage per launch through a caller workspace (ping-pong). Twiddles by sincospi in the working
// precision (exact argument reduction).
#include "common.cuh"

namespace hy {
namespace c2c {

template <typename R> struct Cx;
template <> struct Cx<float> { using T = float2; };
template <> struct Cx<double> { using T = double2; };

__device__ __forceinline__ void sc(float a, float* s, float* c) { sincospif(a, s, c); }
__device__ __forceinline__ void sc(double a, double* s, double* c) { sincospi(a, s, c); }

template <typename R>
__device__ __forceinline__ void butterfly(const typename Cx<R>::T* x, typename Cx<R>::T* y, long long j, long long n,
                                          long long ns, R sign) {
  using T = typename Cx<R>::T;
  const long long k = j & (ns - 1);
  const T v0 = x[j], a = x[j + n / 2];
  R s, c;
  sc(sign * static_cast<R>(k) / static_cast<R>(ns), &s, &c);  // exp(sign * pi i k / ns)
  const T v1 = {a.x * c - a.y * s, a.x * s + a.y * c};
  const long long d = (j / ns) * 2 * ns + k;
  y[d] = {v0.x + v1.x, v0.y + v1.y};
  y[d + ns] = {v0.x - v1.x, v0.y - v1.y};
}

constexpr int THREADS = 512;

// one row per CTA, all log2(n) stages in shared memory (two buffers of n points)
template <typename R>
__global__ void __launch_bounds__(THREADS) fft_smem_kernel(const typename Cx<R>::T* __restrict__ in,
                                                           typename Cx<R>::T* __restrict__ out, int n, R sign) {
  using T = typename Cx<R>::T;
  extern __shared__ __align__(16) unsigned char raw[];
  T* a = reinterpret_cast<T*>(raw);
  T* b = a + n;
  const size_t row = static_cast<size_t>(blockIdx.x) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = in[row + i];
  __syncthreads();
  for (int ns = 1; ns < n; ns *= 2) {
    for (int j = threadIdx.x; j < n / 2; j += blockDim.x) butterfly<R>(a, b, j, n, ns, sign);
    __syncthreads();
    T* t = a;
    a = b;
    b = t;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[row + i] = a[i];
}

// one Stockham stage over every row (global memory)
template <typename R>
__global__ void fft_stage_kernel(const typename Cx<R>::T* __restrict__ x, typename Cx<R>::T* __restrict__ y,
                                 long long batch, long long n, long long ns, R sign) {
  const long long half = n / 2, total = batch * half;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = i / half, j = i - r * half;
    butterfly<R>(x + r * n, y + r * n, j, n, ns, sign);
  }
}

template <typename R>
constexpr long long small_n() {
  return 232448 / (2 * static_cast<long long>(sizeof(typename Cx<R>::T)));  // two buffers in 227 KB
}

template <typename R>
int run(const void* xin, void* yout, long long batch, long long n, int inverse, void* ws, cudaStream_t st) {
  using T = typename Cx<R>::T;
  const R sign = inverse ? R(1) : R(-1);
  const T* x = static_cast<const T*>(xin);
  T* y = static_cast<T*>(yout);
  long long sn = 1;
  while (sn * 2 <= small_n<R>()) sn *= 2;
  if (n <= sn) {
    const int smem = static_cast<int>(2 * n * sizeof(T));
    auto kern = fft_smem_kernel<R>;
    if (smem > 48 * 1024) {
      cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
      if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    }
    const int threads = n / 2 < THREADS ? static_cast<int>(n / 2 > 32 ? n / 2 : 32) : THREADS;
    for (long long b0 = 0; b0 < batch; b0 += 65535) {
      const long long nb = batch - b0 < 65535 ? batch - b0 : 65535;
      kern<<<static_cast<unsigned>(nb), threads, smem, st>>>(x + b0 * n, y + b0 * n, static_cast<int>(n), sign);
    }
    return check_launch("fft_smem_kernel");
  }
  // long rows: log2(n) stages, ping-pong between the workspace and the output; the stage count's
  // parity decides which buffer the first stage writes so the last one lands in the output
  T* w = static_cast<T*>(ws);
  int stages = 0;
  for (long long m = 1; m < n; m *= 2) ++stages;
  const T* src = x;
  T* dst = (stages & 1) ? y : w;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long work = batch * (n / 2);
  const long long grid = (work + 255) / 256 < 8LL * sms ? (work + 255) / 256 : 8LL * sms;
  for (long long ns = 1; ns < n; ns *= 2) {
    fft_stage_kernel<R><<<static_cast<int>(grid), 256, 0, st>>>(src, dst, batch, n, ns, sign);
    src = dst;
    dst = (dst == y) ? w : y;
  }
  return check_launch("fft_stage_kernel");
}

}  // namespace c2c
}  // namespace hy

using namespace hy;

extern "C" HY_API size_t hy_fft_c2c_workspace_size(long long batch, long long n, int dtype) {
  if (dtype == HY_F64) return n <= c2c::small_n<double>() ? 0 : static_cast<size_t>(batch * n) * 16;
  return n <= c2c::small_n<float>() ? 0 : static_cast<size_t>(batch * n) * 8;
}

extern "C" HY_API int hy_fft_c2c(const void* x, void* y, long long batch, long long n, int inverse, int dtype,
                                 void* ws, size_t ws_bytes, void* stream) {
  if (!x || !y) return fail(HY_ERR_INVALID, "null pointer argument");
  if (batch < 1 || n < 1 || (n & (n - 1)) != 0) return fail(HY_ERR_INVALID, "length %lld is not a power of two", n);
  if (dtype != HY_F32 && dtype != HY_F64) return fail(HY_ERR_UNSUPPORTED, "hy_fft_c2c: complex64 / complex128 only");
  if (x == y && n > 1) return fail(HY_ERR_INVALID, "hy_fft_c2c is out of place");
  if (ws_bytes < hy_fft_c2c_workspace_size(batch, n, dtype) || (ws_bytes && !ws && n > 1))
    return fail(HY_ERR_INVALID, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n == 1) {
    const cudaError_t e = cudaMemcpyAsync(y, x, static_cast<size_t>(batch) * (dtype == HY_F64 ? 16 : 8),
                                          cudaMemcpyDeviceToDevice, st);
    return e == cudaSuccess ? HY_OK : fail(HY_ERR_CUDA, "copy: %s", cudaGetErrorString(e));
  }
  if (dtype == HY_F64) return c2c::run<double>(x, y, batch, n, inverse, ws, st);
  return c2c::run<float>(x, y, batch, n, inverse, ws, st);
}
