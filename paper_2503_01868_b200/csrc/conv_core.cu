#include <cstdlib>
// CUDA-core causal FIR kernels (sm_100a):
//   * causal_conv_kernel  — direct_causal_conv / gated two-stage semantics for any
//     filter length (core.py:212-226, blockconv.py:182-220), fp32 / bf16 / fp64.
//   * se_mixer_kernel     — the fused SE mixer: featurizer FIRs on the projected
//     q/k/v rows + gated inner FIR (hyena.py:122-126 + 162-186), one HBM pass.
//   * halo_correction     — p2p_conv_overlapped's correction conv (cpsim.py:498-510).
//
// Data movement: each CTA stages a time window of its row in shared memory with
// 128-bit coalesced global loads (ld.global.nc.L1::no_allocate.v4), taps are
// staged once per CTA and broadcast, and every thread produces V consecutive
// outputs from a register sliding window (one shared-memory load per tap per
// thread, V FMAs per load). Outputs leave as 128-bit stores.
#include <cstdarg>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace hy {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(HY_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return HY_OK;
}

constexpr int kThreads = 128;  // threads per CTA
constexpr int kV = 8;          // consecutive outputs per thread
constexpr int kTT = kThreads * kV;  // outputs per CTA (time tile)
constexpr int kTJ = 256;       // tap tile for long filters

// Fill xs[i] = u(s0 + i), i in [0, n), with u = v (or v*k) and zero outside [0, L).
// s0 and n are multiples of VEC; with vec==true rows are 16-byte aligned and
// L % VEC == 0, so each vector lies entirely inside or outside [0, L).
template <typename T, bool GK>
__device__ __forceinline__ void load_window(typename Elem<T>::A* xs, const T* __restrict__ vrow,
                                            const T* __restrict__ krow, int s0, int n, int L,
                                            bool vec) {
  using A = typename Elem<T>::A;
  constexpr int VEC = Elem<T>::VEC;
  if (vec) {
    for (int i = threadIdx.x * VEC; i < n; i += blockDim.x * VEC) {
      const int t = s0 + i;
      A vals[VEC];
      if (t >= 0 && t < L) {
        unpack16<T>(ld_stream16(vrow + t), vals);
        if (GK) {
          A kv[VEC];
          unpack16<T>(ld_stream16(krow + t), kv);
#pragma unroll
          for (int m = 0; m < VEC; ++m) vals[m] *= kv[m];
        }
      } else {
#pragma unroll
        for (int m = 0; m < VEC; ++m) vals[m] = A(0);
      }
      // 16-byte shared stores (xs is 16-byte aligned, i % VEC == 0)
      constexpr int PER16 = 16 / sizeof(A);
#pragma unroll
      for (int m = 0; m < VEC; m += PER16)
        *reinterpret_cast<int4*>(xs + i + m) = *reinterpret_cast<const int4*>(vals + m);
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int t = s0 + i;
      A val = A(0);
      if (t >= 0 && t < L) {
        val = Elem<T>::to_a(vrow[t]);
        if (GK) val *= Elem<T>::to_a(krow[t]);
      }
      xs[i] = val;
    }
  }
}

__host__ __device__ constexpr int floor_to(int a, int m) { return (a >= 0 ? a / m : -((-a + m - 1) / m)) * m; }
__host__ __device__ constexpr int ceil_to(int a, int m) { return ((a + m - 1) / m) * m; }

// acc[vv] += sum_{jj < nj} hs[jj] * xs[base + vv - jj] with a register sliding window.
template <typename A, int NJ>
__device__ __forceinline__ void fir_accumulate(A (&acc)[kV], const A* xs, const A* hs, int base,
                                               int nj) {
  A r[kV];
#pragma unroll
  for (int vv = 0; vv < kV; ++vv) r[vv] = xs[base + vv];
  if (NJ > 0) {
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) {
      const A h = hs[jj];
#pragma unroll
      for (int vv = 0; vv < kV; ++vv) acc[vv] = fma(h, r[vv], acc[vv]);
#pragma unroll
      for (int vv = kV - 1; vv > 0; --vv) r[vv] = r[vv - 1];
      r[0] = xs[base - jj - 1];
    }
  } else {
#pragma unroll 4
    for (int jj = 0; jj < nj; ++jj) {
      const A h = hs[jj];
#pragma unroll
      for (int vv = 0; vv < kV; ++vv) acc[vv] = fma(h, r[vv], acc[vv]);
#pragma unroll
      for (int vv = kV - 1; vv > 0; --vv) r[vv] = r[vv - 1];
      r[0] = xs[base - jj - 1];
    }
  }
}

// Store V outputs (optionally gated by q) at t = t0 + tid*V.
template <typename T, bool GQ>
__device__ __forceinline__ void store_outputs(typename Elem<T>::A (&acc)[kV], const T* __restrict__ qrow,
                                              T* __restrict__ yrow, int t, int L, bool vec) {
  using A = typename Elem<T>::A;
  constexpr int VEC = Elem<T>::VEC;
  if (vec && t + kV <= L) {
#pragma unroll
    for (int m = 0; m < kV; m += VEC) {
      if (GQ) {
        A qv[VEC];
        unpack16<T>(ld_stream16(qrow + t + m), qv);
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[m + e] *= qv[e];
      }
      st_stream16(yrow + t + m, pack16<T>(acc + m));
    }
  } else {
#pragma unroll
    for (int vv = 0; vv < kV; ++vv) {
      if (t + vv < L) {
        A o = acc[vv];
        if (GQ) o *= Elem<T>::to_a(qrow[t + vv]);
        yrow[t + vv] = Elem<T>::from_a(o);
      }
    }
  }
}

// y = [q *] conv([k *] v). NJ > 0: single tap tile with taps zero-padded to NJ.
template <typename T, bool GK, bool GQ, int NJ>
__global__ void __launch_bounds__(kThreads)
causal_conv_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                   T* __restrict__ y, const typename Elem<T>::A* __restrict__ taps, int C, int L,
                   int lh, int gs, int vec) {
  using A = typename Elem<T>::A;
  constexpr int VEC = Elem<T>::VEC;
  constexpr int TJ = NJ > 0 ? NJ : kTJ;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  A* hs = reinterpret_cast<A*>(smem_raw);         // [TJ]
  A* xs = hs + ceil_to(TJ, 16 / sizeof(A) * 2);   // window, 16B aligned

  const int c = blockIdx.y, b = blockIdx.z;
  const size_t row = (static_cast<size_t>(b) * C + c) * L;
  const int g = c / gs;
  const int t0 = blockIdx.x * kTT;
  const int tl = threadIdx.x * kV;  // local output offset

  A acc[kV];
#pragma unroll
  for (int vv = 0; vv < kV; ++vv) acc[vv] = A(0);

  for (int j0 = 0; j0 < lh; j0 += TJ) {
    const int nj = NJ > 0 ? NJ : min(TJ, lh - j0);
    for (int i = threadIdx.x; i < TJ; i += blockDim.x)
      hs[i] = (j0 + i < lh && i < nj) ? taps[static_cast<size_t>(g) * lh + j0 + i] : A(0);
    const int s0 = floor_to(t0 - j0 - nj + 1, VEC);
    const int n = ceil_to(t0 + kTT - j0 - s0, VEC);
    load_window<T, GK>(xs, v + row, GK ? k + row : nullptr, s0, n, L, vec != 0);
    __syncthreads();
    fir_accumulate<A, NJ>(acc, xs, hs, t0 + tl - j0 - s0, nj);
    __syncthreads();
  }
  store_outputs<T, GQ>(acc, GQ ? q + row : nullptr, y + row, t0 + tl, L, vec != 0);
}

template <typename T, bool GK, bool GQ, int NJ>
static int launch_conv_t(const void* q, const void* k, const void* v, void* y, const void* taps, int B,
                         int C, int L, int lh, int gs, cudaStream_t st) {
  using A = typename Elem<T>::A;
  constexpr int VEC = Elem<T>::VEC;
  constexpr int TJ = NJ > 0 ? NJ : kTJ;
  const bool vec = (L % VEC == 0) && aligned16(v) && aligned16(y) && (!GK || aligned16(k)) &&
                   (!GQ || aligned16(q));
  const size_t win = ceil_to(kTT + TJ + 2 * VEC, VEC);
  const size_t smem = (ceil_to(TJ, 16 / sizeof(A) * 2) + win) * sizeof(A);
  dim3 grid((L + kTT - 1) / kTT, C, B);
  causal_conv_kernel<T, GK, GQ, NJ><<<grid, kThreads, smem, st>>>(
      static_cast<const T*>(q), static_cast<const T*>(k), static_cast<const T*>(v), static_cast<T*>(y),
      static_cast<const A*>(taps), C, L, lh, gs, vec ? 1 : 0);
  return check_launch("causal_conv_kernel");
}

template <typename T, bool GK, bool GQ>
static int launch_conv_nj(const void* q, const void* k, const void* v, void* y, const void* taps, int B,
                          int C, int L, int lh, int gs, cudaStream_t st) {
  // Taps are read as a (n_groups, lh) matrix; the NJ variants zero-pad the tile.
  if (lh <= 4) return launch_conv_t<T, GK, GQ, 4>(q, k, v, y, taps, B, C, L, lh, gs, st);
  if (lh <= 8) return launch_conv_t<T, GK, GQ, 8>(q, k, v, y, taps, B, C, L, lh, gs, st);
  if (lh <= 16) return launch_conv_t<T, GK, GQ, 16>(q, k, v, y, taps, B, C, L, lh, gs, st);
  if (lh <= 32) return launch_conv_t<T, GK, GQ, 32>(q, k, v, y, taps, B, C, L, lh, gs, st);
  return launch_conv_t<T, GK, GQ, 0>(q, k, v, y, taps, B, C, L, lh, gs, st);
}

template <typename T>
static int launch_conv_gates(const void* q, const void* k, const void* v, void* y, const void* taps,
                             int B, int C, int L, int lh, int gs, cudaStream_t st) {
  if (q && k) return launch_conv_nj<T, true, true>(q, k, v, y, taps, B, C, L, lh, gs, st);
  if (k) return launch_conv_nj<T, true, false>(q, k, v, y, taps, B, C, L, lh, gs, st);
  if (q) return launch_conv_nj<T, false, true>(q, k, v, y, taps, B, C, L, lh, gs, st);
  return launch_conv_nj<T, false, false>(q, k, v, y, taps, B, C, L, lh, gs, st);
}

static int check_common(const void* v, void* y, const void* taps, int B, int C, int L, int lh, int gs,
                        int dtype) {
  if (!v || !y || !taps) return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || lh < 1 || gs < 1)
    return fail(HY_ERR_INVALID, "sizes must be >= 1 (B=%d C=%d L=%d lh=%d gs=%d)", B, C, L, lh, gs);
  if (C % gs != 0) return fail(HY_ERR_INVALID, "group_size %d does not divide channel count %d", gs, C);
  if (C > 65535 || B > 65535) return fail(HY_ERR_UNSUPPORTED, "grid limit: C and B must be <= 65535");
  if (dtype != HY_F32 && dtype != HY_BF16 && dtype != HY_F64)
    return fail(HY_ERR_INVALID, "unknown dtype %d", dtype);
  return HY_OK;
}

// Overlap correction: y[t] += sum_{j=t+1}^{lh-1} h[j] * halo[H + t - j], t < H.
template <typename T>
__global__ void halo_correction_kernel(const T* __restrict__ halo, T* __restrict__ y,
                                       const typename Elem<T>::A* __restrict__ taps, int C, int L,
                                       int lh, int gs) {
  using A = typename Elem<T>::A;
  const int H = lh - 1;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y, b = blockIdx.z;
  if (t >= H || t >= L) return;
  const A* h = taps + static_cast<size_t>(c / gs) * lh;
  const T* hr = halo + (static_cast<size_t>(b) * C + c) * H;
  A acc = A(0);
  for (int j = t + 1; j < lh; ++j) acc = fma(h[j], Elem<T>::to_a(hr[H + t - j]), acc);
  T* yr = y + (static_cast<size_t>(b) * C + c) * L;
  yr[t] = Elem<T>::from_a(Elem<T>::to_a(yr[t]) + acc);
}

}  // namespace hy

using namespace hy;

extern "C" {

int hy_version(void) { return 100; }

const char* hy_last_error(void) { return g_last_error.c_str(); }

int hy_gated_conv_fwd(const void* q, const void* k, const void* v, void* y, const void* taps, int B,
                      int C, int L, int lh, int gs, int dtype, void* stream) {
  int s = check_common(v, y, taps, B, C, L, lh, gs, dtype);
  if (s != HY_OK) return s;
  if (fir_stream_eligible(q, k, v, y, lh, L, dtype) && !getenv("HY_FIR_TILED") &&
      static_cast<long long>(B) * C * ((L + 255) / 256) < 0x7fffffffLL)
    return fir_stream_fwd(q, k, v, y, static_cast<const float*>(taps), B, C, L, lh, gs, dtype, stream);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (dtype) {
    case HY_F32: return launch_conv_gates<float>(q, k, v, y, taps, B, C, L, lh, gs, st);
    case HY_BF16: return launch_conv_gates<__nv_bfloat16>(q, k, v, y, taps, B, C, L, lh, gs, st);
    default: return launch_conv_gates<double>(q, k, v, y, taps, B, C, L, lh, gs, st);
  }
}

int hy_causal_conv_fwd(const void* x, void* y, const void* taps, int B, int C, int L, int lh, int gs,
                       int dtype, void* stream) {
  return hy_gated_conv_fwd(nullptr, nullptr, x, y, taps, B, C, L, lh, gs, dtype, stream);
}

int hy_halo_correction_fwd(const void* halo, void* y, const void* taps, int B, int C, int L, int lh,
                           int gs, int dtype, void* stream) {
  int s = check_common(halo, y, taps, B, C, L, lh, gs, dtype);
  if (s != HY_OK) return s;
  if (lh < 2) return HY_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  dim3 grid((lh - 1 + 127) / 128, C, B);
  switch (dtype) {
    case HY_F32:
      halo_correction_kernel<float><<<grid, 128, 0, st>>>(static_cast<const float*>(halo),
                                                          static_cast<float*>(y),
                                                          static_cast<const float*>(taps), C, L, lh, gs);
      break;
    case HY_BF16:
      halo_correction_kernel<__nv_bfloat16><<<grid, 128, 0, st>>>(
          static_cast<const __nv_bfloat16*>(halo), static_cast<__nv_bfloat16*>(y),
          static_cast<const float*>(taps), C, L, lh, gs);
      break;
    default:
      halo_correction_kernel<double><<<grid, 128, 0, st>>>(static_cast<const double*>(halo),
                                                           static_cast<double*>(y),
                                                           static_cast<const double*>(taps), C, L, lh, gs);
  }
  return check_launch("halo_correction_kernel");
}

}  // extern "C"
