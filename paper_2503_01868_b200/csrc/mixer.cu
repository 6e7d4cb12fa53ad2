// Fused Hyena mixer: everything between the input projections and the output
// projection of hyena.py:162-186 in one HBM pass.
//
//   SE (inner lh <= 16, fp32 or bf16): se_mixer_kernel, CUDA cores
//   MR (inner lh <= 129, bf16):        tcgen05 two-stage kernel with in-kernel featurizers
//
// se_mixer_kernel: one CTA per (row tile of 2048 outputs, channel, batch). Raw
// projected q/k/v windows are staged with 16-byte cp.async copies (all in flight at once); the converter step
// forms u = feat_k * feat_v over [t0 - NI, t0 + 2048) in shared memory, then
// every thread produces 8 outputs y = feat_q * (h_inner conv u) from register
// sliding windows and stores them as 128-bit vectors. HBM traffic is the 3
// projected rows in and y out (16 B/token/channel at fp32).
#include "common.cuh"
#include "internal.h"

namespace hy {

constexpr int kMxThreads = 256;
constexpr int kMxV = 8;
constexpr int kMxTT = kMxThreads * kMxV;  // outputs per CTA

template <typename A, typename S, int NJ>
__device__ __forceinline__ void fir8_smem(A (&acc)[kMxV], const S* xs, const A* hs, int base) {
  A r[kMxV];
#pragma unroll
  for (int vv = 0; vv < kMxV; ++vv) r[vv] = static_cast<A>(xs[base + vv]);
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) {
    const A h = hs[jj];
#pragma unroll
    for (int vv = 0; vv < kMxV; ++vv) acc[vv] = fma(h, r[vv], acc[vv]);
#pragma unroll
    for (int vv = kMxV - 1; vv > 0; --vv) r[vv] = r[vv - 1];
    r[0] = static_cast<A>(xs[base - jj - 1]);
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}

// Stage row[s0, s0 + n) into xs (zeros outside [0, L)). vec: every 16-byte unit is issued as
// one asynchronous copy (all of the CTA's loads in flight at once, no register staging).
template <typename T>
__device__ __forceinline__ void stage_row(T* xs, const T* __restrict__ row, int s0, int n, int L, bool vec) {
  constexpr int VEC = Elem<T>::VEC;
  if (vec) {
    for (int i = threadIdx.x * VEC; i < n; i += blockDim.x * VEC) {
      const int t = s0 + i;
      const bool ok = t >= 0 && t < L;  // L % VEC == 0 and s0 % VEC == 0: whole units
      cp_async16(xs + i, ok ? row + t : row, ok);
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int t = s0 + i;
      xs[i] = (t >= 0 && t < L) ? row[t] : Elem<T>::from_a(0.f);
    }
  }
}

// NF: featurizer taps padded (8 or 16); NI: inner taps padded (8 or 16).
template <typename T, int NF, int NI>
__global__ void __launch_bounds__(kMxThreads, 4)
se_mixer_kernel(const T* __restrict__ proj, T* __restrict__ y, const float* __restrict__ feat_taps,
                int lhf, const float* __restrict__ inner_taps, const float* __restrict__ decay, int lh,
                int gs, int C, int L, int vec) {
  constexpr int KW = kMxTT + NI + NF + 8;  // raw k / v window
  constexpr int QW = kMxTT + NF + 8;       // raw q window
  constexpr int UW = kMxTT + NI;           // u window
  __shared__ __align__(16) T pk[KW], pv[KW], pq[QW];
  __shared__ __align__(16) float us[UW];
  __shared__ float hk[NF], hv[NF], hq[NF], hi[NI];

  const int c = blockIdx.y, b = blockIdx.z;
  const int t0 = blockIdx.x * kMxTT;
  const T* qrow = proj + (static_cast<size_t>(b) * 3 * C + c) * L;
  const T* krow = qrow + static_cast<size_t>(C) * L;
  const T* vrow = krow + static_cast<size_t>(C) * L;
  const int tid = threadIdx.x;
  const int tu = t0 - NI;           // u window origin
  const int sk = tu - NF - 8;       // raw k/v window origin
  const int sq = t0 - NF - 8;       // raw q window origin
  stage_row<T>(pk, krow, sk, KW, L, vec != 0);
  stage_row<T>(pv, vrow, sk, KW, L, vec != 0);
  stage_row<T>(pq, qrow, sq, QW, L, vec != 0);
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (tid < NF) {
    const bool ok = tid < lhf;
    hq[tid] = ok ? feat_taps[(static_cast<size_t>(0) * C + c) * lhf + tid] : 0.f;
    hk[tid] = ok ? feat_taps[(static_cast<size_t>(1) * C + c) * lhf + tid] : 0.f;
    hv[tid] = ok ? feat_taps[(static_cast<size_t>(2) * C + c) * lhf + tid] : 0.f;
  }
  if (tid < NI) {
    const int g = c / gs;
    float h = 0.f;
    if (tid < lh) {
      h = inner_taps[static_cast<size_t>(g) * lh + tid];
      if (decay) h *= exp2f(-decay[g] * static_cast<float>(tid));
    }
    hi[tid] = h;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  using S = T;
  // u = feat_k * feat_v over the u window, 8 consecutive times per unit
  for (int unit = tid; unit < UW / kMxV; unit += kMxThreads) {
    float fk[kMxV] = {}, fv[kMxV] = {};
    const int base = (tu + unit * kMxV) - sk;
    fir8_smem<float, S, NF>(fk, pk, hk, base);
    fir8_smem<float, S, NF>(fv, pv, hv, base);
#pragma unroll
    for (int vv = 0; vv < kMxV; ++vv) us[unit * kMxV + vv] = fk[vv] * fv[vv];
  }
  __syncthreads();
  float acc[kMxV] = {}, fq[kMxV] = {};
  fir8_smem<float, float, NI>(acc, us, hi, NI + tid * kMxV);
  fir8_smem<float, S, NF>(fq, pq, hq, t0 + tid * kMxV - sq);
#pragma unroll
  for (int vv = 0; vv < kMxV; ++vv) acc[vv] *= fq[vv];
  T* yrow = y + (static_cast<size_t>(b) * C + c) * L;
  const int t = t0 + tid * kMxV;
  constexpr int VEC = Elem<T>::VEC;
  if (vec && t + kMxV <= L) {
#pragma unroll
    for (int m = 0; m < kMxV; m += VEC) st_stream16(yrow + t + m, pack16<T>(acc + m));
  } else {
    for (int vv = 0; vv < kMxV; ++vv)
      if (t + vv < L) yrow[t + vv] = Elem<T>::from_a(acc[vv]);
  }
}

template <typename T, int NF, int NI>
static int launch_se(const void* proj, void* y, const float* ft, int lhf, const float* it, const float* dec,
                     int lh, int gs, int B, int C, int L, cudaStream_t st) {
  constexpr int VEC = Elem<T>::VEC;
  const bool vec = (L % VEC == 0) && aligned16(proj) && aligned16(y);
  dim3 grid((L + kMxTT - 1) / kMxTT, C, B);
  se_mixer_kernel<T, NF, NI><<<grid, kMxThreads, 0, st>>>(static_cast<const T*>(proj), static_cast<T*>(y),
                                                          ft, lhf, it, dec, lh, gs, C, L, vec ? 1 : 0);
  return check_launch("se_mixer_kernel");
}

template <typename T>
static int launch_se_dispatch(const void* proj, void* y, const float* ft, int lhf, const float* it,
                              const float* dec, int lh, int gs, int B, int C, int L, cudaStream_t st) {
  if (lhf <= 8 && lh <= 8) return launch_se<T, 8, 8>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
  if (lhf <= 8) return launch_se<T, 8, 16>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
  if (lh <= 8) return launch_se<T, 16, 8>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
  return launch_se<T, 16, 16>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
}

}  // namespace hy

using namespace hy;

extern "C" int hy_hyena_mixer_fwd(const void* proj, void* y, const void* feat_taps, const void* feat_pack,
                                  const void* hist, int lhf, const void* inner_taps, const float* inner_decay,
                                  int lh, int gs, int B, int C, int L, int dtype, void* stream) {
  if (!proj || !y || !feat_taps || !inner_taps) return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || lh < 1 || gs < 1 || lhf < 1)
    return fail(HY_ERR_INVALID, "sizes must be >= 1");
  if (C % gs != 0) return fail(HY_ERR_INVALID, "group_size %d does not divide channel count %d", gs, C);
  if (lhf > 16) return fail(HY_ERR_UNSUPPORTED, "featurizer length %d > 16", lhf);
  if (C > 65535 || B > 65535) return fail(HY_ERR_UNSUPPORTED, "grid limit");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float* ft = static_cast<const float*>(feat_taps);
  const float* it = static_cast<const float*>(inner_taps);
  if (dtype == HY_BF16 && lh <= 129 && L % 8 == 0 && aligned16(proj) && aligned16(y) && feat_pack)
    return mr_mixer_fwd(proj, y, ft, feat_pack, hist, lhf, it, inner_decay, lh, gs, B, C, L, stream);
  if (hist) return fail(HY_ERR_UNSUPPORTED, "projection history (context parallel) needs the tcgen05 mixer path");
  if (lh <= 16) {
    if (dtype == HY_F32) return launch_se_dispatch<float>(proj, y, ft, lhf, it, inner_decay, lh, gs, B, C, L, st);
    if (dtype == HY_BF16)
      return launch_se_dispatch<__nv_bfloat16>(proj, y, ft, lhf, it, inner_decay, lh, gs, B, C, L, st);
  }
  return fail(HY_ERR_UNSUPPORTED, "no fused mixer for dtype %d, lh %d (compose the unfused kernels)", dtype, lh);
}

// SE mixer only (CUDA cores), regardless of dtype routing; used by tests and the bf16 SE bench.
extern "C" int hy_se_mixer_fwd(const void* proj, void* y, const void* feat_taps, int lhf, const void* inner_taps,
                               const float* inner_decay, int lh, int gs, int B, int C, int L, int dtype,
                               void* stream) {
  if (!proj || !y || !feat_taps || !inner_taps) return fail(HY_ERR_INVALID, "null pointer argument");
  if (lh > 16 || lhf > 16) return fail(HY_ERR_UNSUPPORTED, "SE mixer needs lh, lhf <= 16");
  if (C % gs != 0) return fail(HY_ERR_INVALID, "group_size %d does not divide channel count %d", gs, C);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float* ft = static_cast<const float*>(feat_taps);
  const float* it = static_cast<const float*>(inner_taps);
  if (dtype == HY_F32) return launch_se_dispatch<float>(proj, y, ft, lhf, it, inner_decay, lh, gs, B, C, L, st);
  if (dtype == HY_BF16)
    return launch_se_dispatch<__nv_bfloat16>(proj, y, ft, lhf, it, inner_decay, lh, gs, B, C, L, st);
  return fail(HY_ERR_UNSUPPORTED, "SE mixer: fp32 / bf16 only");
}
