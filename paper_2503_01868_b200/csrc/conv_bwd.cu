// Adjoints of the causal FIR (core.py:245-268), CUDA cores, fp32 / bf16 (fp32 accumulate) / fp64:
//   dx[t]    = sum_j h[j] dy[t + j]                       (anti-causal FIR, causal_conv_input_grad)
//   dh[g][j] = sum_{c in g} sum_{b, t} dy[t] x[t - j]     (lag correlation, causal_conv_taps_grad)
//
// causal_conv_bwd_kernel: one CTA per (time split, channel, batch) walks its 1024-step tiles of
// the row. Per tile it stages the dy window [t0, t0 + 1024 + lh) and the x window
// [t0 - lh + 1, t0 + 1024) in shared memory with 128-bit loads, then
//   * dx: every thread produces 8 consecutive outputs from a register sliding window of dy;
//   * dh: work items (4 consecutive lags x one time segment) slide a 4-sample window of x
//     against dy (two shared loads per 4 FMAs); per-item partials land in a [segment][lag]
//     shared array and are summed in a fixed order, so the result is deterministic.
// The CTA's lag sums leave as one partial row per (batch, split, channel) in a caller
// workspace; conv_taps_reduce_kernel sums partials over batch, splits and the group's
// channels in fp64 (the reference's two-pass reduce, blockconv.py:246-262).
#include "common.cuh"

namespace hy {

constexpr int kBT = 128;           // threads per CTA
constexpr int kBV = 8;             // dx outputs per thread
constexpr int kBTT = kBT * kBV;    // steps per tile
constexpr int kBwdMaxLh = 2048;
constexpr int kBwdTargetCtas = 148 * 8 * 4;

__host__ __device__ constexpr int bceil_to(int a, int m) { return ((a + m - 1) / m) * m; }
__host__ __device__ constexpr int bfloor_to(int a, int m) { return (a >= 0 ? a / m : -((-a + m - 1) / m)) * m; }

static int bwd_nsplit(int B, int C, int L) {
  const int ntiles = (L + kBTT - 1) / kBTT;
  long long rows = static_cast<long long>(B) * C;
  int ns = static_cast<int>((kBwdTargetCtas + rows - 1) / rows);
  if (ns < 1) ns = 1;
  if (ns > ntiles) ns = ntiles;
  return ns;
}

// dtaps work items are (8 consecutive lags) x (one time segment of a tile); nseg segments
// per tile so that the items fill the CTA (segments are multiples of 8 steps).
__host__ __device__ inline int bwd_nseg(int lh) {
  const int no = (lh + 7) / 8;
  int ns = kBT / no;
  if (ns < 1) ns = 1;
  while (kBTT % (8 * ns) != 0) --ns;
  return ns;
}
__host__ __device__ inline int bwd_lhp(int lh) { return (lh + 7) / 8 * 8; }

// xs[i] = row(s0 + i), zeros outside [0, L); s0, n multiples of VEC when vec.
template <typename T>
__device__ __forceinline__ void stage(typename Elem<T>::A* xs, const T* __restrict__ row, int s0, int n, int L,
                                      bool vec) {
  using A = typename Elem<T>::A;
  constexpr int VEC = Elem<T>::VEC;
  if (vec) {
    for (int i = threadIdx.x * VEC; i < n; i += blockDim.x * VEC) {
      const int t = s0 + i;
      A vals[VEC];
      if (t >= 0 && t < L) {
        unpack16<T>(ld_stream16(row + t), vals);
      } else {
#pragma unroll
        for (int m = 0; m < VEC; ++m) vals[m] = A(0);
      }
      constexpr int PER16 = 16 / sizeof(A);
#pragma unroll
      for (int m = 0; m < VEC; m += PER16)
        *reinterpret_cast<int4*>(xs + i + m) = *reinterpret_cast<const int4*>(vals + m);
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int t = s0 + i;
      xs[i] = (t >= 0 && t < L) ? Elem<T>::to_a(row[t]) : A(0);
    }
  }
}

// r[0..N) = p[0..N) from 16-byte aligned shared memory with 16-byte loads.
template <int N>
__device__ __forceinline__ void lds_vec(float (&r)[N], const float* p) {
#pragma unroll
  for (int e = 0; e < N; e += 4) {
    const float4 v = *reinterpret_cast<const float4*>(p + e);
    r[e] = v.x, r[e + 1] = v.y, r[e + 2] = v.z, r[e + 3] = v.w;
  }
}
template <int N>
__device__ __forceinline__ void lds_vec(double (&r)[N], const double* p) {
#pragma unroll
  for (int e = 0; e < N; e += 2) {
    const double2 v = *reinterpret_cast<const double2*>(p + e);
    r[e] = v.x, r[e + 1] = v.y;
  }
}

template <typename T, bool DX, bool DT>
__global__ void __launch_bounds__(kBT)
causal_conv_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ x, T* __restrict__ dx,
                       const typename Elem<T>::A* __restrict__ taps, typename Elem<T>::A* __restrict__ part,
                       int C, int L, int lh, int gs, int nsplit, int vec) {
  using A = typename Elem<T>::A;
  constexpr int VEC = Elem<T>::VEC;
  constexpr int AL = 16 / sizeof(A) * 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nseg = bwd_nseg(lh), lhp = bwd_lhp(lh);
  const int wdy = kBTT + lhp + 16;
  const int wx = kBTT + lhp + 16;
  A* hs = reinterpret_cast<A*>(smem_raw);        // [lhp], zero padded
  A* dys = hs + bceil_to(lhp, AL);               // dy window: dys[i] = dy[t0 + i]
  A* xs = dys + bceil_to(wdy, AL);               // x window:  xs[i] = x[sx + i], sx = t0 - lhp - 8
  A* ps = xs + bceil_to(wx, AL);                 // [nseg][lhp] item partials, accumulated over tiles

  const int split = blockIdx.x, c = blockIdx.y, b = blockIdx.z;
  const size_t row = (static_cast<size_t>(b) * C + c) * L;
  const int ntiles = (L + kBTT - 1) / kBTT;
  const int tps = (ntiles + nsplit - 1) / nsplit;
  const int tile0 = split * tps, tile1 = min(ntiles, tile0 + tps);
  if (DX)
    for (int i = threadIdx.x; i < lhp; i += blockDim.x)
      hs[i] = i < lh ? taps[static_cast<size_t>(c / gs) * lh + i] : A(0);
  const int no = lhp / 8;
  const int seg_len = kBTT / nseg;
  if (DT)
    for (int i = threadIdx.x; i < nseg * lhp; i += blockDim.x) ps[i] = A(0);

  for (int tile = tile0; tile < tile1; ++tile) {
    const int t0 = tile * kBTT;
    const int sx = t0 - lhp - 8;  // multiple of 8: 16-byte aligned 4-wide reads below
    stage<T>(dys, dy + row, t0, wdy, L, vec != 0);
    if (DT) stage<T>(xs, x + row, sx, wx, L, vec != 0);
    __syncthreads();
    if (DX) {
      // dx[t0 + tl + v] = sum_j h[j] dy[t0 + tl + v + j], 8 taps per block from 16 window values
      const int tl = threadIdx.x * kBV;
      A acc[kBV];
#pragma unroll
      for (int v = 0; v < kBV; ++v) acc[v] = A(0);
      for (int j0 = 0; j0 < lhp; j0 += 8) {
        A r[16], h[8];
        lds_vec(r, dys + tl + j0);
        lds_vec(h, hs + j0);
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
#pragma unroll
          for (int v = 0; v < kBV; ++v) acc[v] = fma(h[jj], r[v + jj], acc[v]);
      }
      const int t = t0 + tl;
      T* drow = dx + row;
      if (vec && t + kBV <= L) {
#pragma unroll
        for (int m = 0; m < kBV; m += VEC) st_stream16(drow + t + m, pack16<T>(acc + m));
      } else {
#pragma unroll
        for (int v = 0; v < kBV; ++v)
          if (t + v < L) drow[t + v] = Elem<T>::from_a(acc[v]);
      }
    }
    if (DT) {
      // item (lag octet o, segment s): a[m] += sum_{i in seg} dy[t0+i] x[t0+i-8o-m], m < 8,
      // 8 steps at a time from the aligned x values [i - 8o - 8, i - 8o + 8)
      for (int w = threadIdx.x; w < no * nseg; w += blockDim.x) {
        const int o = w % no, s = w / no;
        const int ta = s * seg_len;
        A a[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) a[m] = A(0);
        const int xo = t0 - sx - 8 * o;  // x[t0 + i - 8o + e] = xs[xo + i + e]
        for (int i = ta; i < ta + seg_len; i += 8) {
          A d[8], xw[16];
          lds_vec(d, dys + i);
          lds_vec(xw, xs + xo + i - 8);  // x[t0+i-8o-8 .. +8)
#pragma unroll
          for (int e = 0; e < 8; ++e)
#pragma unroll
            for (int m = 0; m < 8; ++m) a[m] = fma(d[e], xw[8 + e - m], a[m]);
        }
        A* pp = ps + s * lhp + 8 * o;
#pragma unroll
        for (int m = 0; m < 8; ++m) pp[m] += a[m];
      }
    }
    __syncthreads();
  }
  if (DT) {
    A* out = part + ((static_cast<size_t>(b) * nsplit + split) * C + c) * lh;
    for (int j = threadIdx.x; j < lh; j += blockDim.x) {
      A sum = A(0);
      for (int s2 = 0; s2 < nseg; ++s2) sum += ps[s2 * lhp + j];
      out[j] = sum;
    }
  }
}

// dtaps[g][j] = sum over partial rows p and channels c of group g of part[p][c][j] (fp64 sum).
template <typename A>
__global__ void conv_taps_reduce_kernel(const A* __restrict__ part, A* __restrict__ dtaps, int P, int C, int lh,
                                        int gs) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int g = blockIdx.y;
  if (j >= lh) return;
  double s = 0.0;
  for (int p = 0; p < P; ++p)
    for (int c = g * gs; c < (g + 1) * gs; ++c) s += static_cast<double>(part[(static_cast<size_t>(p) * C + c) * lh + j]);
  dtaps[static_cast<size_t>(g) * lh + j] = static_cast<A>(s);
}

static size_t bwd_smem_bytes(int lh, size_t asz) {
  const int al = static_cast<int>(16 / asz * 2);
  const int lhp = bwd_lhp(lh);
  const int w = kBTT + lhp + 16;
  return (static_cast<size_t>(bceil_to(lhp, al)) + 2 * bceil_to(w, al) + bceil_to(bwd_nseg(lh) * lhp, al)) * asz;
}

template <typename T, bool DX, bool DT>
static int launch_bwd_t(const void* dy, const void* x, void* dx, const void* taps, void* part, int B, int C, int L,
                        int lh, int gs, int nsplit, cudaStream_t st) {
  using A = typename Elem<T>::A;
  constexpr int VEC = Elem<T>::VEC;
  const bool vec = (L % VEC == 0) && aligned16(dy) && (!DX || aligned16(dx)) && (!DT || aligned16(x));
  const size_t smem = bwd_smem_bytes(lh, sizeof(A));
  auto kern = causal_conv_bwd_kernel<T, DX, DT>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  dim3 grid(nsplit, C, B);
  kern<<<grid, kBT, smem, st>>>(static_cast<const T*>(dy), static_cast<const T*>(x), static_cast<T*>(dx),
                                static_cast<const A*>(taps), static_cast<A*>(part), C, L, lh, gs, nsplit,
                                vec ? 1 : 0);
  return check_launch("causal_conv_bwd_kernel");
}

template <typename T>
static int launch_bwd(const void* dy, const void* x, void* dx, void* dtaps, const void* taps, int B, int C, int L,
                      int lh, int gs, void* ws, cudaStream_t st) {
  using A = typename Elem<T>::A;
  const int nsplit = bwd_nsplit(B, C, L);
  int s;
  if (dx && dtaps) s = launch_bwd_t<T, true, true>(dy, x, dx, taps, ws, B, C, L, lh, gs, nsplit, st);
  else if (dx) s = launch_bwd_t<T, true, false>(dy, x, dx, taps, ws, B, C, L, lh, gs, nsplit, st);
  else s = launch_bwd_t<T, false, true>(dy, x, dx, taps, ws, B, C, L, lh, gs, nsplit, st);
  if (s != HY_OK || !dtaps) return s;
  dim3 grid((lh + 127) / 128, C / gs);
  conv_taps_reduce_kernel<A><<<grid, 128, 0, st>>>(static_cast<const A*>(ws), static_cast<A*>(dtaps), B * nsplit, C,
                                                   lh, gs);
  return check_launch("conv_taps_reduce_kernel");
}

}  // namespace hy

using namespace hy;

extern "C" {

size_t hy_causal_conv_bwd_workspace_size(int B, int C, int L, int lh, int dtype) {
  if (B < 1 || C < 1 || L < 1 || lh < 1) return 0;
  return static_cast<size_t>(B) * bwd_nsplit(B, C, L) * C * lh * (dtype == HY_F64 ? 8 : 4);
}

int hy_causal_conv_bwd(const void* dy, const void* x, void* dx, void* dtaps, const void* taps, int B, int C, int L,
                       int lh, int gs, int dtype, void* ws, size_t ws_bytes, void* stream) {
  if (!dy) return fail(HY_ERR_INVALID, "null pointer argument (dy)");
  if (!dx && !dtaps) return fail(HY_ERR_INVALID, "nothing to compute: dx and dtaps are both null");
  if (dx && !taps) return fail(HY_ERR_INVALID, "dx needs taps");
  if (dtaps && (!x || !ws)) return fail(HY_ERR_INVALID, "dtaps needs x and a workspace");
  if (B < 1 || C < 1 || L < 1 || lh < 1 || gs < 1)
    return fail(HY_ERR_INVALID, "sizes must be >= 1 (B=%d C=%d L=%d lh=%d gs=%d)", B, C, L, lh, gs);
  if (C % gs != 0) return fail(HY_ERR_INVALID, "group_size %d does not divide channel count %d", gs, C);
  if (C > 65535 || B > 65535) return fail(HY_ERR_UNSUPPORTED, "grid limit: C and B must be <= 65535");
  if (lh > kBwdMaxLh) return fail(HY_ERR_UNSUPPORTED, "conv backward: filter length %d > %d", lh, kBwdMaxLh);
  if (dtype != HY_F32 && dtype != HY_BF16 && dtype != HY_F64) return fail(HY_ERR_INVALID, "unknown dtype %d", dtype);
  if (dtaps && ws_bytes < hy_causal_conv_bwd_workspace_size(B, C, L, lh, dtype))
    return fail(HY_ERR_INVALID, "workspace too small (%zu < %zu bytes)", ws_bytes,
                hy_causal_conv_bwd_workspace_size(B, C, L, lh, dtype));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  switch (dtype) {
    case HY_F32: return launch_bwd<float>(dy, x, dx, dtaps, taps, B, C, L, lh, gs, ws, st);
    case HY_BF16: return launch_bwd<__nv_bfloat16>(dy, x, dx, dtaps, taps, B, C, L, lh, gs, ws, st);
    default: return launch_bwd<double>(dy, x, dx, dtaps, taps, B, C, L, lh, gs, ws, st);
  }
}

}  // extern "C"

// ---------------------------------------------------------------- two-stage filter gradient, pass 2
// Pass 1 (tensor-core batched GEMMs over the chunked rows, ops.two_stage_taps_grad) leaves per
// channel the chunk-summed outer products P0 = sum_n dC_n U_n^T and P1 = sum_n dC_n U_{n-1}^T
// (lb x lb, fp32). Pass 2 scatters their block diagonals onto the taps (blockconv.py:253-262):
//   dtaps[g][j] = sum_{c in g} ( sum_{i-i'=j} P0[c][i][i'] + sum_{lb+i-i'=j} P1[c][i][i'] ),  j < lh.
namespace hy {
__global__ void toeplitz_diag_kernel(const float* __restrict__ P0, const float* __restrict__ P1,
                                     float* __restrict__ part, int lb, int lh) {
  const int c = blockIdx.x;
  const size_t base = static_cast<size_t>(c) * lb * lb;
  for (int j = threadIdx.x; j < lh; j += blockDim.x) {
    double s = 0.0;
    if (j < lb)
      for (int i = j; i < lb; ++i) s += P0[base + static_cast<size_t>(i) * lb + (i - j)];
    const int d = j - lb;  // i - i' = d for P1 (d in (-lb, 0] .. )
    for (int i = max(0, d); i < lb && i - d < lb; ++i) s += P1[base + static_cast<size_t>(i) * lb + (i - d)];
    part[static_cast<size_t>(c) * lh + j] = static_cast<float>(s);
  }
}
}  // namespace hy

extern "C" int hy_toeplitz_taps_reduce(const float* P0, const float* P1, float* dtaps, float* ws, size_t ws_bytes,
                                       int C, int lb, int lh, int gs, void* stream) {
  if (!P0 || !P1 || !dtaps || !ws) return fail(HY_ERR_INVALID, "null pointer argument");
  if (C < 1 || lb < 1 || lh < 1 || gs < 1 || C % gs) return fail(HY_ERR_INVALID, "bad sizes");
  if (lh > 2 * lb) return fail(HY_ERR_INELIGIBLE, "filter length %d needs more than one spill factor", lh);
  if (ws_bytes < static_cast<size_t>(C) * lh * sizeof(float)) return fail(HY_ERR_INVALID, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  toeplitz_diag_kernel<<<C, 128, 0, st>>>(P0, P1, ws, lb, lh);
  int s = check_launch("toeplitz_diag_kernel");
  if (s != HY_OK) return s;
  dim3 grid((lh + 127) / 128, C / gs);
  conv_taps_reduce_kernel<float><<<grid, 128, 0, st>>>(ws, dtaps, 1, C, lh, gs);
  return check_launch("conv_taps_reduce_kernel");
}
