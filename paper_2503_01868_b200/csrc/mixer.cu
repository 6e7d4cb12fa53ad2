// se_mixer_kernel: register-resident, warp-shuffle filter reuse. A warp covers 256
// consecutive steps of one (batch, channel) row, 8 per lane, loaded with 16-byte vector
// loads of the raw projected q / k / v rows (coalesced 512 B per warp per row). Every FIR
// tap window reads the previous lanes' samples by rotation shuffles, so no sample is staged
// through shared memory:
//     k, v, q = featurizers(raw)      (history: lanes l-1, l-2)
//     u = k * v                       (registers)
//     y = q * (h_inner conv u)        (history of u: lanes l-1, l-2)
// The first H lanes of a warp block lack history and only feed their neighbours, so blocks
// advance by 8 * (32 - H) steps (H = 2 for filters of <= 8 taps: 6% re-read, from L2).
// Persistent warps walk the blocks row by row and prefetch the next block's rows into
// registers before computing the current one. HBM traffic is the 3 projected rows in and y
// out (16 B/token/channel at fp32, 8 at bf16).
#include "common.cuh"
#include "internal.h"

namespace hy {

constexpr int kSeThreads = 256;
constexpr unsigned kFull = 0xffffffffu;

// 8 consecutive samples row[t .. t+7] as floats (zeros outside [0, L)). VEC (L % 8 == 0,
// 16-byte aligned rows): t is a multiple of 8, so a run is wholly inside or outside.
template <typename T, bool VEC>
__device__ __forceinline__ void load8(float (&x)[8], const T* __restrict__ row, int t, int L) {
  if (VEC) {
    const bool in = t >= 0 && t < L;
    const T* p = row + (in ? t : 0);
    if constexpr (sizeof(T) == 4) {
      int4 a = ld_stream16(p), b = ld_stream16(p + 4);
      x[0] = __int_as_float(a.x), x[1] = __int_as_float(a.y), x[2] = __int_as_float(a.z), x[3] = __int_as_float(a.w);
      x[4] = __int_as_float(b.x), x[5] = __int_as_float(b.y), x[6] = __int_as_float(b.z), x[7] = __int_as_float(b.w);
    } else {
      unpack16<T>(ld_stream16(p), x);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = in ? x[e] : 0.f;
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = (t + e >= 0 && t + e < L) ? Elem<T>::to_a(row[t + e]) : 0.f;
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0)
               : "memory");
}

// Packed fp32 FMA (FFMA2: two fp32 lanes per instruction on sm_100), elementwise a * b + c.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long x, y, z, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(z) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(y), "l"(z));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}

// acc[i] = sum_{j < NJ} h[j] x[t + i - j] with this lane's 8 samples x and the history from
// lanes l-1 (and l-2 for NJ > 8) by rotation shuffles; output pairs (2p, 2p+1) accumulate
// with packed FMAs (scalar tap broadcast). Used for fp32 rows (register-resident windows).
template <int NJ>
__device__ __forceinline__ void fir8_shfl(float (&acc)[8], const float (&x)[8], const float2* hs, int comp,
                                          int lane) {
  float h[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) h[j] = comp ? hs[j].y : hs[j].x;
  float w[24];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    w[16 + e] = x[e];
    w[8 + e] = __shfl_sync(kFull, x[e], (lane + 31) & 31);
    if (NJ > 8) w[e] = __shfl_sync(kFull, x[e], (lane + 30) & 31);
  }
#pragma unroll
  for (int pr = 0; pr < 4; ++pr) {
    float2 a = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < NJ; ++j) a = ffma2(make_float2(h[j], h[j]), make_float2(w[16 + 2 * pr - j], w[17 + 2 * pr - j]), a);
    acc[2 * pr] = a.x;
    acc[2 * pr + 1] = a.y;
  }
}

// Two FIRs at once on interleaved rows: for i < 8,
//   acc[i] = (sum_j h[j].x a[t+i-j], sum_j h[j].y b[t+i-j]),  j < NJ
// with this lane's 8 samples of (a, b) and the history from lanes l-1 (and l-2 for NJ > 8)
// by rotation shuffles (lanes 0 / 1 receive wrapped values and are history-only). Every
// FFMA2 operand is a naturally aligned (a, b) pair; each tap is one fp32 rounding per row.
template <int NJ>
__device__ __forceinline__ void fir8x2(float2 (&acc)[8], const float (&a)[8], const float (&b)[8],
                                       const float2* hs, int lane) {
  float2 h[NJ];  // interleaved taps: broadcast 16-byte shared loads
#pragma unroll
  for (int j = 0; j < NJ; j += 2) {
    const float4 t4 = *reinterpret_cast<const float4*>(hs + j);
    h[j] = make_float2(t4.x, t4.y);
    if (j + 1 < NJ) h[j + 1] = make_float2(t4.z, t4.w);
  }
  float2 w[24];  // w[16 + e] = this lane, w[8 + e] = lane - 1, w[e] = lane - 2
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    w[16 + e] = make_float2(a[e], b[e]);
    if (e >= 9 - NJ || NJ > 8) {
      w[8 + e] = make_float2(__shfl_sync(kFull, a[e], (lane + 31) & 31), __shfl_sync(kFull, b[e], (lane + 31) & 31));
    }
    if (NJ > 8 && e >= 17 - NJ) {
      w[e] = make_float2(__shfl_sync(kFull, a[e], (lane + 30) & 31), __shfl_sync(kFull, b[e], (lane + 30) & 31));
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float2 s = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < NJ; ++j) s = ffma2(h[j], w[16 + i - j], s);
    acc[i] = s;
  }
}

// NF: featurizer taps (7 exactly, or padded to 8 / 16); NI: inner taps (likewise).
template <typename T, int NF, int NI, bool VEC>
__global__ void __launch_bounds__(kSeThreads, 3)
se_mixer_kernel(const T* __restrict__ proj, T* __restrict__ y, const float* __restrict__ feat_taps,
                int lhf, const float* __restrict__ inner_taps, const float* __restrict__ decay, int lh,
                int gs, int B, int C, int L) {
  constexpr int N2 = NF > NI ? NF : NI;                    // (q featurizer, inner conv) pass
  constexpr int H = (NF > 8 ? 2 : 1) + (N2 > 8 ? 2 : 1);  // history-only lanes
  constexpr int STEP = 8 * (32 - H);
  const int lane = threadIdx.x & 31;
  const int warp0 = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int n_warps = static_cast<int>((gridDim.x * blockDim.x) >> 5);
  const int nb = (L + STEP - 1) / STEP;
  // work items (b, c, blk), blk fastest; warps stride by n_warps (incremental, no divisions)
  const int sb = n_warps % nb, sr = n_warps / nb;
  struct Pos {
    int blk, c, b;
  };
  auto advance = [&](Pos& q) {
    q.blk += sb;
    int dr = sr;
    if (q.blk >= nb) q.blk -= nb, ++dr;
    q.c += dr;
    while (q.c >= C) q.c -= C, ++q.b;
  };
  Pos nxt{warp0 % nb, (warp0 / nb) % C, (warp0 / nb) / C};

  // this warp's taps, interleaved: (k, v) featurizers and (q featurizer, inner)
  constexpr int P1 = (NF + 1) / 2 * 2, P2 = (N2 + 1) / 2 * 2;
  __shared__ __align__(16) float2 taps_s[kSeThreads / 32][P1 + P2];
  float2* hkv = taps_s[threadIdx.x >> 5];
  float2* hqi = hkv + P1;
  int cur_c = -1;

  // the next item's raw rows (k, v, q) stream into this warp's two-stage shared ring with
  // 16-byte cp.async copies (zero-filled outside [0, L)) in two halves of 16 bytes per lane,
  // so each 16-byte read below is bank-conflict free (!VEC: register prefetch)
  // (measured: the ring wins for bf16, register prefetch for fp32)
  constexpr bool RING = VEC && sizeof(T) == 2;
  extern __shared__ __align__(16) unsigned char se_ring[];
  constexpr int HALF = 32 * (16 / static_cast<int>(sizeof(T)));
  constexpr int NHALF = 8 * static_cast<int>(sizeof(T)) / 16;
  constexpr int ROW = 256;
  T* ring = reinterpret_cast<T*>(se_ring) + (threadIdx.x >> 5) * (2 * 3 * ROW);
  float nq[8], nk[8], nv[8];
  auto fetch = [&](const Pos& q, int stage) {
    const T* qrow = proj + (static_cast<size_t>(q.b) * 3 * C + q.c) * L;
    const int t = q.blk * STEP + 8 * (lane - H);
    if (RING) {
      const bool ok = t >= 0 && t < L;
      const T* rows[3] = {qrow + static_cast<size_t>(C) * L, qrow + 2 * static_cast<size_t>(C) * L, qrow};
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        T* dst = ring + (stage * 3 + r) * ROW + lane * (16 / static_cast<int>(sizeof(T)));
#pragma unroll
        for (int hh = 0; hh < NHALF; ++hh)
          cp_async16(dst + hh * HALF, ok ? rows[r] + t + hh * HALF / 32 : rows[r], ok);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    } else {
      load8<T, VEC>(nk, qrow + static_cast<size_t>(C) * L, t, L);
      load8<T, VEC>(nv, qrow + 2 * static_cast<size_t>(C) * L, t, L);
      load8<T, VEC>(nq, qrow, t, L);
    }
  };
  auto read = [&](float (&x)[8], int stage, int r) {
    const T* src = ring + (stage * 3 + r) * ROW + lane * (16 / static_cast<int>(sizeof(T)));
    if constexpr (sizeof(T) == 4) {
      const float4 a = *reinterpret_cast<const float4*>(src), b = *reinterpret_cast<const float4*>(src + HALF);
      x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
    } else {
      unpack16<T>(*reinterpret_cast<const int4*>(src), x);
    }
  };
  int stage = 0;
  if (nxt.b < B) fetch(nxt, 0);
  while (nxt.b < B) {
    const Pos cur = nxt;
    float rq[8], rk[8], rv[8];
    if (!RING) {
#pragma unroll
      for (int e = 0; e < 8; ++e) rq[e] = nq[e], rk[e] = nk[e], rv[e] = nv[e];
    }
    advance(nxt);
    if (nxt.b < B) {
      fetch(nxt, stage ^ 1);
      if (RING) asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else if (RING) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    if (RING) {
      __syncwarp();
      read(rk, stage, 0);
      read(rv, stage, 1);
      read(rq, stage, 2);
      __syncwarp();  // the stage is refilled two items from now, after these reads
      stage ^= 1;
    }
    const int blk = cur.blk, c = cur.c, b = cur.b;
    if (c != cur_c) {
      cur_c = c;
      __syncwarp();
      if (lane < P2) {
        float hq = 0.f, hk = 0.f, hv = 0.f, hi = 0.f;
        if (lane < lhf) {
          hq = __ldg(feat_taps + (static_cast<size_t>(0) * C + c) * lhf + lane);
          hk = __ldg(feat_taps + (static_cast<size_t>(1) * C + c) * lhf + lane);
          hv = __ldg(feat_taps + (static_cast<size_t>(2) * C + c) * lhf + lane);
        }
        const int g = c / gs;
        if (lane < lh) {
          hi = __ldg(inner_taps + static_cast<size_t>(g) * lh + lane);
          if (decay) hi *= exp2f(-__ldg(decay + g) * static_cast<float>(lane));
        }
        if (lane < P1) hkv[lane] = make_float2(hk, hv);
        hqi[lane] = make_float2(hq, hi);
      }
    }
    __syncwarp();
    float out[8];
    if constexpr (RING) {
      // bf16: both passes as interleaved pairs, (k, v) then (q, u)
      float2 kv[8], qc[8];
      float u[8];
      fir8x2<NF>(kv, rk, rv, hkv, lane);
#pragma unroll
      for (int e = 0; e < 8; ++e) u[e] = kv[e].x * kv[e].y;
      fir8x2<N2>(qc, rq, u, hqi, lane);
#pragma unroll
      for (int e = 0; e < 8; ++e) out[e] = qc[e].y * qc[e].x;
    } else {
      // fp32: one row at a time (fewer live registers)
      float fk[8], fv[8], u[8], acc[8];
      fir8_shfl<NF>(fk, rk, hkv, 0, lane);
      fir8_shfl<NF>(fv, rv, hkv, 1, lane);
#pragma unroll
      for (int e = 0; e < 8; ++e) u[e] = fk[e] * fv[e];
      fir8_shfl<N2>(acc, u, hqi, 1, lane);
      fir8_shfl<N2>(fk, rq, hqi, 0, lane);
#pragma unroll
      for (int e = 0; e < 8; ++e) out[e] = acc[e] * fk[e];
    }
    const int t = blk * STEP + 8 * (lane - H);
    if (lane >= H && t < L) {
      T* yrow = y + (static_cast<size_t>(b) * C + c) * L;
      if (VEC) {
        if constexpr (sizeof(T) == 4) {
          st_stream16(yrow + t, pack16<T>(out));
          st_stream16(yrow + t + 4, pack16<T>(out + 4));
        } else {
          st_stream16(yrow + t, pack16<T>(out));
        }
      } else {
        for (int e = 0; e < 8; ++e)
          if (t + e < L) yrow[t + e] = Elem<T>::from_a(out[e]);
      }
    }
  }
}

template <typename T, int NF, int NI>
static int launch_se(const void* proj, void* y, const float* ft, int lhf, const float* it, const float* dec,
                     int lh, int gs, int B, int C, int L, cudaStream_t st) {
  const bool vec = (L % 8 == 0) && aligned16(proj) && aligned16(y);
  auto kern = vec ? se_mixer_kernel<T, NF, NI, true> : se_mixer_kernel<T, NF, NI, false>;
  constexpr int RING = sizeof(T) == 2 ? (kSeThreads / 32) * 2 * 3 * 256 * static_cast<int>(sizeof(T)) : 0;
  const int smem = vec ? RING : 0;
  static bool attr_set = false;
  if (!attr_set && RING > 0) {
    cudaError_t e = cudaFuncSetAttribute(se_mixer_kernel<T, NF, NI, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, RING);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSeThreads, smem);
  constexpr int N2 = NF > NI ? NF : NI;
  constexpr int H = (NF > 8 ? 2 : 1) + (N2 > 8 ? 2 : 1);
  const long long items = static_cast<long long>((L + 8 * (32 - H) - 1) / (8 * (32 - H))) * C * B;
  if (items > 0x7fffffffLL) return fail(HY_ERR_UNSUPPORTED, "too many work items");
  const long long warps_per_cta = kSeThreads / 32;
  long long grid = (items + warps_per_cta - 1) / warps_per_cta;
  const long long cap = static_cast<long long>(sms) * (per_sm > 0 ? per_sm : 1);
  if (grid > cap) grid = cap;
  kern<<<static_cast<int>(grid), kSeThreads, smem, st>>>(static_cast<const T*>(proj), static_cast<T*>(y), ft, lhf,
                                                        it, dec, lh, gs, B, C, L);
  return check_launch("se_mixer_kernel");
}

template <typename T>
static int launch_se_dispatch(const void* proj, void* y, const float* ft, int lhf, const float* it,
                              const float* dec, int lh, int gs, int B, int C, int L, cudaStream_t st) {
  if (lhf == 7 && lh == 7) return launch_se<T, 7, 7>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
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
