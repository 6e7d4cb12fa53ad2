// Fused featurizer backward of the Hyena mixer (hyena.py:234-247 applied to q, k, v, plus the
// gate products of hyena.py:262-270), one HBM pass:
//   fk = Fk * pk, fv = Fv * pv                         (featurizers recomputed, causal FIR)
//   dfq = g * c,  dfk = du * fv,  dfv = du * fk         (g = dmixed, c = inner conv output)
//   dpx[t] = sum_j Fx[j] dfx[t + j]                     (anti-causal FIR, x in q, k, v)
//   dFx[j] += sum_t dfx[t] px[t - j]                    (tap gradient)
// Reads the three projected rows and g, c, du; writes dproj = [dpq; dpk; dpv].
//
// feat_bwd_kernel: every warp owns a contiguous range of chunks (row-major over (b, c,
// chunk)); a chunk covers 248 output steps but stages 256 + 8 steps: lane l holds steps
// [t0 + 8l, t0 + 8l + 8), the 8 steps before t0 come along with the raw rows (each lane reads
// its causal history straight from shared memory), and lane 31's steps are only the
// anti-causal future of lane 30 (they are recomputed as lane 0 of the next chunk). So chunks
// are independent: no carried state, no warm-up. Chunks stream in by 1-D bulk copies (TMA)
// issued by one lane into a 6-stage per-warp ring with an mbarrier per stage. Tap gradients
// accumulate in registers per lane and leave by a warp reduction and fp64 atomics when the
// warp moves to another channel.
#include "common.cuh"
#include "sm100.cuh"

namespace hy {

constexpr int kFbStages = 6;
constexpr int kFbStep = 248;   // output steps per chunk
constexpr int kFbRaw = 264;    // staged raw steps per chunk: 8 history + 256
constexpr int kFbGrad = 256;   // staged g / c / du steps per chunk
constexpr unsigned kFbFull = 0xffffffffu;

template <typename T>
constexpr int fb_warps() { return 4; }  // 164 registers: 4-warp CTAs fit 3 per SM (8-warp CTAs only 1)
template <typename T>
constexpr int fb_stage_elems() { return 3 * kFbRaw + 3 * kFbGrad; }
template <typename T>
constexpr int fb_smem() { return fb_warps<T>() * kFbStages * (fb_stage_elems<T>() * static_cast<int>(sizeof(T)) + 8); }

template <typename T>
__device__ __forceinline__ void fb_lds8(float (&x)[8], const T* p) {
  if constexpr (sizeof(T) == 4) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
  } else {
    unpack16<T>(*reinterpret_cast<const int4*>(p), x);
  }
}

// x[0..16) = p[0..16): the 8 history steps and this lane's 8 steps
template <typename T>
__device__ __forceinline__ void fb_lds16(float (&x)[16], const T* p) {
  float a[8], b[8];
  fb_lds8<T>(a, p);
  fb_lds8<T>(b, p + 8);
#pragma unroll
  for (int e = 0; e < 8; ++e) x[e] = a[e], x[8 + e] = b[e];
}

template <typename T>
__device__ __forceinline__ void fb_st8(T* p, const float (&x)[8]) {
  if constexpr (sizeof(T) == 4) {
    st_stream16(p, pack16<T>(x));
    st_stream16(p + 4, pack16<T>(x + 4));
  } else {
    st_stream16(p, pack16<T>(x));
  }
}

template <typename T, int NF>
__global__ void __launch_bounds__(fb_warps<T>() * 32)
feat_bwd_kernel(const T* __restrict__ proj, const T* __restrict__ gmix, const T* __restrict__ cout,
                const T* __restrict__ dU, const float* __restrict__ feat_taps, int lhf, int B, int C, int L,
                T* __restrict__ dproj, double* __restrict__ dfeat64, int du_rev) {
  using namespace sm100;
  constexpr int W = fb_warps<T>();
  constexpr int SE = fb_stage_elems<T>();
  extern __shared__ __align__(128) unsigned char fb_smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* ring = reinterpret_cast<T*>(fb_smem_raw) + static_cast<size_t>(warp) * kFbStages * SE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(fb_smem_raw + static_cast<size_t>(W) * kFbStages * SE * sizeof(T)) +
                   warp * kFbStages;

  const int nch = (L + kFbStep - 1) / kFbStep;
  const long long total = static_cast<long long>(B) * C * nch;
  const long long gw = static_cast<long long>(blockIdx.x) * W + warp, nw = static_cast<long long>(gridDim.x) * W;
  const int i0 = static_cast<int>(total * gw / nw), i1 = static_cast<int>(total * (gw + 1) / nw);
  if (i0 >= i1) return;
  if (lane == 0) {
    for (int s = 0; s < kFbStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const int n_items = i1 - i0;
  const size_t CL = static_cast<size_t>(C) * L;

  // lane 0's issue cursor
  int is_row = i0 / nch, is_k = i0 % nch, is_st = 0, n_iss = 0;
  auto issue = [&]() {
    const int b = is_row / C, c = is_row - b * C;
    const T* qrow = proj + (static_cast<size_t>(b) * 3 * C + c) * L;  // [q; k; v] rows of (b, c)
    const size_t grow = static_cast<size_t>(is_row) * L;
    const int t0 = is_k * kFbStep;
    T* dst = ring + is_st * SE;
    int rs = t0 - 8, roff = 0;
    if (rs < 0) rs = 0, roff = 8;  // row start: history stays stale, lane 0 zeroes it
    const int rcnt = min(kFbRaw - roff, L - rs);
    const int gcnt = min(kFbGrad, L - t0);
    const uint32_t rb = static_cast<uint32_t>(rcnt * sizeof(T)), gb = static_cast<uint32_t>(gcnt * sizeof(T));
    fence_proxy_async();
    mbar_arrive_expect_tx(&bars[is_st], 3 * rb + 3 * gb);
    bulk_g2s(dst + roff, qrow + CL + rs, rb, &bars[is_st]);                      // pk
    bulk_g2s(dst + kFbRaw + roff, qrow + 2 * CL + rs, rb, &bars[is_st]);         // pv
    bulk_g2s(dst + 2 * kFbRaw + roff, qrow + rs, rb, &bars[is_st]);              // pq
    // du; du_rev: the row is stored time-reversed, steps [t0, t0 + gcnt) sit at [L - t0 - gcnt, L - t0)
    // and land at the top of the slot so step t0 + i is element kFbGrad - 1 - i
    if (du_rev) bulk_g2s(dst + 3 * kFbRaw + kFbGrad - gcnt, dU + grow + (L - t0 - gcnt), gb, &bars[is_st]);
    else bulk_g2s(dst + 3 * kFbRaw, dU + grow + t0, gb, &bars[is_st]);
    bulk_g2s(dst + 3 * kFbRaw + kFbGrad, gmix + grow + t0, gb, &bars[is_st]);    // g
    bulk_g2s(dst + 3 * kFbRaw + 2 * kFbGrad, cout + grow + t0, gb, &bars[is_st]);  // c
    if (++is_k == nch) is_k = 0, ++is_row;
    if (++is_st == kFbStages) is_st = 0;
    ++n_iss;
  };
  if (lane == 0)
    while (n_iss < kFbStages - 1 && n_iss < n_items) issue();

  float Fq[NF], Fk[NF], Fv[NF];
  float aq[NF], ak[NF], av[NF];  // this lane's tap-gradient partial sums
  int cur_row = -1;
  auto flush = [&](int row) {  // warp-reduce the partials and add them to channel row % C
#pragma unroll
    for (int j = 0; j < NF; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        aq[j] += __shfl_xor_sync(kFbFull, aq[j], o);
        ak[j] += __shfl_xor_sync(kFbFull, ak[j], o);
        av[j] += __shfl_xor_sync(kFbFull, av[j], o);
      }
    }
    const int c = row % C;
    if (lane < NF && lane < lhf) {
      float vq = 0.f, vk = 0.f, vv = 0.f;
#pragma unroll
      for (int j = 0; j < NF; ++j)
        if (j == lane) vq = aq[j], vk = ak[j], vv = av[j];
      atomicAdd(dfeat64 + (static_cast<size_t>(0) * C + c) * lhf + lane, static_cast<double>(vq));
      atomicAdd(dfeat64 + (static_cast<size_t>(1) * C + c) * lhf + lane, static_cast<double>(vk));
      atomicAdd(dfeat64 + (static_cast<size_t>(2) * C + c) * lhf + lane, static_cast<double>(vv));
    }
  };

  int row = i0 / nch, k = i0 % nch, st = 0;
  uint32_t parity = 0;
  for (int n = 0; n < n_items; ++n) {
    if (row != cur_row) {
      if (cur_row >= 0) flush(cur_row);
      cur_row = row;
      const int c = row % C;
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const bool ok = j < lhf;
        Fq[j] = ok ? __ldg(feat_taps + (static_cast<size_t>(0) * C + c) * lhf + j) : 0.f;
        Fk[j] = ok ? __ldg(feat_taps + (static_cast<size_t>(1) * C + c) * lhf + j) : 0.f;
        Fv[j] = ok ? __ldg(feat_taps + (static_cast<size_t>(2) * C + c) * lhf + j) : 0.f;
        aq[j] = ak[j] = av[j] = 0.f;
      }
    }
    mbar_wait(&bars[st], parity);
    const T* sb = ring + st * SE;
    const int t0 = k * kFbStep;
    const int tl = t0 + 8 * lane;  // this lane's first step
    // windows: w[0..7] = steps tl-8..tl-1, w[8..15] = tl..tl+7
    float wk[16], wv[16], d[8], gq[8], cq[8];
    fb_lds16<T>(wk, sb + 8 * lane);
    fb_lds16<T>(wv, sb + kFbRaw + 8 * lane);
    if (du_rev) {
      float r[8];
      fb_lds8<T>(r, sb + 3 * kFbRaw + kFbGrad - 8 - 8 * lane);
#pragma unroll
      for (int e = 0; e < 8; ++e) d[e] = r[7 - e];
    } else {
      fb_lds8<T>(d, sb + 3 * kFbRaw + 8 * lane);
    }
    fb_lds8<T>(gq, sb + 3 * kFbRaw + kFbGrad + 8 * lane);
    fb_lds8<T>(cq, sb + 3 * kFbRaw + 2 * kFbGrad + 8 * lane);
    float wq[16];
    fb_lds16<T>(wq, sb + 2 * kFbRaw + 8 * lane);
    __syncwarp();
    if (lane == 0 && n_iss < n_items) issue();  // refills the stage read one entry ago
    if (++st == kFbStages) st = 0, parity ^= 1u;
    if (k == 0 && lane == 0) {
#pragma unroll
      for (int e = 0; e < 8; ++e) wk[e] = wv[e] = wq[e] = 0.f;
    }
    if (tl + 8 > L) {  // row tail: nothing at or beyond L (stale shared memory) may contribute
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const bool ok = tl - 8 + i < L;
        wk[i] = ok ? wk[i] : 0.f;
        wv[i] = ok ? wv[i] : 0.f;
        wq[i] = ok ? wq[i] : 0.f;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool ok = tl + e < L;
        d[e] = ok ? d[e] : 0.f;
        gq[e] = ok ? gq[e] : 0.f;
        cq[e] = ok ? cq[e] : 0.f;
      }
    }
    if (++k == nch) k = 0, ++row;
    // featurizers and gate products
    // (packed FFMA2 on output pairs (e, e + 1); each output keeps the scalar accumulation order)
    float dk[8], dv[8], dq[8];
    {
      float2 fk2[4], fv2[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fk2[i] = fv2[i] = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const float2 tk = make_float2(Fk[j], Fk[j]), tv = make_float2(Fv[j], Fv[j]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int x0 = 8 + 2 * i - j;
          fk2[i] = __ffma2_rn(tk, make_float2(wk[x0], wk[x0 + 1]), fk2[i]);
          fv2[i] = __ffma2_rn(tv, make_float2(wv[x0], wv[x0 + 1]), fv2[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        dk[2 * i] = d[2 * i] * fv2[i].x;
        dk[2 * i + 1] = d[2 * i + 1] * fv2[i].y;
        dv[2 * i] = d[2 * i] * fk2[i].x;
        dv[2 * i + 1] = d[2 * i + 1] * fk2[i].y;
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) dq[e] = gq[e] * cq[e];
    }
    // tap gradients (lane 31's steps belong to the next chunk)
    if (lane < 31) {
#pragma unroll
      for (int j = 0; j < NF; ++j)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          aq[j] = fmaf(dq[e], wq[8 + e - j], aq[j]);
          ak[j] = fmaf(dk[e], wk[8 + e - j], ak[j]);
          av[j] = fmaf(dv[e], wv[8 + e - j], av[j]);
        }
    }
    // anti-causal FIRs with the next lane's first NF - 1 d-features
    float nq[8], nk[8], nv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (e < NF - 1) {
        nq[e] = __shfl_down_sync(kFbFull, dq[e], 1);
        nk[e] = __shfl_down_sync(kFbFull, dk[e], 1);
        nv[e] = __shfl_down_sync(kFbFull, dv[e], 1);
      } else {
        nq[e] = nk[e] = nv[e] = 0.f;
      }
    }
    float oq[8], ok_[8], ov[8];
    {
      float xq[16], xk[16], xv[16];  // this lane's d-features, then the next lane's first NF - 1
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xq[e] = dq[e], xk[e] = dk[e], xv[e] = dv[e];
        xq[8 + e] = nq[e], xk[8 + e] = nk[e], xv[8 + e] = nv[e];
      }
      float2 sq2[4], sk2[4], sv2[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) sq2[i] = sk2[i] = sv2[i] = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const float2 tq = make_float2(Fq[j], Fq[j]), tk = make_float2(Fk[j], Fk[j]), tv = make_float2(Fv[j], Fv[j]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int x0 = 2 * i + j;
          sq2[i] = __ffma2_rn(tq, make_float2(xq[x0], xq[x0 + 1]), sq2[i]);
          sk2[i] = __ffma2_rn(tk, make_float2(xk[x0], xk[x0 + 1]), sk2[i]);
          sv2[i] = __ffma2_rn(tv, make_float2(xv[x0], xv[x0 + 1]), sv2[i]);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        oq[2 * i] = sq2[i].x, oq[2 * i + 1] = sq2[i].y;
        ok_[2 * i] = sk2[i].x, ok_[2 * i + 1] = sk2[i].y;
        ov[2 * i] = sv2[i].x, ov[2 * i + 1] = sv2[i].y;
      }
    }
    if (lane < 31 && tl < L) {
      const int b = cur_row / C, c = cur_row - b * C;
      T* base = dproj + (static_cast<size_t>(b) * 3 * C + c) * L + tl;
      fb_st8<T>(base, oq);
      fb_st8<T>(base + CL, ok_);
      fb_st8<T>(base + 2 * CL, ov);
    }
  }
  flush(cur_row);
}

__global__ void fb_finish_kernel(const double* __restrict__ in, float* __restrict__ out, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = static_cast<float>(in[i]);
}

template <typename T, int NF>
static int launch_fb(const void* proj, const void* g, const void* c, const void* du, const float* ft, int lhf, int B,
                     int C, int L, void* dproj, float* dfeat, double* ws, int du_rev, cudaStream_t st) {
  auto kern = feat_bwd_kernel<T, NF>;
  constexpr int SMEM = fb_smem<T>();
  constexpr int THREADS = fb_warps<T>() * 32;
  {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), SMEM);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  const long long cap = resident_cap(reinterpret_cast<const void*>(kern), THREADS, SMEM);
  const long long total = static_cast<long long>((L + kFbStep - 1) / kFbStep) * C * B;
  if (total > 0x7fffffffLL) return fail(HY_ERR_UNSUPPORTED, "too many chunks");
  long long grid = (total + fb_warps<T>() - 1) / fb_warps<T>();
  if (grid > cap) grid = cap;
  const int n = 3 * C * lhf;
  cudaError_t e = cudaMemsetAsync(ws, 0, static_cast<size_t>(n) * sizeof(double), st);
  if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaMemsetAsync: %s", cudaGetErrorString(e));
  kern<<<static_cast<int>(grid), THREADS, SMEM, st>>>(
      static_cast<const T*>(proj), static_cast<const T*>(g), static_cast<const T*>(c), static_cast<const T*>(du), ft,
      lhf, B, C, L, static_cast<T*>(dproj), ws, du_rev);
  int s = check_launch("feat_bwd_kernel");
  if (s != HY_OK) return s;
  fb_finish_kernel<<<(n + 255) / 256, 256, 0, st>>>(ws, dfeat, n);
  return check_launch("fb_finish_kernel");
}

}  // namespace hy

using namespace hy;

extern "C" {

size_t hy_featurizer_bwd_workspace_size(int C, int lhf) {
  return C < 1 || lhf < 1 ? 0 : static_cast<size_t>(3) * C * lhf * sizeof(double);
}

int hy_featurizer_bwd(const void* proj, const void* dmixed, const void* conv_out, const void* du,
                      const float* feat_taps, int lhf, int B, int C, int L, int dtype, void* dproj, float* dfeat,
                      void* ws, size_t ws_bytes, int du_reversed, void* stream) {
  if (!proj || !dmixed || !conv_out || !du || !feat_taps || !dproj || !dfeat || !ws)
    return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || lhf < 1) return fail(HY_ERR_INVALID, "sizes must be >= 1");
  if (lhf > 8) return fail(HY_ERR_UNSUPPORTED, "featurizer backward: lhf %d > 8", lhf);
  if (L % 8 != 0) return fail(HY_ERR_UNSUPPORTED, "featurizer backward needs L %% 8 == 0 (L=%d)", L);
  if (!aligned16(proj) || !aligned16(dmixed) || !aligned16(conv_out) || !aligned16(du) || !aligned16(dproj))
    return fail(HY_ERR_UNSUPPORTED, "featurizer backward needs 16-byte aligned tensors");
  if (ws_bytes < hy_featurizer_bwd_workspace_size(C, lhf)) return fail(HY_ERR_INVALID, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* w = static_cast<double*>(ws);
  if (dtype == HY_BF16) {
    if (lhf == 7) return launch_fb<__nv_bfloat16, 7>(proj, dmixed, conv_out, du, feat_taps, lhf, B, C, L, dproj, dfeat, w, du_reversed, st);
    return launch_fb<__nv_bfloat16, 8>(proj, dmixed, conv_out, du, feat_taps, lhf, B, C, L, dproj, dfeat, w, du_reversed, st);
  }
  if (dtype == HY_F32) {
    if (lhf == 7) return launch_fb<float, 7>(proj, dmixed, conv_out, du, feat_taps, lhf, B, C, L, dproj, dfeat, w, du_reversed, st);
    return launch_fb<float, 8>(proj, dmixed, conv_out, du, feat_taps, lhf, B, C, L, dproj, dfeat, w, du_reversed, st);
  }
  return fail(HY_ERR_UNSUPPORTED, "featurizer backward: fp32 / bf16 only");
}

}  // extern "C"
