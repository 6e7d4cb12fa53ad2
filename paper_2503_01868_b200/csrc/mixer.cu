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
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"

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
  constexpr bool RING = VEC;
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

// se_stream_kernel: the SE mixer for filters of <= 8 taps on 16-byte aligned rows. Each warp
// owns a contiguous range of 256-step chunks (row-major over (b, c, chunk)), so every chunk's
// FIR history is carried from the previous chunk instead of re-read: lane l holds steps
// [8l, 8l + 8), takes the last samples of lane l - 1 by one rotation shuffle, and lane 0
// takes them from the previous chunk (raw rows: the previous ring stage, still resident;
// u = k * v: a register carried across chunks). Chunks stream in by 1-D bulk copies (TMA)
// issued by one lane into a per-warp ring of kSsStages stages with an mbarrier each; a warp
// whose range starts mid-row first loads the 16 preceding steps (a warm-up chunk, no store).
// FIRs run on packed fp32 FMAs with the tap broadcast as a scalar operand and both sample
// pair alignments of the window built once per row. HBM traffic: 3 rows in, 1 out, once.
constexpr int kSsWarps = 8;
constexpr int kSsStages = 3;
constexpr int kSsChunk = 256;

template <typename T>
__device__ __forceinline__ void lds8(float (&x)[8], const T* p) {
  if constexpr (sizeof(T) == 4) {
    const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    x[0] = a.x, x[1] = a.y, x[2] = a.z, x[3] = a.w, x[4] = b.x, x[5] = b.y, x[6] = b.z, x[7] = b.w;
  } else {
    unpack16<T>(*reinterpret_cast<const int4*>(p), x);
  }
}

// out[i] = sum_{j < NJ} h[j] x[i - j], i < 8, from this lane's samples x[0..7] and the window
// history x[-8..-1] (hist[e] = x[e - 8]); output pairs on packed FMAs. Even taps read the
// naturally aligned pairs (x[2q], x[2q+1]); odd taps the pairs (x[2q-1], x[2q]), built once.
template <int NJ>
__device__ __forceinline__ void fir_pairs(float (&out)[8], const float (&x)[8], const float (&hist)[8],
                                          const float (&h)[NJ]) {
  auto at = [&](int i) { return i >= 0 ? x[i] : hist[8 + i]; };
  float2 ev[8], od[8];  // ev[q + 4] = (x[2q], x[2q+1]); od[q + 4] = (x[2q-1], x[2q]), q in [-4, 3]
#pragma unroll
  for (int q = -4; q < 4; ++q) {
    ev[q + 4] = make_float2(at(2 * q), at(2 * q + 1));
    od[q + 4] = make_float2(2 * q - 1 >= -8 ? at(2 * q - 1) : 0.f, at(2 * q));
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    float2 a = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
      const float2 w = (j & 1) ? od[p - (j - 1) / 2 + 4] : ev[p - j / 2 + 4];
      a = ffma2(make_float2(h[j], h[j]), w, a);
    }
    out[2 * p] = a.x;
    out[2 * p + 1] = a.y;
  }
}

// hist[e] (e >= 8 - NH) = sample e - 8 of this row window: lane l - 1's x[e] by a rotation
// shuffle; lane 0 takes `first` (the previous chunk's tail, or zeros at the row start).
template <int NH>
__device__ __forceinline__ void hist_shfl(float (&hist)[8], const float (&x)[8], const float (&first)[8], int lane) {
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    if (e >= 8 - NH) {
      const float s = __shfl_sync(kFull, x[e], (lane + 31) & 31);
      hist[e] = lane == 0 ? first[e] : s;
    } else {
      hist[e] = 0.f;
    }
  }
}

// PREP: the featurizer / gate stream instead of the mixer: u = fk * fv into y and
// dc = gmix * fq into dc_out (gmix = gradient at the mixer output: the backward's prologue),
// or fq itself when gmix is null (the context-parallel LI forward). rhist (nullable,
// (B, 3C, 8)): the 8 raw projected steps before t = 0 of every row (the predecessor rank's),
// used instead of zeros as the featurizers' history.
template <typename T, int NF, int NI, bool PREP = false>
__global__ void __launch_bounds__(kSsWarps * 32, 2)
se_stream_kernel(const T* __restrict__ proj, T* __restrict__ y, const float* __restrict__ feat_taps, int lhf,
                 const float* __restrict__ inner_taps, const float* __restrict__ decay, int lh, int gs, int B,
                 int C, int L, const T* __restrict__ gmix = nullptr, T* __restrict__ dc_out = nullptr,
                 T* __restrict__ dc_rev = nullptr, const T* __restrict__ rhist = nullptr) {
  using namespace sm100;
  constexpr int ROWB = kSsChunk * static_cast<int>(sizeof(T));  // bytes per row per stage
  constexpr int NHF = NF - 1, NHI = NI - 1;  // history samples each FIR needs
  extern __shared__ __align__(128) unsigned char ss_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NR = PREP ? 4 : 3;  // staged rows: k, v, q (+ gmix)
  T* ring = reinterpret_cast<T*>(ss_smem + warp * (kSsStages * NR * ROWB));  // [stage][k, v, q, g][256]
  uint64_t* bars = reinterpret_cast<uint64_t*>(ss_smem + kSsWarps * kSsStages * NR * ROWB) + warp * kSsStages;

  const int nch = (L + kSsChunk - 1) / kSsChunk;
  const long long total = static_cast<long long>(B) * C * nch;  // < 2^31 (host check)
  const long long gw = static_cast<long long>(blockIdx.x) * kSsWarps + warp, nw = static_cast<long long>(gridDim.x) * kSsWarps;
  const int i0 = static_cast<int>(total * gw / nw), i1 = static_cast<int>(total * (gw + 1) / nw);
  if (i0 >= i1) return;
  if (lane == 0) {
    for (int s = 0; s < kSsStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();

  // issue list: [warm-up chunk (when i0 starts mid-row)] + items i0 .. i1 - 1
  const bool warm = (i0 % nch) != 0;
  const int n_issue = (i1 - i0) + (warm ? 1 : 0);
  const int base = i0 - (warm ? 1 : 0);
  struct Cur {  // (row, chunk) of an issue-list entry, advanced without divisions
    int row, k;
    __device__ void next(int nch_) {
      if (++k == nch_) k = 0, ++row;
    }
  };
  const Cur start{base / nch, base % nch};
  // lane 0's issue cursor: the q row of the next entry to issue, its chunk, channel, stage
  const size_t CL = static_cast<size_t>(C) * L;
  const T* iss_q = proj + (static_cast<size_t>(start.row / C) * 3 * C + start.row % C) * L;
  const T* iss_g = (PREP && gmix) ? gmix + static_cast<size_t>(start.row) * L : nullptr;
  int iss_k = start.k, iss_c = start.row % C, iss_st = 0, n_iss = 0;
  auto issue = [&]() {  // lane 0: entry n_iss into stage n_iss % S
    int t0 = iss_k * kSsChunk, cnt = min(kSsChunk, L - t0), off = 0;
    if (warm && n_iss == 0) off = kSsChunk - 16, t0 += kSsChunk - 16, cnt = 16;  // the 16 steps before i0
    T* dst = ring + iss_st * NR * kSsChunk + off;
    const uint32_t bytes = static_cast<uint32_t>(cnt * sizeof(T));
    const T* src = iss_q + t0;
    fence_proxy_async();
    mbar_arrive_expect_tx(&bars[iss_st], (PREP && !gmix ? 3 : NR) * bytes);
    bulk_g2s(dst, src + CL, bytes, &bars[iss_st]);                  // k
    bulk_g2s(dst + kSsChunk, src + 2 * CL, bytes, &bars[iss_st]);  // v
    bulk_g2s(dst + 2 * kSsChunk, src, bytes, &bars[iss_st]);       // q
    if (PREP && gmix) bulk_g2s(dst + 3 * kSsChunk, iss_g + t0, bytes, &bars[iss_st]);  // gmix
    if (++iss_k == nch) {
      iss_k = 0;
      iss_q += L;
      if (PREP && gmix) iss_g += L;
      if (++iss_c == C) iss_c = 0, iss_q += 2 * CL;
    }
    if (++iss_st == kSsStages) iss_st = 0;
    ++n_iss;
  };
  if (lane == 0)
    while (n_iss < kSsStages - 1 && n_iss < n_issue) issue();

  float hq[NF], hk[NF], hv[NF], hi[NI];
  int cur_row = -1;
  float ucarry[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) ucarry[e] = 0.f;

  Cur pos = start;
  int st = 0, prv_st = kSsStages - 1;
  uint32_t parity = 0;
  for (int n = 0; n < n_issue; ++n) {
    const int row = pos.row, k = pos.k;
    if (row != cur_row) {  // new channel: taps into registers
      cur_row = row;
      const int c = row % C;
      const int g = c / gs;
      const float dr = decay ? __ldg(decay + g) : 0.f;
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        hq[j] = j < lhf ? __ldg(feat_taps + (static_cast<size_t>(0) * C + c) * lhf + j) : 0.f;
        hk[j] = j < lhf ? __ldg(feat_taps + (static_cast<size_t>(1) * C + c) * lhf + j) : 0.f;
        hv[j] = j < lhf ? __ldg(feat_taps + (static_cast<size_t>(2) * C + c) * lhf + j) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < NI; ++j) {
        float h = (!PREP && j < lh) ? __ldg(inner_taps + static_cast<size_t>(g) * lh + j) : 0.f;
        if (decay) h *= exp2f(-dr * static_cast<float>(j));
        hi[j] = h;
      }
    }
    mbar_wait(&bars[st], parity);
    const T* cur = ring + st * NR * kSsChunk;
    const T* prv = ring + prv_st * NR * kSsChunk;
    const bool row_start = (k == 0);
    float rk[8], rv[8], rq[8], pk[8], pv[8], pq[8];
    lds8<T>(rk, cur + 8 * lane);
    lds8<T>(rv, cur + kSsChunk + 8 * lane);
    lds8<T>(rq, cur + 2 * kSsChunk + 8 * lane);
    lds8<T>(pk, prv + kSsChunk - 8);  // the previous chunk's last 8 steps (broadcast)
    lds8<T>(pv, prv + 2 * kSsChunk - 8);
    lds8<T>(pq, prv + 3 * kSsChunk - 8);
    float gq[8];
    if (PREP) {
      if (gmix) {
        lds8<T>(gq, cur + 3 * kSsChunk + 8 * lane);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) gq[e] = 1.f;
      }
    }
    __syncwarp();
    // the stage read before this one is free now: refill it S - 1 entries ahead
    if (lane == 0 && n_iss < n_issue) issue();
    prv_st = st;
    if (++st == kSsStages) st = 0, parity ^= 1u;
    pos.next(nch);
    if (row_start) {
#pragma unroll
      for (int e = 0; e < 8; ++e) pk[e] = pv[e] = pq[e] = ucarry[e] = 0.f;
      if (PREP && rhist) {  // the predecessor's last 8 raw steps of this row's q / k / v
        const int b = row / C, c = row - b * C;
        const T* hq = rhist + (static_cast<size_t>(b) * 3 * C + c) * 8;
        lds8<T>(pq, hq);
        lds8<T>(pk, hq + static_cast<size_t>(C) * 8);
        lds8<T>(pv, hq + 2 * static_cast<size_t>(C) * 8);
      }
    }
    float hist[8], fk[8], fv[8], u[8], acc[8], fq[8];
    hist_shfl<NHF>(hist, rk, pk, lane);
    fir_pairs<NF>(fk, rk, hist, hk);
    hist_shfl<NHF>(hist, rv, pv, lane);
    fir_pairs<NF>(fv, rv, hist, hv);
#pragma unroll
    for (int e = 0; e < 8; ++e) u[e] = fk[e] * fv[e];
    if constexpr (PREP) {
      hist_shfl<NHF>(hist, rq, pq, lane);
      fir_pairs<NF>(fq, rq, hist, hq);
      const int t = k * kSsChunk + 8 * lane;
      if (!(warm && n == 0) && t < L) {
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = gq[e] * fq[e];
        T* up = y + static_cast<size_t>(row) * L + t;
        T* dp = dc_out + static_cast<size_t>(row) * L + t;
        if constexpr (sizeof(T) == 4) {
          st_stream16(up, pack16<T>(u)), st_stream16(up + 4, pack16<T>(u + 4));
          st_stream16(dp, pack16<T>(o)), st_stream16(dp + 4, pack16<T>(o + 4));
        } else {
          st_stream16(up, pack16<T>(u));
          st_stream16(dp, pack16<T>(o));
        }
        if (dc_rev) {  // dc time-reversed (the anti-causal conv runs as a causal one on it)
          float r[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) r[e] = o[7 - e];
          T* rp = dc_rev + static_cast<size_t>(row) * L + (L - 8 - t);
          if constexpr (sizeof(T) == 4) {
            st_stream16(rp, pack16<T>(r)), st_stream16(rp + 4, pack16<T>(r + 4));
          } else {
            st_stream16(rp, pack16<T>(r));
          }
        }
      }
      continue;
    }
    // u history: lane l - 1's u; lane 0 the previous chunk's lane 31 (carried)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (e >= 8 - NHI) {
        const float s = __shfl_sync(kFull, u[e], (lane + 31) & 31);
        hist[e] = lane == 0 ? ucarry[e] : s;
        ucarry[e] = s;  // lane 0 receives lane 31's u: the next chunk's carry
      } else {
        hist[e] = 0.f;
      }
    }
    fir_pairs<NI>(acc, u, hist, hi);
    hist_shfl<NHF>(hist, rq, pq, lane);
    fir_pairs<NF>(fq, rq, hist, hq);
    const bool store = !(warm && n == 0);
    const int t = k * kSsChunk + 8 * lane;
    if (store && t < L) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = acc[e] * fq[e];
      T* yp = y + static_cast<size_t>(row) * L + t;
      if constexpr (sizeof(T) == 4) {
        st_stream16(yp, pack16<T>(o));
        st_stream16(yp + 4, pack16<T>(o + 4));
      } else {
        st_stream16(yp, pack16<T>(o));
      }
    }
  }
}

template <typename T, int NF, int NI>
static int launch_se(const void* proj, void* y, const float* ft, int lhf, const float* it, const float* dec,
                     int lh, int gs, int B, int C, int L, cudaStream_t st) {
  const bool vec = (L % 8 == 0) && aligned16(proj) && aligned16(y);
  auto kern = vec ? se_mixer_kernel<T, NF, NI, true> : se_mixer_kernel<T, NF, NI, false>;
  constexpr int RING = (kSeThreads / 32) * 2 * 3 * 256 * static_cast<int>(sizeof(T));
  const int smem = vec ? RING : 0;
  if (RING > 0) {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(se_mixer_kernel<T, NF, NI, true>), RING);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  const long long cap = resident_cap(reinterpret_cast<const void*>(kern), kSeThreads, smem);
  constexpr int N2 = NF > NI ? NF : NI;
  constexpr int H = (NF > 8 ? 2 : 1) + (N2 > 8 ? 2 : 1);
  const long long items = static_cast<long long>((L + 8 * (32 - H) - 1) / (8 * (32 - H))) * C * B;
  if (items > 0x7fffffffLL) return fail(HY_ERR_UNSUPPORTED, "too many work items");
  const long long warps_per_cta = kSeThreads / 32;
  long long grid = (items + warps_per_cta - 1) / warps_per_cta;
  if (grid > cap) grid = cap;
  kern<<<static_cast<int>(grid), kSeThreads, smem, st>>>(static_cast<const T*>(proj), static_cast<T*>(y), ft, lhf,
                                                        it, dec, lh, gs, B, C, L);
  return check_launch("se_mixer_kernel");
}

template <typename T, int NF, int NI, bool PREP = false>
static int launch_se_stream(const void* proj, void* y, const float* ft, int lhf, const float* it, const float* dec,
                            int lh, int gs, int B, int C, int L, cudaStream_t st, const void* gmix = nullptr,
                            void* dc_out = nullptr, void* dc_rev = nullptr, const void* rhist = nullptr) {
  auto kern = se_stream_kernel<T, NF, NI, PREP>;
  constexpr int SMEM = kSsWarps * kSsStages * ((PREP ? 4 : 3) * kSsChunk * static_cast<int>(sizeof(T)) + 8);
  {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), SMEM);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  const long long cap = resident_cap(reinterpret_cast<const void*>(kern), kSsWarps * 32, SMEM);
  const long long total = static_cast<long long>((L + kSsChunk - 1) / kSsChunk) * C * B;
  if (total > 0x7fffffffLL) return fail(HY_ERR_UNSUPPORTED, "too many chunks");
  long long grid = (total + kSsWarps - 1) / kSsWarps;
  if (grid > cap) grid = cap;
  kern<<<static_cast<int>(grid), kSsWarps * 32, SMEM, st>>>(static_cast<const T*>(proj), static_cast<T*>(y), ft, lhf,
                                                             it, dec, lh, gs, B, C, L, static_cast<const T*>(gmix),
                                                             static_cast<T*>(dc_out), static_cast<T*>(dc_rev),
                                                             static_cast<const T*>(rhist));
  return check_launch("se_stream_kernel");
}

template <typename T>
static int launch_se_dispatch(const void* proj, void* y, const float* ft, int lhf, const float* it,
                              const float* dec, int lh, int gs, int B, int C, int L, cudaStream_t st) {
  const bool vec = (L % 8 == 0) && aligned16(proj) && aligned16(y);
  if (vec && lhf == 7 && lh == 7) return launch_se_stream<T, 7, 7>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
  if (vec && lhf <= 8 && lh <= 8) return launch_se_stream<T, 8, 8>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
  if (lhf == 7 && lh == 7) return launch_se<T, 7, 7>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
  if (lhf <= 8 && lh <= 8) return launch_se<T, 8, 8>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
  if (lhf <= 8) return launch_se<T, 8, 16>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
  if (lh <= 8) return launch_se<T, 16, 8>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
  return launch_se<T, 16, 16>(proj, y, ft, lhf, it, dec, lh, gs, B, C, L, st);
}

// fir_stream_kernel: y = [q *] (h conv ([k *] v)) for filters of <= 8 taps on 16-byte
// aligned rows (kernel F: direct_causal_conv / the featurizer, core.py:212-226, and the short
// gated two-stage conv). The se_stream_kernel scheme on one (or, gated, three) staged rows:
// warps own contiguous ranges of 256-step chunks (row-major over rows), chunks arrive by 1-D
// bulk copies into a per-warp ring, lane l holds steps [8l, 8l + 8) and takes its FIR history
// from lane l - 1 by a rotation shuffle and, for lane 0, from the previous ring stage; packed
// fp32 FMAs. Every byte is read once and written once.
constexpr int kFsWarps = 8;
constexpr int kFsStages = 4;

template <typename T, int NJ, bool GK, bool GQ>
__global__ void __launch_bounds__(kFsWarps * 32, 2)
fir_stream_kernel(const T* __restrict__ q, const T* __restrict__ kk, const T* __restrict__ v, T* __restrict__ y,
                  const float* __restrict__ taps, int lh, int gs, int C, int rows, int L) {
  using namespace sm100;
  constexpr int NR = 1 + (GK ? 1 : 0) + (GQ ? 1 : 0);  // staged rows: v [, k] [, q]
  extern __shared__ __align__(128) unsigned char fs_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* ring = reinterpret_cast<T*>(fs_smem + warp * (kFsStages * NR * kSsChunk * static_cast<int>(sizeof(T))));
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(fs_smem + kFsWarps * kFsStages * NR * kSsChunk * static_cast<int>(sizeof(T))) +
      warp * kFsStages;
  const int nch = (L + kSsChunk - 1) / kSsChunk;
  const long long total = static_cast<long long>(rows) * nch;
  const long long gw = static_cast<long long>(blockIdx.x) * kFsWarps + warp;
  const long long nw = static_cast<long long>(gridDim.x) * kFsWarps;
  const int i0 = static_cast<int>(total * gw / nw), i1 = static_cast<int>(total * (gw + 1) / nw);
  if (i0 >= i1) return;
  if (lane == 0) {
    for (int s = 0; s < kFsStages; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const bool warm = (i0 % nch) != 0;  // starts mid-row: first load the 16 steps before i0
  const int n_issue = (i1 - i0) + (warm ? 1 : 0);
  const int base = i0 - (warm ? 1 : 0);
  int iss_row = base / nch, iss_k = base % nch, iss_st = 0, n_iss = 0;
  auto issue = [&]() {
    int t0 = iss_k * kSsChunk, cnt = min(kSsChunk, L - t0), off = 0;
    if (warm && n_iss == 0) off = kSsChunk - 16, t0 += kSsChunk - 16, cnt = 16;
    T* dst = ring + iss_st * NR * kSsChunk + off;
    const uint32_t bytes = static_cast<uint32_t>(cnt * sizeof(T));
    const size_t src = static_cast<size_t>(iss_row) * L + t0;
    fence_proxy_async();  // the stage's earlier generic reads before the async refill
    mbar_arrive_expect_tx(&bars[iss_st], NR * bytes);
    bulk_g2s(dst, v + src, bytes, &bars[iss_st]);
    if (GK) bulk_g2s(dst + kSsChunk, kk + src, bytes, &bars[iss_st]);
    if (GQ) bulk_g2s(dst + (NR - 1) * kSsChunk, q + src, bytes, &bars[iss_st]);
    if (++iss_k == nch) iss_k = 0, ++iss_row;
    if (++iss_st == kFsStages) iss_st = 0;
    ++n_iss;
  };
  if (lane == 0)
    while (n_iss < kFsStages - 1 && n_iss < n_issue) issue();
  float h[NJ];
  int cur_row = -1;
  int row = base / nch, k = base % nch;
  int st = 0, prv_st = kFsStages - 1;
  uint32_t parity = 0;
  for (int n = 0; n < n_issue; ++n) {
    if (row != cur_row) {
      cur_row = row;
      const int g = (row % C) / gs;
#pragma unroll
      for (int j = 0; j < NJ; ++j) h[j] = j < lh ? __ldg(taps + static_cast<size_t>(g) * lh + j) : 0.f;
    }
    mbar_wait(&bars[st], parity);
    const T* cur = ring + st * NR * kSsChunk;
    const T* prv = ring + prv_st * NR * kSsChunk;
    float x[8], px[8], rq[8];
    lds8<T>(x, cur + 8 * lane);
    lds8<T>(px, prv + kSsChunk - 8);
    if (GK) {
      float xk[8], pk[8];
      lds8<T>(xk, cur + kSsChunk + 8 * lane);
      lds8<T>(pk, prv + 2 * kSsChunk - 8);
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] *= xk[e], px[e] *= pk[e];
    }
    if (GQ) lds8<T>(rq, cur + (NR - 1) * kSsChunk + 8 * lane);
    __syncwarp();
    if (lane == 0 && n_iss < n_issue) issue();
    const bool row_start = (k == 0);
    const int t = k * kSsChunk + 8 * lane;
    const int out_row = row;
    prv_st = st;
    if (++st == kFsStages) st = 0, parity ^= 1u;
    if (++k == nch) k = 0, ++row;
    if (row_start) {
#pragma unroll
      for (int e = 0; e < 8; ++e) px[e] = 0.f;
    }
    float hist[8], o[8];
    hist_shfl<NJ - 1>(hist, x, px, lane);
    fir_pairs<NJ>(o, x, hist, h);
    if (GQ) {
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] *= rq[e];
    }
    if (!(warm && n == 0) && t < L) {
      T* yp = y + static_cast<size_t>(out_row) * L + t;
      if constexpr (sizeof(T) == 4) {
        st_stream16(yp, pack16<T>(o));
        st_stream16(yp + 4, pack16<T>(o + 4));
      } else {
        st_stream16(yp, pack16<T>(o));
      }
    }
  }
}

template <typename T, int NJ, bool GK, bool GQ>
static int launch_fir_stream_t(const void* q, const void* k, const void* v, void* y, const float* taps, int lh,
                               int gs, int C, int rows, int L, cudaStream_t st) {
  auto kern = fir_stream_kernel<T, NJ, GK, GQ>;
  constexpr int NR = 1 + (GK ? 1 : 0) + (GQ ? 1 : 0);
  constexpr int SMEM = kFsWarps * kFsStages * (NR * kSsChunk * static_cast<int>(sizeof(T)) + 8);
  {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), SMEM);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  const long long cap = resident_cap(reinterpret_cast<const void*>(kern), kFsWarps * 32, SMEM);
  const long long total = static_cast<long long>((L + kSsChunk - 1) / kSsChunk) * rows;
  if (total > 0x7fffffffLL) return fail(HY_ERR_UNSUPPORTED, "too many chunks");
  long long grid = (total + kFsWarps - 1) / kFsWarps;
  if (grid > cap) grid = cap;
  kern<<<static_cast<int>(grid), kFsWarps * 32, SMEM, st>>>(static_cast<const T*>(q), static_cast<const T*>(k),
                                                           static_cast<const T*>(v), static_cast<T*>(y), taps, lh, gs,
                                                           C, rows, L);
  return check_launch("fir_stream_kernel");
}

template <typename T, int NJ>
static int launch_fir_stream_g(const void* q, const void* k, const void* v, void* y, const float* taps, int lh,
                               int gs, int C, int rows, int L, cudaStream_t st) {
  if (q && k) return launch_fir_stream_t<T, NJ, true, true>(q, k, v, y, taps, lh, gs, C, rows, L, st);
  if (k) return launch_fir_stream_t<T, NJ, true, false>(q, k, v, y, taps, lh, gs, C, rows, L, st);
  if (q) return launch_fir_stream_t<T, NJ, false, true>(q, k, v, y, taps, lh, gs, C, rows, L, st);
  return launch_fir_stream_t<T, NJ, false, false>(q, k, v, y, taps, lh, gs, C, rows, L, st);
}

bool fir_stream_eligible(const void* q, const void* k, const void* v, const void* y, int lh, int L, int dtype) {
  return (dtype == HY_F32 || dtype == HY_BF16) && lh <= 8 && L % 8 == 0 && aligned16(v) && aligned16(y) &&
         (!q || aligned16(q)) && (!k || aligned16(k));
}

int fir_stream_fwd(const void* q, const void* k, const void* v, void* y, const float* taps, int B, int C, int L,
                   int lh, int gs, int dtype, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int rows = B * C;
  if (dtype == HY_F32)
    return lh == 7 ? launch_fir_stream_g<float, 7>(q, k, v, y, taps, lh, gs, C, rows, L, st)
                   : launch_fir_stream_g<float, 8>(q, k, v, y, taps, lh, gs, C, rows, L, st);
  return lh == 7 ? launch_fir_stream_g<__nv_bfloat16, 7>(q, k, v, y, taps, lh, gs, C, rows, L, st)
                 : launch_fir_stream_g<__nv_bfloat16, 8>(q, k, v, y, taps, lh, gs, C, rows, L, st);
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
  static const bool kb_mixer = [] { const char* e = getenv("HY_MR_KB"); return e && atoi(e) != 0; }();
  if (dtype == HY_BF16 && L % 8 == 0 && aligned16(proj) && aligned16(y) && !hist && lhf <= 8 && kb_mixer &&
      lh <= 129)  // HY_MR_KB=1: the MR mixer on the staged-row kernel (CUDA-core featurizers, 64-chunk tiles)
    return mixer_tc_fwd(proj, y, ft, lhf, it, inner_decay, lh, nullptr, nullptr, 0, gs, B, C, L, stream);
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

// Backward prologue of the mixer (hyena.py:262-270): u = (Fk conv pk) * (Fv conv pv) and
// dc = dmixed * (Fq conv pq) from the projections in one stream (se_stream_kernel<PREP>).
extern "C" int hy_mixer_bwd_prep(const void* proj, const void* dmixed, const float* feat_taps, int lhf, int B, int C,
                                 int L, int dtype, void* u, void* dc, void* dc_rev, void* stream) {
  if (!proj || !dmixed || !feat_taps || !u || !dc) return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || lhf < 1) return fail(HY_ERR_INVALID, "sizes must be >= 1");
  if (lhf > 8) return fail(HY_ERR_UNSUPPORTED, "mixer backward prologue: lhf %d > 8", lhf);
  if (L % 8 != 0 || !aligned16(proj) || !aligned16(dmixed) || !aligned16(u) || !aligned16(dc) ||
      (dc_rev && !aligned16(dc_rev)))
    return fail(HY_ERR_UNSUPPORTED, "mixer backward prologue needs L %% 8 == 0 and 16-byte aligned rows");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == HY_BF16)
    return lhf == 7 ? launch_se_stream<__nv_bfloat16, 7, 1, true>(proj, u, feat_taps, lhf, nullptr, nullptr, 1, 1, B, C,
                                                                 L, st, dmixed, dc, dc_rev)
                    : launch_se_stream<__nv_bfloat16, 8, 1, true>(proj, u, feat_taps, lhf, nullptr, nullptr, 1, 1, B, C,
                                                                 L, st, dmixed, dc, dc_rev);
  if (dtype == HY_F32)
    return lhf == 7 ? launch_se_stream<float, 7, 1, true>(proj, u, feat_taps, lhf, nullptr, nullptr, 1, 1, B, C, L, st,
                                                         dmixed, dc, dc_rev)
                    : launch_se_stream<float, 8, 1, true>(proj, u, feat_taps, lhf, nullptr, nullptr, 1, 1, B, C, L, st,
                                                         dmixed, dc, dc_rev);
  return fail(HY_ERR_UNSUPPORTED, "mixer backward prologue: fp32 / bf16 only");
}

// Featurizers + k*v gate from the projections in one stream (se_stream_kernel<PREP> without a
// gradient input): u = (Fk conv pk) * (Fv conv pv) and fq = Fq conv pq, with the optional
// (B, 3C, 8) raw history rhist in place of zeros before t = 0 (context parallel).
extern "C" int hy_featurize_fwd(const void* proj, const void* rhist, const float* feat_taps, int lhf, int B, int C,
                                int L, int dtype, void* u, void* fq, void* stream) {
  if (!proj || !feat_taps || !u || !fq) return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || lhf < 1) return fail(HY_ERR_INVALID, "sizes must be >= 1");
  if (lhf > 8) return fail(HY_ERR_UNSUPPORTED, "featurize: lhf %d > 8", lhf);
  if (L % 8 != 0 || !aligned16(proj) || !aligned16(u) || !aligned16(fq) || (rhist && !aligned16(rhist)))
    return fail(HY_ERR_UNSUPPORTED, "featurize needs L %% 8 == 0 and 16-byte aligned rows");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == HY_BF16)
    return lhf == 7 ? launch_se_stream<__nv_bfloat16, 7, 1, true>(proj, u, feat_taps, lhf, nullptr, nullptr, 1, 1, B, C,
                                                                 L, st, nullptr, fq, nullptr, rhist)
                    : launch_se_stream<__nv_bfloat16, 8, 1, true>(proj, u, feat_taps, lhf, nullptr, nullptr, 1, 1, B, C,
                                                                 L, st, nullptr, fq, nullptr, rhist);
  if (dtype == HY_F32)
    return lhf == 7 ? launch_se_stream<float, 7, 1, true>(proj, u, feat_taps, lhf, nullptr, nullptr, 1, 1, B, C, L, st,
                                                         nullptr, fq, nullptr, rhist)
                    : launch_se_stream<float, 8, 1, true>(proj, u, feat_taps, lhf, nullptr, nullptr, 1, 1, B, C, L, st,
                                                         nullptr, fq, nullptr, rhist);
  return fail(HY_ERR_UNSUPPORTED, "featurize: fp32 / bf16 only");
}
