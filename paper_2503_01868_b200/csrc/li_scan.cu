// Hyena-LI long convolution as an exact modal state scan on CUDA cores (any dtype, any pole count).
//
// The implicit filter h_t = sum_n R_n lam_n^t (core.py:147-151) makes the causal conv
// (fft.py:128-145 in the reference, O(L log L) per channel) a sum of first-order recurrences:
//
//     y[t] = sum_n R_n s_n[t],   s_n[t] = lam_n s_n[t-1] + u[t],   u = k * v,   out = q * y
//
// exact in exact arithmetic (no FFT, no length-L filter). This kernel is the reference-precision
// path (fp32; also fp64, and bf16 with more than 8 poles), where the tcgen05 kernel's bf16
// operands / tf32 state MMA would miss the fp32 bar. HBM-bound: q, k, v in, y out, once.
//
// Work decomposition: one CTA (8 warps) walks whole rows (b, c); a row is cut into tiles of
// 256 lanes x S consecutive steps. Per tile and block of 8 modes:
//   1. each lane runs the recurrence over its S steps from zero -> its segment's end state b_l;
//   2. warp inclusive scan over lanes (Kogge-Stone, multiplier lam^(S d) at offset d);
//   3. warp totals through shared memory; each warp's incoming state is
//      lam^(32 S w) C + sum_{w' < w} lam^(32 S (w - 1 - w')) T_w'   (fp64), C = the state
//      carried into the tile (fp64, updated once per tile);
//   4. each lane's incoming state lam^(S l) in_w + I_{l-1}; the recurrence is re-run from it and
//      R_n s_n[t] accumulated into y.
// Powers of lam are evaluated in fp64 once per row (pow with integer exponents: exact sign,
// 0^0 = 1 as numpy); states are fp32 for fp32 / bf16 rows, fp64 for fp64 rows.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace hy {
namespace lis {

constexpr int WARPS = 8, THREADS = WARPS * 32;
constexpr int MB = 8;     // modes per register block
#ifndef HY_LIS_LA
#define HY_LIS_LA 1
#endif
constexpr int LA = HY_LIS_LA;  // one-shot kernel: tiles prefetched into L2 ahead of the loads
constexpr int MAXP = 64;  // poles per group
// one-shot kernel: CTAs per SM it is compiled for (3: 24 warps at <= 80 registers, no spills;
// the loads are latency-bound, so occupancy pays: the C3 fp32 mixer 2.40 -> 2.32 ms)
#ifndef LIS_MINB
#define LIS_MINB 3
#endif

template <typename T> struct Cfg;
template <> struct Cfg<float> {
  using A = float;
  static constexpr int S = 16;
};
template <> struct Cfg<__nv_bfloat16> {
  using A = float;
  static constexpr int S = 16;
};
template <> struct Cfg<double> {
  using A = double;
  static constexpr int S = 8;
};

template <typename T, int S, bool VEC>
__device__ __forceinline__ void load_seg(const T* __restrict__ p, int nv, typename Cfg<T>::A* out) {
  if (VEC && nv == S) {
    constexpr int PER = 16 / static_cast<int>(sizeof(T));
#pragma unroll
    for (int i = 0; i < S / PER; ++i) {
      const int4 raw = __ldcs(reinterpret_cast<const int4*>(p) + i);
      const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
      for (int j = 0; j < PER; ++j) out[i * PER + j] = Elem<T>::to_a(e[j]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < S; ++j) out[j] = j < nv ? Elem<T>::to_a(p[j]) : typename Cfg<T>::A(0);
  }
}

// steps [t - 8, t + S) of a row of length L into out[0 .. S + 8) (zeros outside [0, L))
template <typename T, int S, bool VEC>
__device__ __forceinline__ void load_halo_seg(const T* __restrict__ row, int t, int L, typename Cfg<T>::A* out) {
  using A = typename Cfg<T>::A;
  constexpr int PER = 16 / static_cast<int>(sizeof(T));
  if (VEC && t >= 8 && t + S <= L) {
#pragma unroll
    for (int i = 0; i < (S + 8) / PER; ++i) {
      const int4 raw = __ldg(reinterpret_cast<const int4*>(row + t - 8) + i);
      const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
      for (int j = 0; j < PER; ++j) out[i * PER + j] = Elem<T>::to_a(e[j]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < S + 8; ++j) {
      const int tt = t - 8 + j;
      out[j] = (tt >= 0 && tt < L) ? Elem<T>::to_a(row[tt]) : A(0);
    }
  }
}

// featurizer FIR (hyena.py:122-126, lhf <= 8 taps zero padded to 8) over S outputs
template <typename A, int S>
__device__ __forceinline__ void fir8(const A* raw, const A* h, A* out) {
#pragma unroll
  for (int t = 0; t < S; ++t) {
    A acc = A(0);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc = fma(h[j], raw[8 + t - j], acc);
    out[t] = acc;
  }
}
// fp32: the same FIR on output pairs (t, t+1) as packed FFMA2; the odd-aligned input pairs
// (raw[i], raw[i+1]) for odd i are formed once (S / 2 + 4 register moves) and reused by every tap
template <int S>
__device__ __forceinline__ void fir8_pairs(const float* raw, const float* h, float* out) {
  float2 ev[(S + 8) / 2], od[(S + 8) / 2];  // ev[i] = (raw[2i], raw[2i+1]); od[i] = (raw[2i+1], raw[2i+2])
#pragma unroll
  for (int i = 0; i < (S + 8) / 2; ++i) {
    ev[i] = make_float2(raw[2 * i], raw[2 * i + 1]);
    od[i] = make_float2(raw[2 * i + 1], 2 * i + 2 < S + 8 ? raw[2 * i + 2] : 0.f);
  }
#pragma unroll
  for (int t = 0; t < S; t += 2) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i0 = 8 + t - j;  // first input of the pair
      const float2 x = (i0 & 1) ? od[i0 >> 1] : ev[i0 >> 1];
      acc = __ffma2_rn(make_float2(h[j], h[j]), x, acc);
    }
    out[t] = acc.x;
    out[t + 1] = acc.y;
  }
}

template <typename T, int S, bool VEC>
__device__ __forceinline__ void store_seg(T* __restrict__ p, int nv, const typename Cfg<T>::A* in) {
  if (VEC && nv == S) {
    constexpr int PER = 16 / static_cast<int>(sizeof(T));
#pragma unroll
    for (int i = 0; i < S / PER; ++i) {
      int4 raw;
      T* e = reinterpret_cast<T*>(&raw);
#pragma unroll
      for (int j = 0; j < PER; ++j) e[j] = Elem<T>::from_a(in[i * PER + j]);
      __stcs(reinterpret_cast<int4*>(p) + i, raw);
    }
  } else {
#pragma unroll
    for (int j = 0; j < S; ++j)
      if (j < nv) p[j] = Elem<T>::from_a(in[j]);
  }
}

// FEAT: q, k, v are the raw projections (B, 3C, L) = [q; k; v] rows (`q` points at them), the
// featurizers (feat_taps (3, C, lhf) fp32, lhf <= 8) run in registers on each lane's segment
// with its 8-step history read from the row (L1 / L2 hits), so the fused mixer reads every
// projected row once and writes y once.
template <typename T, bool VEC, bool FEAT>
__global__ void __launch_bounds__(THREADS, LIS_MINB)
li_scan_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v, T* __restrict__ y,
               const double* __restrict__ res, const double* __restrict__ poles, int np, int gs, int C, int L,
               long long rows, const void* __restrict__ feat_raw, int lhf) {
  // featurizer taps: fp32 for fp32 / bf16 rows, fp64 for fp64 rows (the header's tap convention)
  using FT = typename std::conditional<sizeof(T) == 8, double, float>::type;
  const FT* feat = static_cast<const FT*>(feat_raw);
  using A = typename Cfg<T>::A;
  constexpr int S = Cfg<T>::S;
  constexpr int TILE = THREADS * S;
  constexpr bool PAIR = sizeof(A) == 4;  // fp32 states: FIRs and recurrences as packed FFMA2
  __shared__ A s_lam[MAXP], s_r[MAXP];
  __shared__ A s_pk[MAXP][5];           // lam^(S 2^k): the scan multipliers
  __shared__ A s_pl[MAXP][32];          // lam^(S l): a lane's offset in its warp
  __shared__ double s_pw[MAXP][WARPS + 1];  // lam^(32 S w): a warp's offset in the tile
  __shared__ double s_carry[MAXP];      // state entering the tile
  __shared__ A s_tot[2][WARPS][MB];     // warp totals (double-buffered by block iteration)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = (np + MB - 1) / MB;
  int it = 0;
  for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
    const int c = static_cast<int>(row % C);
    const int g = c / gs;
    A fh[3][8];  // FEAT: this channel's [q, k, v] featurizer taps
    const T* rq = nullptr;
    const T* rk = nullptr;
    const T* rv = nullptr;
    if constexpr (FEAT) {
#pragma unroll
      for (int x = 0; x < 3; ++x)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          fh[x][j] = j < lhf ? static_cast<A>(feat[(static_cast<size_t>(x) * C + c) * lhf + j]) : A(0);
      const long long b = row / C;
      rq = q + (static_cast<size_t>(b) * 3 * C + c) * L;
      rk = rq + static_cast<size_t>(C) * L;
      rv = rk + static_cast<size_t>(C) * L;
    }
    __syncthreads();  // the previous row's readers of the tables are done
    for (int i = threadIdx.x; i < nb * MB * 32; i += THREADS) {
      const int p = i >> 5, l = i & 31;
      const double lam = p < np ? poles[static_cast<size_t>(g) * np + p] : 0.0;
      s_pl[p][l] = static_cast<A>(pow(lam, static_cast<double>(S * l)));
      if (l < 5) s_pk[p][l] = static_cast<A>(pow(lam, static_cast<double>(S << l)));
      if (l <= WARPS) s_pw[p][l] = pow(lam, static_cast<double>(32 * S * l));
      if (l == 0) {
        s_lam[p] = static_cast<A>(lam);
        s_r[p] = p < np ? static_cast<A>(res[static_cast<size_t>(g) * np + p]) : A(0);
        s_carry[p] = 0.0;
      }
    }
    __syncthreads();
    const size_t base = static_cast<size_t>(row) * L;
    for (int t0 = 0; t0 < L; t0 += TILE) {
      const int ts = t0 + threadIdx.x * S;
      const int nv = max(0, min(S, L - ts));
      if (VEC && threadIdx.x < 3) {
        // the rows LA tiles ahead into L2 while this one computes (the loads below are
        // latency-bound at 16 warps per SM; no registers or shared memory are spent on it)
        const T* pr = FEAT ? (threadIdx.x == 0 ? rq : threadIdx.x == 1 ? rk : rv)
                           : (threadIdx.x == 0 ? q : threadIdx.x == 1 ? k : v);
        if (pr != nullptr) {
          if (!FEAT) pr += base;
          for (int a = t0 == 0 ? 1 : LA; a <= LA; ++a) {
            const int tn = t0 + a * TILE;
            const int n = min(TILE, L - tn);
            const unsigned bytes = n > 0 ? static_cast<unsigned>(n * sizeof(T)) & ~15u : 0u;
            if (bytes)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pr + tn), "r"(bytes) : "memory");
          }
        }
      }
      A u[S], yv[S];
      auto fir = [&](const A* r, const A* h, A* o) {
        if constexpr (PAIR) fir8_pairs<S>(r, h, o);
        else fir8<A, S>(r, h, o);
      };
      if constexpr (FEAT) {
        A raw[S + 8], fk[S];
        load_halo_seg<T, S, VEC>(rv, ts, L, raw);
        fir(raw, fh[2], u);
        load_halo_seg<T, S, VEC>(rk, ts, L, raw);
        fir(raw, fh[1], fk);
#pragma unroll
        for (int j = 0; j < S; ++j) u[j] *= fk[j];
      } else {
        load_seg<T, S, VEC>(v + base + ts, nv, u);
        if (k != nullptr) {
          A kk[S];
          load_seg<T, S, VEC>(k + base + ts, nv, kk);
#pragma unroll
          for (int j = 0; j < S; ++j) u[j] *= kk[j];
        }
      }
#pragma unroll
      for (int j = 0; j < S; ++j) yv[j] = A(0);
      float2 uu[PAIR ? S : 1];  // (u, u): the packed FFMA2 addend, built once per tile
      if constexpr (PAIR) {
#pragma unroll
        for (int j = 0; j < S; ++j) uu[j] = make_float2(u[j], u[j]);
      }
      for (int b = 0; b < nb; ++b, ++it) {
        const int buf = it & 1;
        A lam[MB], st[MB];
#pragma unroll
        for (int n = 0; n < MB; ++n) lam[n] = s_lam[b * MB + n];
        // 1. segment end state from zero
        if constexpr (PAIR) {
#pragma unroll
          for (int n = 0; n < MB; n += 2) {
            const float2 l2 = make_float2(lam[n], lam[n + 1]);
            float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < S; ++j) s2 = __ffma2_rn(l2, s2, uu[j]);
            st[n] = s2.x;
            st[n + 1] = s2.y;
          }
        } else {
#pragma unroll
          for (int n = 0; n < MB; ++n) {
            A s = A(0);
#pragma unroll
            for (int j = 0; j < S; ++j) s = fma(lam[n], s, u[j]);
            st[n] = s;
          }
        }
        // 2. inclusive scan over the warp's lanes
#pragma unroll
        for (int kk = 0; kk < 5; ++kk) {
          const int d = 1 << kk;
#pragma unroll
          for (int n = 0; n < MB; ++n) {
            const A o = __shfl_up_sync(0xffffffffu, st[n], d);
            if (lane >= d) st[n] = fma(s_pk[b * MB + n][kk], o, st[n]);
          }
        }
        if (lane == 31) {
#pragma unroll
          for (int n = 0; n < MB; ++n) s_tot[buf][warp][n] = st[n];
        }
        __syncthreads();
        // 3. this warp's incoming state (lane n < MB computes mode n, fp64)
        A inw_l = A(0);
        if (lane < MB) {
          const int p = b * MB + lane;
          double acc = s_carry[p] * s_pw[p][warp];
          for (int w = 0; w < warp; ++w) acc += s_pw[p][warp - 1 - w] * static_cast<double>(s_tot[buf][w][lane]);
          inw_l = static_cast<A>(acc);
        }
        // 4. each lane's incoming state, then the recurrence again with the output sum
#pragma unroll
        for (int n = 0; n < MB; ++n) {
          const A inw = __shfl_sync(0xffffffffu, inw_l, n);
          A ex = __shfl_up_sync(0xffffffffu, st[n], 1);
          if (lane == 0) ex = A(0);
          st[n] = fma(s_pl[b * MB + n][lane], inw, ex);
        }
        __syncthreads();  // every warp has read s_carry / s_tot[buf]
        if (warp == 0 && lane < MB) {
          const int p = b * MB + lane;
          double acc = s_carry[p] * s_pw[p][WARPS];
          for (int w = 0; w < WARPS; ++w) acc += s_pw[p][WARPS - 1 - w] * static_cast<double>(s_tot[buf][w][lane]);
          s_carry[p] = acc;
        }
        if constexpr (PAIR) {
          float2 y2[S];
#pragma unroll
          for (int j = 0; j < S; ++j) y2[j] = make_float2(0.f, 0.f);
#pragma unroll
          for (int n = 0; n < MB; n += 2) {
            const float2 l2 = make_float2(lam[n], lam[n + 1]);
            const float2 r2 = make_float2(s_r[b * MB + n], s_r[b * MB + n + 1]);
            float2 s2 = make_float2(st[n], st[n + 1]);
#pragma unroll
            for (int j = 0; j < S; ++j) {
              s2 = __ffma2_rn(l2, s2, uu[j]);
              y2[j] = __ffma2_rn(r2, s2, y2[j]);
            }
          }
#pragma unroll
          for (int j = 0; j < S; ++j) yv[j] += y2[j].x + y2[j].y;
        } else {
#pragma unroll
          for (int n = 0; n < MB; ++n) {
            const A r = s_r[b * MB + n];
            A s = st[n];
#pragma unroll
            for (int j = 0; j < S; ++j) {
              s = fma(lam[n], s, u[j]);
              yv[j] = fma(r, s, yv[j]);
            }
          }
        }
      }
      if constexpr (FEAT) {
        A raw[S + 8], fq[S];
        load_halo_seg<T, S, VEC>(rq, ts, L, raw);
        fir(raw, fh[0], fq);
#pragma unroll
        for (int j = 0; j < S; ++j) yv[j] *= fq[j];
      } else if (q != nullptr) {
        A qq[S];
        load_seg<T, S, VEC>(q + base + ts, nv, qq);
#pragma unroll
        for (int j = 0; j < S; ++j) yv[j] *= qq[j];
      }
      store_seg<T, S, VEC>(y + base + ts, nv, yv);
    }
  }
}

// ---------------------------------------------------------------- pipelined variant
// 16-byte aligned rows (the common case): each CTA of PW warps stages its next tile (all q / k / v
// rows, plus an 8-step featurizer history for FEAT) into shared memory with cp.async while it
// computes the current one, so the row loads' latency overlaps the scan instead of stalling it
// (the one-shot version above is latency-bound: ncu long-scoreboard stalls 4.5 per issue).
// Segments live in 16-byte-padded slots (slot pitch SB + 16), which makes every lane's 16-byte
// reads conflict-free; the fp32 recurrences run as packed FFMA2 on mode pairs.
constexpr int PW = 4;            // warps per CTA
constexpr int PMAXP = 16;        // poles per group in the pipelined kernel (else the one-shot one)

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <typename T>
struct PipeCfg {
  static constexpr int S = Cfg<T>::S;
  static constexpr int SB = S * static_cast<int>(sizeof(T));  // slot payload (bytes)
  static constexpr int SP = SB + 16;                          // slot pitch
  static constexpr int SLOTS = PW * 32 + 1;                   // slot 0: the history before the tile
  static constexpr int TENSOR_BYTES = SLOTS * SP;
  static constexpr int STAGE_BYTES = 3 * TENSOR_BYTES;
  static constexpr int SMEM = 2 * STAGE_BYTES;
};

// fp32 recurrence helpers on mode pairs (packed FFMA2) / scalars (fp64)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

template <typename T, bool FEAT>
__global__ void __launch_bounds__(PW * 32)
li_scan_pipe_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v, T* __restrict__ y,
                    const double* __restrict__ res, const double* __restrict__ poles, int np, int gs, int C, int L,
                    long long rows, const void* __restrict__ feat_raw, int lhf) {
  using A = typename Cfg<T>::A;
  using FT = typename std::conditional<sizeof(T) == 8, double, float>::type;
  using PC = PipeCfg<T>;
  constexpr int S = PC::S, TILE = PW * 32 * S, NT = PW * 32;
  constexpr int PER = 16 / static_cast<int>(sizeof(T));  // elements per 16-byte chunk
  constexpr int CH = PC::SB / 16;                          // chunks per slot
  constexpr bool PAIR = sizeof(A) == 4;                    // FFMA2 on mode pairs
  extern __shared__ __align__(16) unsigned char stage[];
  __shared__ A s_lam[PMAXP], s_r[PMAXP];
  __shared__ A s_pk[PMAXP][5];
  __shared__ A s_pl[PMAXP][32];
  __shared__ double s_pw[PMAXP][PW + 1];
  __shared__ double s_carry[PMAXP];
  __shared__ A s_tot[2][PW][MB];
  const FT* feat = static_cast<const FT*>(feat_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = (np + MB - 1) / MB;
  const bool gk = FEAT || k != nullptr, gq = FEAT || q != nullptr;
  int it = 0;
  for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
    const int c = static_cast<int>(row % C);
    const int g = c / gs;
    A fh[3][8];
    const T* src[3];  // [q, k, v] rows
    if constexpr (FEAT) {
#pragma unroll
      for (int x = 0; x < 3; ++x)
#pragma unroll
        for (int j = 0; j < 8; ++j)
          fh[x][j] = j < lhf ? static_cast<A>(feat[(static_cast<size_t>(x) * C + c) * lhf + j]) : A(0);
      const long long b = row / C;
      src[0] = q + (static_cast<size_t>(b) * 3 * C + c) * L;
      src[1] = src[0] + static_cast<size_t>(C) * L;
      src[2] = src[1] + static_cast<size_t>(C) * L;
    } else {
      const size_t base = static_cast<size_t>(row) * L;
      src[0] = q ? q + base : nullptr;
      src[1] = k ? k + base : nullptr;
      src[2] = v + base;
    }
    // stage tile t0 into buffer sb: slot 1 + i = steps [t0 + S i, t0 + S (i + 1)); slot 0 = the S
    // steps before t0 (FEAT history); bytes past L (or before 0) are zero-filled
    auto stage_tile = [&](int t0, int sb) {
      const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(stage)) + sb * PC::STAGE_BYTES;
#pragma unroll
      for (int x = 0; x < 3; ++x) {
        if ((x == 0 && !gq) || (x == 1 && !gk)) continue;
        const uint32_t tb = sbase + x * PC::TENSOR_BYTES;
        const int t = t0 + threadIdx.x * S;
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
          const int e = t + ch * PER;
          const int nbytes = max(0, min(16, (L - e) * static_cast<int>(sizeof(T))));
          cp_async16(tb + (threadIdx.x + 1) * PC::SP + ch * 16, nbytes ? src[x] + e : src[x], nbytes);
        }
        if (FEAT && threadIdx.x == 0) {
#pragma unroll
          for (int ch = 0; ch < CH; ++ch) {
            const int e = t0 - S + ch * PER;
            cp_async16(tb + ch * 16, e >= 0 ? src[x] + e : src[x], e >= 0 ? 16 : 0);
          }
        }
      }
      cp_async_commit();
    };
    __syncthreads();  // the previous row's readers of the tables and stages are done
    stage_tile(0, it & 1);
    for (int i = threadIdx.x; i < nb * MB * 32; i += NT) {
      const int p = i >> 5, l = i & 31;
      const double lam = p < np ? poles[static_cast<size_t>(g) * np + p] : 0.0;
      s_pl[p][l] = static_cast<A>(pow(lam, static_cast<double>(S * l)));
      if (l < 5) s_pk[p][l] = static_cast<A>(pow(lam, static_cast<double>(S << l)));
      if (l <= PW) s_pw[p][l] = pow(lam, static_cast<double>(32 * S * l));
      if (l == 0) {
        s_lam[p] = static_cast<A>(lam);
        s_r[p] = p < np ? static_cast<A>(res[static_cast<size_t>(g) * np + p]) : A(0);
        s_carry[p] = 0.0;
      }
    }
    for (int t0 = 0; t0 < L; t0 += TILE, ++it) {
      const int sb = it & 1;
      cp_async_wait_all();
      __syncthreads();  // this tile landed everywhere; the other buffer's readers (last tile) are done
      if (t0 + TILE < L) stage_tile(t0 + TILE, sb ^ 1);
      const unsigned char* stb = stage + sb * PC::STAGE_BYTES;
      // this lane's S steps (and FEAT: the 8 before them) of tensor x from its slot(s)
      auto read = [&](int x, A* out, bool halo) {
        const unsigned char* tb = stb + x * PC::TENSOR_BYTES;
        if (halo) {  // 8 steps = the last 8 * sizeof(T) bytes of the previous slot
          constexpr int HB = 8 * static_cast<int>(sizeof(T));
#pragma unroll
          for (int ch = 0; ch < HB / 16; ++ch) {
            const int4 raw = *reinterpret_cast<const int4*>(tb + threadIdx.x * PC::SP + PC::SB - HB + ch * 16);
            const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
            for (int j = 0; j < PER; ++j) out[ch * PER + j] = Elem<T>::to_a(e[j]);
          }
          out += 8;
        }
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
          const int4 raw = *reinterpret_cast<const int4*>(tb + (threadIdx.x + 1) * PC::SP + ch * 16);
          const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
          for (int j = 0; j < PER; ++j) out[ch * PER + j] = Elem<T>::to_a(e[j]);
        }
      };
      A u[S], fq[S];
      if constexpr (FEAT) {
        A raw[S + 8], fk[S];
        auto fir = [&](const A* r, const A* h, A* o) {
          if constexpr (PAIR) fir8_pairs<S>(r, h, o);
          else fir8<A, S>(r, h, o);
        };
        read(2, raw, true);
        fir(raw, fh[2], u);
        read(1, raw, true);
        fir(raw, fh[1], fk);
#pragma unroll
        for (int j = 0; j < S; ++j) u[j] *= fk[j];
        read(0, raw, true);
        fir(raw, fh[0], fq);
      } else {
        read(2, u, false);
        if (gk) {
          A kk[S];
          read(1, kk, false);
#pragma unroll
          for (int j = 0; j < S; ++j) u[j] *= kk[j];
        }
        if (gq) read(0, fq, false);
      }
      A yv[S];
#pragma unroll
      for (int j = 0; j < S; ++j) yv[j] = A(0);
      float2 uu[PAIR ? S : 1];  // (u, u): the packed FFMA2 addend, built once per tile
      if constexpr (PAIR) {
#pragma unroll
        for (int j = 0; j < S; ++j) uu[j] = make_float2(u[j], u[j]);
      }
      for (int b = 0; b < nb; ++b) {
        const int buf = (it * nb + b) & 1;
        A lam[MB], st[MB];
#pragma unroll
        for (int n = 0; n < MB; ++n) lam[n] = s_lam[b * MB + n];
        // 1. segment end states from zero
        if constexpr (PAIR) {
#pragma unroll
          for (int n = 0; n < MB; n += 2) {
            const float2 l2 = make_float2(lam[n], lam[n + 1]);
            float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
            for (int j = 0; j < S; ++j) s2 = ffma2(l2, s2, uu[j]);
            st[n] = s2.x;
            st[n + 1] = s2.y;
          }
        } else {
#pragma unroll
          for (int n = 0; n < MB; ++n) {
            A s = A(0);
#pragma unroll
            for (int j = 0; j < S; ++j) s = fma(lam[n], s, u[j]);
            st[n] = s;
          }
        }
        // 2. inclusive scan over the warp's lanes
#pragma unroll
        for (int kk = 0; kk < 5; ++kk) {
          const int d = 1 << kk;
#pragma unroll
          for (int n = 0; n < MB; ++n) {
            const A o = __shfl_up_sync(0xffffffffu, st[n], d);
            if (lane >= d) st[n] = fma(s_pk[b * MB + n][kk], o, st[n]);
          }
        }
        if (lane == 31) {
#pragma unroll
          for (int n = 0; n < MB; ++n) s_tot[buf][warp][n] = st[n];
        }
        __syncthreads();
        // 3. this warp's incoming state (lane n < MB computes mode n, fp64)
        A inw_l = A(0);
        if (lane < MB) {
          const int p = b * MB + lane;
          double acc = s_carry[p] * s_pw[p][warp];
          for (int w = 0; w < warp; ++w) acc += s_pw[p][warp - 1 - w] * static_cast<double>(s_tot[buf][w][lane]);
          inw_l = static_cast<A>(acc);
        }
#pragma unroll
        for (int n = 0; n < MB; ++n) {
          const A inw = __shfl_sync(0xffffffffu, inw_l, n);
          A ex = __shfl_up_sync(0xffffffffu, st[n], 1);
          if (lane == 0) ex = A(0);
          st[n] = fma(s_pl[b * MB + n][lane], inw, ex);
        }
        __syncthreads();  // every warp has read s_carry / s_tot[buf]
        if (warp == 0 && lane < MB) {
          const int p = b * MB + lane;
          double acc = s_carry[p] * s_pw[p][PW];
          for (int w = 0; w < PW; ++w) acc += s_pw[p][PW - 1 - w] * static_cast<double>(s_tot[buf][w][lane]);
          s_carry[p] = acc;
        }
        // 4. the recurrence again from the incoming states, R_n s_n[t] summed into y
        if constexpr (PAIR) {
          float2 y2[S];
#pragma unroll
          for (int j = 0; j < S; ++j) y2[j] = make_float2(0.f, 0.f);
#pragma unroll
          for (int n = 0; n < MB; n += 2) {
            const float2 l2 = make_float2(lam[n], lam[n + 1]);
            const float2 r2 = make_float2(s_r[b * MB + n], s_r[b * MB + n + 1]);
            float2 s2 = make_float2(st[n], st[n + 1]);
#pragma unroll
            for (int j = 0; j < S; ++j) {
              s2 = ffma2(l2, s2, uu[j]);
              y2[j] = ffma2(r2, s2, y2[j]);
            }
          }
#pragma unroll
          for (int j = 0; j < S; ++j) yv[j] += y2[j].x + y2[j].y;
        } else {
#pragma unroll
          for (int n = 0; n < MB; ++n) {
            const A r = s_r[b * MB + n];
            A s = st[n];
#pragma unroll
            for (int j = 0; j < S; ++j) {
              s = fma(lam[n], s, u[j]);
              yv[j] = fma(r, s, yv[j]);
            }
          }
        }
      }
      if (gq) {
#pragma unroll
        for (int j = 0; j < S; ++j) yv[j] *= fq[j];
      }
      const int ts = t0 + threadIdx.x * S;
      store_seg<T, S, true>(y + static_cast<size_t>(row) * L + ts, max(0, min(S, L - ts)), yv);
    }
  }
}

template <typename T, bool FEAT = false>
int launch(const void* q, const void* k, const void* v, void* y, const double* res, const double* poles, int np,
           int gs, int B, int C, int L, cudaStream_t st, const void* feat = nullptr, int lhf = 0) {
  const bool vec = (static_cast<size_t>(L) * sizeof(T)) % 16 == 0 && aligned16(y) && (!v || aligned16(v)) &&
                   (!q || aligned16(q)) && (!k || aligned16(k));
  const long long rows = static_cast<long long>(B) * C;
  // the pipelined kernel wins for bf16 rows (1.80 vs 2.20 ms for the C3 mixer); fp32 rows stay on
  // the one-shot kernel (2.60 vs 2.87 ms: with fp32 slots its shared-memory ring caps the SM at
  // 12 warps, and the kernel turns issue-latency bound, ncu mio / short-scoreboard stalls)
  static const int mode = [] { const char* e = getenv("HY_LI_SCAN_PIPE"); return e ? atoi(e) : -1; }();
  const bool pipe = mode < 0 ? sizeof(T) == 2 : mode != 0;
  if (vec && np <= PMAXP && pipe) {
    auto pk = li_scan_pipe_kernel<T, FEAT>;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(pk), PipeCfg<T>::SMEM);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    const long long pcap = resident_cap(reinterpret_cast<const void*>(pk), PW * 32, PipeCfg<T>::SMEM);
    const long long pgrid = rows < pcap ? rows : pcap;
    pk<<<static_cast<int>(pgrid), PW * 32, PipeCfg<T>::SMEM, st>>>(
        static_cast<const T*>(q), static_cast<const T*>(k), static_cast<const T*>(v), static_cast<T*>(y), res, poles,
        np, gs, C, L, rows, feat, lhf);
    return check_launch("li_scan_pipe_kernel");
  }
  auto kern = vec ? li_scan_kernel<T, true, FEAT> : li_scan_kernel<T, false, FEAT>;
  const long long cap = resident_cap(reinterpret_cast<const void*>(kern), THREADS, 0);
  const long long grid = rows < cap ? rows : cap;
  kern<<<static_cast<int>(grid), THREADS, 0, st>>>(static_cast<const T*>(q), static_cast<const T*>(k),
                                                   static_cast<const T*>(v), static_cast<T*>(y), res, poles, np, gs,
                                                   C, L, rows, feat, lhf);
  return check_launch("li_scan_kernel");
}

}  // namespace lis
}  // namespace hy

using namespace hy;

extern "C" HY_API int hy_li_scan_fwd(const void* q, const void* k, const void* v, void* y, const double* residues,
                                     const double* poles, int npoles, int gs, int B, int C, int L, int dtype,
                                     void* stream) {
  if (!v || !y || !residues || !poles) return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || gs < 1) return fail(HY_ERR_INVALID, "sizes must be >= 1");
  if (C % gs != 0) return fail(HY_ERR_INVALID, "group_size %d does not divide channel count %d", gs, C);
  if (npoles < 1 || npoles > lis::MAXP) return fail(HY_ERR_UNSUPPORTED, "modal scan supports 1..%d poles", lis::MAXP);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == HY_F32) return lis::launch<float>(q, k, v, y, residues, poles, npoles, gs, B, C, L, st);
  if (dtype == HY_BF16) return lis::launch<__nv_bfloat16>(q, k, v, y, residues, poles, npoles, gs, B, C, L, st);
  if (dtype == HY_F64) return lis::launch<double>(q, k, v, y, residues, poles, npoles, gs, B, C, L, st);
  return fail(HY_ERR_UNSUPPORTED, "hy_li_scan_fwd: unknown dtype %d", dtype);
}

// Fused LI mixer on the modal scan: featurizers (lhf <= 8) + u = k*v + implicit long conv + q gate
// from the (B, 3C, L) projections, one pass (hyena.py:162-186 for variant LI).
extern "C" HY_API int hy_li_scan_mixer_fwd(const void* proj, void* y, const void* feat_taps, int lhf,
                                           const double* residues, const double* poles, int npoles, int gs, int B,
                                           int C, int L, int dtype, void* stream) {
  if (!proj || !y || !feat_taps || !residues || !poles) return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || gs < 1) return fail(HY_ERR_INVALID, "sizes must be >= 1");
  if (C % gs != 0) return fail(HY_ERR_INVALID, "group_size %d does not divide channel count %d", gs, C);
  if (lhf < 1 || lhf > 8) return fail(HY_ERR_UNSUPPORTED, "fused modal-scan mixer needs featurizer length <= 8");
  if (npoles < 1 || npoles > lis::MAXP) return fail(HY_ERR_UNSUPPORTED, "modal scan supports 1..%d poles", lis::MAXP);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == HY_F32)
    return lis::launch<float, true>(proj, nullptr, nullptr, y, residues, poles, npoles, gs, B, C, L, st, feat_taps, lhf);
  if (dtype == HY_BF16)
    return lis::launch<__nv_bfloat16, true>(proj, nullptr, nullptr, y, residues, poles, npoles, gs, B, C, L, st,
                                            feat_taps, lhf);
  if (dtype == HY_F64)
    return lis::launch<double, true>(proj, nullptr, nullptr, y, residues, poles, npoles, gs, B, C, L, st, feat_taps, lhf);
  return fail(HY_ERR_UNSUPPORTED, "hy_li_scan_mixer_fwd: unknown dtype %d", dtype);
}
