// Register-blocked four-step FFT causal convolution (the fast path of hy_fft_conv_fwd for
// 2^14 <= N <= 2^18, i.e. the long-filter / LI-FFT sizes of config C3):
//
//     y[t] = q[t] * (h conv (k * v))[t] = q * IFFT(FFT(pad(k * v)) . FFT(pad(h)))[t] / N
//
// (fft.py:128-145 / hyena.py:183-186), N = N1 * M with the row length M = 8192 fixed and
// N1 = N / M in {2, ..., 32}; n = M n1 + n2, k = k1 + N1 k2.
//
//   column pass  one thread per column n2: the N1 samples x[M n1 + n2] (k * v or the taps,
//                zero padded; coalesced across threads) are transformed in registers
//                (radix-2 network, natural order in and out), times W_N^(n2 k1), stored as
//                row k1
//   row pass     one CTA per row (k1, channel): 8192 = 32 x 16 x 16, each stage one
//                register radix-32 / radix-16 DFT per thread between shared-memory
//                exchanges. The first stage reads the row straight from HBM and the last
//                writes it straight back; the last forward stage and the first inverse
//                stage work on the same 16-element groups, so the spectrum product sits
//                between them in registers: 4 shared-memory round trips for forward +
//                product + inverse (a radix-2^2 loop needs 13). Spectra stay in the
//                transform's digit-reversed order; the filter spectrum is produced by the
//                same forward stages, so no permutation pass exists anywhere.
//   inverse col  one thread per column: inverse register DFT over k1, 1/N, gate q, store y
//
// Shared rows are padded by one element per 16 (conflict-free half-warp access at every
// stage). Twiddles are two-level tables (64-entry fine x coarse) evaluated in double
// precision, so each twiddle is one complex product of exactly rounded factors.
#include <cstdint>

#include "common.cuh"
#include "internal.h"

namespace hy {
namespace fftf {

constexpr int M = 8192;  // row length
constexpr int ROW_THREADS = 256;
constexpr int COL_THREADS = 128;
constexpr int PHYS = M + M / 16;  // padded shared row
constexpr int ROW_SMEM = (PHYS + 128 + 32) * 8;

// cos / sin of 2 pi e / 32 (compile-time twiddles of the register DFTs)
__host__ __device__ constexpr float w32c(int e) {
  switch (e) {
    case 0: return 1.000000000e+00f;
    case 1: return 9.807852804e-01f;
    case 2: return 9.238795325e-01f;
    case 3: return 8.314696123e-01f;
    case 4: return 7.071067812e-01f;
    case 5: return 5.555702330e-01f;
    case 6: return 3.826834324e-01f;
    case 7: return 1.950903220e-01f;
    case 8: return 6.123233996e-17f;
    case 9: return -1.950903220e-01f;
    case 10: return -3.826834324e-01f;
    case 11: return -5.555702330e-01f;
    case 12: return -7.071067812e-01f;
    case 13: return -8.314696123e-01f;
    case 14: return -9.238795325e-01f;
    case 15: return -9.807852804e-01f;
    default: return 0.f;
  }
}
__host__ __device__ constexpr float w32s(int e) {
  switch (e) {
    case 0: return 0.000000000e+00f;
    case 1: return 1.950903220e-01f;
    case 2: return 3.826834324e-01f;
    case 3: return 5.555702330e-01f;
    case 4: return 7.071067812e-01f;
    case 5: return 8.314696123e-01f;
    case 6: return 9.238795325e-01f;
    case 7: return 9.807852804e-01f;
    case 8: return 1.000000000e+00f;
    case 9: return 9.807852804e-01f;
    case 10: return 9.238795325e-01f;
    case 11: return 8.314696123e-01f;
    case 12: return 7.071067812e-01f;
    case 13: return 5.555702330e-01f;
    case 14: return 3.826834324e-01f;
    case 15: return 1.950903220e-01f;
    default: return 0.f;
  }
}

__device__ __forceinline__ int phys(int i) { return i + (i >> 4); }

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

template <int R>
__host__ __device__ constexpr int brev(int i) {
  int r = 0;
  for (int b = 1; b < R; b <<= 1) {
    r = (r << 1) | (i & 1);
    i >>= 1;
  }
  return r;
}

// In-register DFT of R = 2..32 points, natural order in and out: a radix-2 decimation-in-
// frequency network with compile-time twiddles, then the bit-reversal as register renaming.
// Forward uses exp(-2 pi i / R); INV the conjugate (unnormalised).
template <int R, bool INV>
__device__ __forceinline__ void dft(float2 (&v)[R]) {
#pragma unroll
  for (int span = R; span >= 2; span >>= 1) {
    const int h = span >> 1;
#pragma unroll
    for (int base = 0; base < R; base += span) {
#pragma unroll
      for (int j = 0; j < h; ++j) {
        const float2 a = v[base + j], b = v[base + j + h];
        v[base + j] = make_float2(a.x + b.x, a.y + b.y);
        const float2 d = make_float2(a.x - b.x, a.y - b.y);
        const int e = j * (32 / span);
        if (e == 0) {
          v[base + j + h] = d;
        } else if (e == 8) {
          v[base + j + h] = INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x);
        } else {
          const float c = w32c(e), s = INV ? w32s(e) : -w32s(e);
          v[base + j + h] = make_float2(d.x * c - d.y * s, d.x * s + d.y * c);
        }
      }
    }
  }
  float2 t[R];
#pragma unroll
  for (int i = 0; i < R; ++i) t[i] = v[brev<R>(i)];
#pragma unroll
  for (int i = 0; i < R; ++i) v[i] = t[i];
}

// exp(-2 pi i l / n) for 0 <= l < 64 and n >= 8192 (angle < 0.05): Taylor terms to x^5 are
// exact to fp32 rounding, so the fine factor of a twiddle costs FMAs, not a table read.
__device__ __forceinline__ float2 w_fine(int l, float step) {
  const float x = static_cast<float>(l) * step, x2 = x * x;
  const float c = fmaf(x2, fmaf(x2, 1.f / 24.f, -0.5f), 1.f);
  const float s = x * fmaf(x2, fmaf(x2, 1.f / 120.f, -1.f / 6.f), 1.f);
  return make_float2(c, -s);
}

// W_N^e = hi[e >> 6] * fine(e & 63): hi[m] = W_N^(64 m) from the global table (double precision).
__device__ __forceinline__ float2 tw_n(const float2* __restrict__ hi, int e, float step) {
  return cmul(__ldg(hi + (e >> 6)), w_fine(e & 63, step));
}

__global__ void table_kernel(float2* hi, float2* lo, int N) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int nhi = N / 64;
  if (i >= nhi + 64) return;
  const long long e = i < nhi ? 64LL * i : i - nhi;
  double s, c;
  sincospi(-2.0 * static_cast<double>(e) / static_cast<double>(N), &s, &c);
  (i < nhi ? hi[i] : lo[i - nhi]) = make_float2(static_cast<float>(c), static_cast<float>(s));
}

template <typename T>
__device__ __forceinline__ float ldf(const T* p) { return Elem<T>::to_a(*p); }

// Column pass: a CTA covers COL_THREADS consecutive columns n2 of one row r (blockIdx.y);
// FILTER: group g0 + r's taps (length lh), else k * v of activation row row0 + r (length L).
// The N1 x COL_THREADS input tile is staged through shared memory — with 16-byte streaming
// loads when rows are 16-byte aligned (L a multiple of the vector width) — then every thread
// transforms its column in registers and stores row k1 of r's N-point workspace row.
// PAIR (activations only, filter groups of even size): block row r carries the two channels
// row0 + 2r and row0 + 2r + 1, which share a filter, as the real and imaginary parts of one
// complex sequence: IFFT((A + iB) H) = A*h + i B*h for real a, b, h, so one complex transform
// pair does the work of two (the reference's real-input FFT conv, two channels at a time).
template <typename T, int N1, bool FILTER, bool PAIR = false>
__global__ void __launch_bounds__(COL_THREADS) col_fwd(float2* __restrict__ X, const float2* __restrict__ hi,
                                                       const float2* __restrict__ lo, const T* __restrict__ k,
                                                       const T* __restrict__ v, const float* __restrict__ taps,
                                                       int row0, int g0, int L, int lh, int N) {
  constexpr int VEC = Elem<T>::VEC, VPR = COL_THREADS / VEC;
  __shared__ __align__(16) float tile[(PAIR ? 2 : 1) * N1 * COL_THREADS];
  const int n2_0 = blockIdx.x * COL_THREADS, tid = threadIdx.x, n2 = n2_0 + tid;
  const int r = blockIdx.y;
  (void)lo;
  for (int part = 0; part < (PAIR ? 2 : 1); ++part) {
  float* tl = tile + part * N1 * COL_THREADS;
  const int arow = PAIR ? row0 + 2 * r + part : row0 + r;
  if (!FILTER && L % VEC == 0) {
    const size_t rowoff = static_cast<size_t>(arow) * L;
    for (int i = tid; i < N1 * VPR; i += COL_THREADS) {
      const int n1 = i / VPR, jv = i % VPR;
      const int t = n1 * M + n2_0 + jv * VEC;
      float val[VEC];
      if (t < L) {
        unpack16<T>(ld_stream16(v + rowoff + t), val);
        if (k) {
          float kk[VEC];
          unpack16<T>(ld_stream16(k + rowoff + t), kk);
#pragma unroll
          for (int e = 0; e < VEC; ++e) val[e] *= kk[e];
        }
      } else {
#pragma unroll
        for (int e = 0; e < VEC; ++e) val[e] = 0.f;
      }
      float4* dst = reinterpret_cast<float4*>(tl + n1 * COL_THREADS + jv * VEC);
#pragma unroll
      for (int e = 0; e < VEC / 4; ++e) dst[e] = make_float4(val[4 * e], val[4 * e + 1], val[4 * e + 2], val[4 * e + 3]);
    }
  } else if (FILTER && lh % 4 == 0) {  // fp32 taps rows 16-byte aligned
    const float* trow = taps + static_cast<size_t>(g0 + r) * lh;
    for (int i = tid; i < N1 * (COL_THREADS / 4); i += COL_THREADS) {
      const int n1 = i / (COL_THREADS / 4), jv = i % (COL_THREADS / 4);
      const int t = n1 * M + n2_0 + jv * 4;
      float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < lh) f = __ldg(reinterpret_cast<const float4*>(trow + t));
      *reinterpret_cast<float4*>(tl + n1 * COL_THREADS + jv * 4) = f;
    }
  } else {
    for (int i = tid; i < N1 * COL_THREADS; i += COL_THREADS) {
      const int t = (i / COL_THREADS) * M + n2_0 + i % COL_THREADS;
      float val = 0.f;
      if (FILTER) {
        if (t < lh) val = taps[static_cast<size_t>(g0 + r) * lh + t];
      } else if (t < L) {
        const size_t off = static_cast<size_t>(arow) * L + t;
        val = ldf(v + off);
        if (k) val *= ldf(k + off);
      }
      tl[i] = val;
    }
  }
  }
  __syncthreads();
  float2 x[N1];
#pragma unroll
  for (int n1 = 0; n1 < N1; ++n1)
    x[n1] = make_float2(tile[n1 * COL_THREADS + tid], PAIR ? tile[(N1 + n1) * COL_THREADS + tid] : 0.f);
  dft<N1, false>(x);
  const float step_n = 6.283185307179586f / static_cast<float>(N);
  float2* out = X + static_cast<size_t>(r) * N + n2;
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1)
    out[static_cast<size_t>(k1) * M] = k1 ? cmul(x[k1], tw_n(hi, (n2 * k1) & (N - 1), step_n)) : x[k1];
}

// Inverse column pass: inverse DFT over k1, then y = q * Re(x) / N for t < L, the output tile
// staged through shared memory for 16-byte stores (and gate loads) where rows are aligned.
template <typename T, int N1, bool PAIR = false>
__global__ void __launch_bounds__(COL_THREADS) col_inv(const float2* __restrict__ X, const T* __restrict__ q,
                                                       T* __restrict__ y, int row0, int L, int N) {
  constexpr int VEC = Elem<T>::VEC, VPR = COL_THREADS / VEC;
  __shared__ __align__(16) float tile[(PAIR ? 2 : 1) * N1 * COL_THREADS];
  const int n2_0 = blockIdx.x * COL_THREADS, tid = threadIdx.x, n2 = n2_0 + tid;
  const int r = blockIdx.y;
  const float2* in = X + static_cast<size_t>(r) * N + n2;
  float2 x[N1];
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) x[k1] = in[static_cast<size_t>(k1) * M];
  dft<N1, true>(x);
  const float scale = 1.f / static_cast<float>(N);
#pragma unroll
  for (int n1 = 0; n1 < N1; ++n1) {
    tile[n1 * COL_THREADS + tid] = x[n1].x * scale;
    if (PAIR) tile[(N1 + n1) * COL_THREADS + tid] = x[n1].y * scale;  // the odd channel of the pair
  }
  __syncthreads();
  for (int part = 0; part < (PAIR ? 2 : 1); ++part) {
  const float* tl = tile + part * N1 * COL_THREADS;
  const size_t rowoff = static_cast<size_t>(PAIR ? row0 + 2 * r + part : row0 + r) * L;
  if (L % VEC == 0) {
    for (int i = tid; i < N1 * VPR; i += COL_THREADS) {
      const int n1 = i / VPR, jv = i % VPR;
      const int t = n1 * M + n2_0 + jv * VEC;
      if (t >= L) continue;
      float val[VEC];
      const float4* src = reinterpret_cast<const float4*>(tl + n1 * COL_THREADS + jv * VEC);
#pragma unroll
      for (int e = 0; e < VEC / 4; ++e) {
        const float4 f = src[e];
        val[4 * e] = f.x;
        val[4 * e + 1] = f.y;
        val[4 * e + 2] = f.z;
        val[4 * e + 3] = f.w;
      }
      if (q) {
        float qq[VEC];
        unpack16<T>(ld_stream16(q + rowoff + t), qq);
#pragma unroll
        for (int e = 0; e < VEC; ++e) val[e] *= qq[e];
      }
      st_stream16(y + rowoff + t, pack16<T>(val));
    }
  } else {
    for (int i = tid; i < N1 * COL_THREADS; i += COL_THREADS) {
      const int t = (i / COL_THREADS) * M + n2_0 + i % COL_THREADS;
      if (t >= L) continue;
      float val = tl[i];
      if (q) val *= ldf(q + rowoff + t);
      y[rowoff + t] = Elem<T>::from_a(val);
    }
  }
  }
}

// W_M^e: coarse factor rhi[m] = W_M^(64 m) from shared memory, fine factor by polynomial
constexpr float STEP_M = 6.283185307179586f / M;
__device__ __forceinline__ float2 tw_m(const float2* rhi, int e) {
  return cmul(rhi[(e >> 6) & 127], w_fine(e & 63, STEP_M));
}

// Row pass over row k1 = blockIdx.x of block row r = blockIdx.y (X + r N + k1 M).
// FILTER: the forward transform is stored in place as the group spectrum. Else: forward,
// times the spectrum of the row's group, inverse, times W_N^(-n2 k1), in place.
template <bool FILTER>
__global__ void __launch_bounds__(ROW_THREADS, 2) row_kernel(float2* X, const float2* __restrict__ Hf,
                                                           const float2* __restrict__ hi,
                                                           const float2* __restrict__ lo, int N, int c0, int g0,
                                                           int gs) {
  extern __shared__ float2 sm[];
  float2* xs = sm;
  float2* rhi = sm + PHYS;
  const int k1 = blockIdx.x, r = blockIdx.y, tid = threadIdx.x;
  float2* rk1 = rhi + 128;  // [32] W_N^(256 a k1)
  if (tid < 128) {
    double s, c;
    sincospi(-2.0 * static_cast<double>(64 * tid) / static_cast<double>(M), &s, &c);
    rhi[tid] = make_float2(static_cast<float>(c), static_cast<float>(s));
  } else if (tid < 160) {
    const long long e = (256LL * (tid - 128) * k1) % N;
    double s, c;
    sincospi(-2.0 * static_cast<double>(e) / static_cast<double>(N), &s, &c);
    rk1[tid - 128] = make_float2(static_cast<float>(c), static_cast<float>(s));
  }
  float2* row = X + static_cast<size_t>(r) * N + static_cast<size_t>(k1) * M;
  const float step_n = 6.283185307179586f / static_cast<float>(N);
  (void)lo;
  const float2 w0 = FILTER ? make_float2(1.f, 0.f) : tw_n(hi, (tid * k1) & (N - 1), step_n);
  float2 v32[32];
  // A: DIF radix 32 over span M (group j = tid: x[j + 256 a]) straight from HBM
#pragma unroll
  for (int a = 0; a < 32; ++a) v32[a] = row[tid + 256 * a];
  __syncthreads();  // twiddle tables
  dft<32, false>(v32);
#pragma unroll
  for (int c = 0; c < 32; ++c) xs[phys(tid + 256 * c)] = c ? cmul(v32[c], tw_m(rhi, tid * c)) : v32[c];
  __syncthreads();
  // B: DIF radix 16 over span 256 (group (blk, j): x[256 blk + j + 16 a]), twiddle W_256^(j c)
#pragma unroll 1
  for (int gg = 0; gg < 2; ++gg) {
    const int g = tid + gg * ROW_THREADS, j = g & 15, base = (g >> 4) * 256;
    float2 v[16];
#pragma unroll
    for (int a = 0; a < 16; ++a) v[a] = xs[phys(base + j + 16 * a)];
    dft<16, false>(v);
#pragma unroll
    for (int c = 0; c < 16; ++c) xs[phys(base + j + 16 * c)] = c ? cmul(v[c], tw_m(rhi, 32 * j * c)) : v[c];
  }
  __syncthreads();
  // C: DIF radix 16 over span 16 -> spectrum at logical index 16 g + c; then (conv) the
  //    product and the first inverse stage on the same group
  const float2* hrow = nullptr;
  if (!FILTER) {
    const int grp = (c0 + r) / gs - g0;
    hrow = Hf + static_cast<size_t>(grp) * N + static_cast<size_t>(k1) * M;
  }
#pragma unroll 1
  for (int gg = 0; gg < 2; ++gg) {
    const int g = tid + gg * ROW_THREADS;
    float2 v[16];
#pragma unroll
    for (int a = 0; a < 16; ++a) v[a] = xs[phys(16 * g + a)];
    dft<16, false>(v);
    if (FILTER) {  // back to shared memory; stored coalesced below
#pragma unroll
      for (int c = 0; c < 16; ++c) xs[phys(16 * g + c)] = v[c];
    } else {
      const float4* h4 = reinterpret_cast<const float4*>(hrow + 16 * g);
#pragma unroll
      for (int c = 0; c < 16; c += 2) {
        const float4 hv = __ldg(h4 + c / 2);
        v[c] = cmul(v[c], make_float2(hv.x, hv.y));
        v[c + 1] = cmul(v[c + 1], make_float2(hv.z, hv.w));
      }
      dft<16, true>(v);
#pragma unroll
      for (int a = 0; a < 16; ++a) xs[phys(16 * g + a)] = v[a];
    }
  }
  __syncthreads();
  if (FILTER) {  // the spectrum row in logical order, coalesced
#pragma unroll 4
    for (int i = tid; i < M; i += ROW_THREADS) row[i] = xs[phys(i)];
    return;
  }
  // D: DIT radix 16 over span 256: conj twiddle, inverse DFT
#pragma unroll 1
  for (int gg = 0; gg < 2; ++gg) {
    const int g = tid + gg * ROW_THREADS, j = g & 15, base = (g >> 4) * 256;
    float2 v[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      const float2 x = xs[phys(base + j + 16 * c)];
      v[c] = c ? cmulc(x, tw_m(rhi, 32 * j * c)) : x;
    }
    dft<16, true>(v);
#pragma unroll
    for (int a = 0; a < 16; ++a) xs[phys(base + j + 16 * a)] = v[a];
  }
  __syncthreads();
  // E: DIT radix 32 over span M, times W_N^(-n2 k1), straight to HBM
#pragma unroll
  for (int c = 0; c < 32; ++c) {
    const float2 x = xs[phys(tid + 256 * c)];
    v32[c] = c ? cmulc(x, tw_m(rhi, tid * c)) : x;
  }
  dft<32, true>(v32);
#pragma unroll
  for (int a = 0; a < 32; ++a) {
    const int n2 = tid + 256 * a;
    // W_N^(n2 k1) = W_N^(tid k1) * W_N^(256 a k1): per-thread factor times a per-CTA table
    row[n2] = k1 ? cmulc(v32[a], cmul(w0, rk1[a])) : v32[a];
  }
}

// Row pass for channel pairs with per-channel filters (gs = 1). Block row r carries channels
// a = 2r, b = 2r + 1 (relative to the block) as Z = FFT(a + i b); with Zm(k) = conj(Z(-k)) the
// Hermitian symmetry of the real transforms gives A = (Z + Zm) / 2, B = (Z - Zm) / (2i), so
//     W(k) = A Ha + i B Hb = Z (Ha + Hb) / 2 + Zm (Ha - Hb) / 2,   IFFT(W) = a*ha + i (b*hb).
// -k lives in row N1 - k1 (row 0 and row N1/2: themselves), so a CTA of 2 x 256 threads takes the
// row pair (q, N1 - q): both forward transforms into shared memory, the mirror-bin product, both
// inverse transforms. Position p of a row after the forward stages holds frequency
// k2 = (p >> 8) + 32 ((p >> 4) & 15) + 512 (p & 15) (the DIF digit order of the 32 x 16 x 16 stages).
constexpr int PAIR_THREADS = 2 * ROW_THREADS;
constexpr int PAIR_SMEM = (2 * PHYS + 128 + 64) * 8;
__device__ __forceinline__ int rowpos_to_k2(int p) { return (p >> 8) + 32 * ((p >> 4) & 15) + 512 * (p & 15); }
__device__ __forceinline__ int k2_to_rowpos(int k) { return 256 * (k & 31) + 16 * ((k >> 5) & 15) + (k >> 9); }

__global__ void __launch_bounds__(PAIR_THREADS, 1) row_pair_kernel(float2* X, const float2* __restrict__ Hf,
                                                                  const float2* __restrict__ hi, int N, int N1) {
  extern __shared__ float2 sm[];
  const int q = blockIdx.x, r = blockIdx.y;
  const int half = threadIdx.x / ROW_THREADS, tid = threadIdx.x % ROW_THREADS;
  const bool self = (q == 0 || 2 * q == N1);
  const int k1 = half == 0 ? q : N1 - q;  // this half's row
  const bool active = half == 0 || !self;
  float2* xs = sm + half * PHYS;
  float2* rhi = sm + 2 * PHYS;
  float2* rk1 = rhi + 128 + 32 * half;  // [32] W_N^(256 a k1) of this half's row
  if (tid < 128) {
    if (half == 0) {
      double s, c;
      sincospi(-2.0 * static_cast<double>(64 * tid) / static_cast<double>(M), &s, &c);
      rhi[tid] = make_float2(static_cast<float>(c), static_cast<float>(s));
    }
  } else if (tid < 160) {
    const long long e = (256LL * (tid - 128) * k1) % N;
    double s, c;
    sincospi(-2.0 * static_cast<double>(e) / static_cast<double>(N), &s, &c);
    rk1[tid - 128] = make_float2(static_cast<float>(c), static_cast<float>(s));
  }
  float2* row = X + static_cast<size_t>(r) * N + static_cast<size_t>(k1) * M;
  const float step_n = 6.283185307179586f / static_cast<float>(N);
  const float2 w0 = tw_n(hi, (tid * k1) & (N - 1), step_n);
  float2 v32[32];
  // A: DIF radix 32 over span M from HBM
  if (active) {
#pragma unroll
    for (int a = 0; a < 32; ++a) v32[a] = row[tid + 256 * a];
  }
  __syncthreads();  // twiddle tables
  if (active) {
    dft<32, false>(v32);
#pragma unroll
    for (int c = 0; c < 32; ++c) xs[phys(tid + 256 * c)] = c ? cmul(v32[c], tw_m(rhi, tid * c)) : v32[c];
  }
  __syncthreads();
  // B: DIF radix 16 over span 256
  if (active) {
#pragma unroll 1
    for (int gg = 0; gg < 2; ++gg) {
      const int g = tid + gg * ROW_THREADS, j = g & 15, base = (g >> 4) * 256;
      float2 v[16];
#pragma unroll
      for (int a = 0; a < 16; ++a) v[a] = xs[phys(base + j + 16 * a)];
      dft<16, false>(v);
#pragma unroll
      for (int c = 0; c < 16; ++c) xs[phys(base + j + 16 * c)] = c ? cmul(v[c], tw_m(rhi, 32 * j * c)) : v[c];
    }
  }
  __syncthreads();
  // C: DIF radix 16 over span 16: the forward spectra of both rows in shared memory
  if (active) {
#pragma unroll 1
    for (int gg = 0; gg < 2; ++gg) {
      const int g = tid + gg * ROW_THREADS;
      float2 v[16];
#pragma unroll
      for (int a = 0; a < 16; ++a) v[a] = xs[phys(16 * g + a)];
      dft<16, false>(v);
#pragma unroll
      for (int a = 0; a < 16; ++a) xs[phys(16 * g + a)] = v[a];
    }
  }
  __syncthreads();
  // mirror-bin product: every position of this half's row, W = Z S + conj(Z(-k)) T with
  // S, T = (Ha +- Hb) / 2 read from the two channels' spectra at the same position
  const float2* ha = Hf + static_cast<size_t>(2 * r) * N + static_cast<size_t>(k1) * M;
  const float2* hb = ha + N;
  const float2* xm = sm + (self ? 0 : (1 - half)) * PHYS;  // the mirror row
  float2 w[32];
  if (active) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int p = tid + 256 * i;
      const int k2 = rowpos_to_k2(p);
      const int k2m = k1 == 0 ? (M - k2) & (M - 1) : M - 1 - k2;
      const float2 z = xs[phys(p)];
      const float2 zmv = xm[phys(k2_to_rowpos(k2m))];
      const float2 zm = make_float2(zmv.x, -zmv.y);
      const float2 a = __ldg(ha + p), b = __ldg(hb + p);
      const float2 S = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y + b.y));
      const float2 T = make_float2(0.5f * (a.x - b.x), 0.5f * (a.y - b.y));
      const float2 zs = cmul(z, S), zt = cmul(zm, T);
      w[i] = make_float2(zs.x + zt.x, zs.y + zt.y);
    }
  }
  __syncthreads();  // every mirror read is done before the rows are overwritten
  if (active) {
#pragma unroll
    for (int i = 0; i < 32; ++i) xs[phys(tid + 256 * i)] = w[i];
  }
  __syncthreads();
  // C': inverse radix 16 over span 16
  if (active) {
#pragma unroll 1
    for (int gg = 0; gg < 2; ++gg) {
      const int g = tid + gg * ROW_THREADS;
      float2 v[16];
#pragma unroll
      for (int a = 0; a < 16; ++a) v[a] = xs[phys(16 * g + a)];
      dft<16, true>(v);
#pragma unroll
      for (int a = 0; a < 16; ++a) xs[phys(16 * g + a)] = v[a];
    }
  }
  __syncthreads();
  // D: DIT radix 16 over span 256: conj twiddle, inverse DFT
  if (active) {
#pragma unroll 1
    for (int gg = 0; gg < 2; ++gg) {
      const int g = tid + gg * ROW_THREADS, j = g & 15, base = (g >> 4) * 256;
      float2 v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const float2 x = xs[phys(base + j + 16 * c)];
        v[c] = c ? cmulc(x, tw_m(rhi, 32 * j * c)) : x;
      }
      dft<16, true>(v);
#pragma unroll
      for (int a = 0; a < 16; ++a) xs[phys(base + j + 16 * a)] = v[a];
    }
  }
  __syncthreads();
  // E: DIT radix 32 over span M, times W_N^(-n2 k1), to HBM
  if (active) {
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const float2 x = xs[phys(tid + 256 * c)];
      v32[c] = c ? cmulc(x, tw_m(rhi, tid * c)) : x;
    }
    dft<32, true>(v32);
#pragma unroll
    for (int a = 0; a < 32; ++a) {
      const int n2 = tid + 256 * a;
      row[n2] = k1 ? cmulc(v32[a], cmul(w0, rk1[a])) : v32[a];
    }
  }
}

// One block of `rows` activation rows (channels c0.., batch row offset row0): column pass, row
// pass (times the group spectra Hf, relative to group g0), inverse column pass. Even group sizes
// go two channels per complex transform (PAIR): the row pass then sees channel pairs, i.e. c0 / 2
// and group size gs / 2 in its group arithmetic.
template <typename T, int N1>
void act_pass(float2* X, const float2* Hf, const float2* hi, const float2* lo, const void* q, const void* k,
              const void* v, void* y, int row0, int c0, int g0, int gs, int rows, int L, int N, cudaStream_t st) {
  const T* kk = static_cast<const T*>(k);
  const T* vv = static_cast<const T*>(v);
  if (gs % 2 == 0 && rows % 2 == 0 && c0 % 2 == 0) {
    const int pr = rows / 2;
    col_fwd<T, N1, false, true><<<dim3(M / COL_THREADS, pr), COL_THREADS, 0, st>>>(X, hi, lo, kk, vv, nullptr, row0,
                                                                                  0, L, 0, N);
    row_kernel<false><<<dim3(N1, pr), ROW_THREADS, ROW_SMEM, st>>>(X, Hf, hi, lo, N, c0 / 2, g0, gs / 2);
    col_inv<T, N1, true><<<dim3(M / COL_THREADS, pr), COL_THREADS, 0, st>>>(X, static_cast<const T*>(q),
                                                                            static_cast<T*>(y), row0, L, N);
    return;
  }
  if (gs == 1 && rows % 2 == 0) {  // per-channel filters: channel pairs with the mirror-bin product
    const int pr = rows / 2;
    col_fwd<T, N1, false, true><<<dim3(M / COL_THREADS, pr), COL_THREADS, 0, st>>>(X, hi, lo, kk, vv, nullptr, row0,
                                                                                  0, L, 0, N);
    row_pair_kernel<<<dim3(N1 / 2 + 1, pr), PAIR_THREADS, PAIR_SMEM, st>>>(X, Hf + static_cast<size_t>(c0 - g0) * N, hi,
                                                                          N, N1);
    col_inv<T, N1, true><<<dim3(M / COL_THREADS, pr), COL_THREADS, 0, st>>>(X, static_cast<const T*>(q),
                                                                            static_cast<T*>(y), row0, L, N);
    return;
  }
  col_fwd<T, N1, false><<<dim3(M / COL_THREADS, rows), COL_THREADS, 0, st>>>(X, hi, lo, kk, vv, nullptr, row0, 0, L, 0,
                                                                            N);
  row_kernel<false><<<dim3(N1, rows), ROW_THREADS, ROW_SMEM, st>>>(X, Hf, hi, lo, N, c0, g0, gs);
  col_inv<T, N1><<<dim3(M / COL_THREADS, rows), COL_THREADS, 0, st>>>(X, static_cast<const T*>(q), static_cast<T*>(y),
                                                                      row0, L, N);
}

template <typename T, int N1>
int run_n1(const void* q, const void* k, const void* v, void* y, const float* taps, int B, int C, int L, int lh,
           int gs, int N, int row_block, float2* hi, float2* lo, float2* Hf, float2* X, cudaStream_t st) {
  ensure_smem_attr(reinterpret_cast<const void*>(row_kernel<true>), ROW_SMEM);
  ensure_smem_attr(reinterpret_cast<const void*>(row_kernel<false>), ROW_SMEM);
  ensure_smem_attr(reinterpret_cast<const void*>(row_pair_kernel), PAIR_SMEM);
  const dim3 cgrid_x(M / COL_THREADS);
  for (int c0 = 0; c0 < C; c0 += row_block) {
    const int rows = C - c0 < row_block ? C - c0 : row_block;
    const int g0 = c0 / gs, g1 = (c0 + rows - 1) / gs, ng = g1 - g0 + 1;
    col_fwd<T, N1, true><<<dim3(M / COL_THREADS, ng), COL_THREADS, 0, st>>>(Hf, hi, lo, nullptr, nullptr, taps, 0,
                                                                           g0, L, lh, N);
    row_kernel<true><<<dim3(N1, ng), ROW_THREADS, ROW_SMEM, st>>>(Hf, nullptr, hi, lo, N, 0, 0, 1);
    for (int b = 0; b < B; ++b) {
      const int row0 = b * C + c0;
      act_pass<T, N1>(X, Hf, hi, lo, q, k, v, y, row0, c0, g0, gs, rows, L, N, st);
    }
  }
  (void)cgrid_x;
  return check_launch("fft_conv (register four-step)");
}

// Spectra of all G groups (cached by the caller) and the conv that reads them.
template <int N1>
int spectrum_n1(const float* taps, int G, int lh, int N, float2* hi, float2* lo, float2* spec, cudaStream_t st) {
  ensure_smem_attr(reinterpret_cast<const void*>(row_kernel<true>), ROW_SMEM);
  for (int g0 = 0; g0 < G; g0 += 32768) {  // grid.y limit
    const int ng = G - g0 < 32768 ? G - g0 : 32768;
    col_fwd<float, N1, true><<<dim3(M / COL_THREADS, ng), COL_THREADS, 0, st>>>(
        spec + static_cast<size_t>(g0) * N, hi, lo, nullptr, nullptr, taps, 0, g0, 0, lh, N);
    row_kernel<true><<<dim3(N1, ng), ROW_THREADS, ROW_SMEM, st>>>(spec + static_cast<size_t>(g0) * N, nullptr, hi,
                                                                  lo, N, 0, 0, 1);
  }
  return check_launch("fft spectrum");
}

template <typename T, int N1>
int conv_spec_n1(const void* q, const void* k, const void* v, void* y, const float2* spec, int B, int C, int L,
                 int gs, int N, int row_block, float2* hi, float2* lo, float2* X, cudaStream_t st) {
  ensure_smem_attr(reinterpret_cast<const void*>(row_kernel<false>), ROW_SMEM);
  ensure_smem_attr(reinterpret_cast<const void*>(row_pair_kernel), PAIR_SMEM);
  for (int c0 = 0; c0 < C; c0 += row_block) {
    const int rows = C - c0 < row_block ? C - c0 : row_block;
    const int g0 = c0 / gs;
    for (int b = 0; b < B; ++b) {
      const int row0 = b * C + c0;
      act_pass<T, N1>(X, spec + static_cast<size_t>(g0) * N, hi, lo, q, k, v, y, row0, c0, g0, gs, rows, L, N, st);
    }
  }
  return check_launch("fft_conv (cached spectrum)");
}

template <typename T>
int run(const void* q, const void* k, const void* v, void* y, const float* taps, int B, int C, int L, int lh,
        int gs, int N, int row_block, void* tw, void* hf, void* x, cudaStream_t st) {
  float2* hi = static_cast<float2*>(tw);
  float2* lo = hi + N / 64;
  table_kernel<<<(N / 64 + 64 + 255) / 256, 256, 0, st>>>(hi, lo, N);
  float2* Hf = static_cast<float2*>(hf);
  float2* X = static_cast<float2*>(x);
  switch (N / M) {
    case 2: return run_n1<T, 2>(q, k, v, y, taps, B, C, L, lh, gs, N, row_block, hi, lo, Hf, X, st);
    case 4: return run_n1<T, 4>(q, k, v, y, taps, B, C, L, lh, gs, N, row_block, hi, lo, Hf, X, st);
    case 8: return run_n1<T, 8>(q, k, v, y, taps, B, C, L, lh, gs, N, row_block, hi, lo, Hf, X, st);
    case 16: return run_n1<T, 16>(q, k, v, y, taps, B, C, L, lh, gs, N, row_block, hi, lo, Hf, X, st);
    case 32: return run_n1<T, 32>(q, k, v, y, taps, B, C, L, lh, gs, N, row_block, hi, lo, Hf, X, st);
    default: return fail(HY_ERR_UNSUPPORTED, "register FFT path: N = %d outside [2^14, 2^18]", N);
  }
}

}  // namespace fftf

bool fft_fast_supported(int N) { return N >= 2 * fftf::M && N <= 32 * fftf::M; }

int fft_fast_spectrum(const float* taps, int G, int lh, int N, void* spec, void* tw, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  float2* hi = static_cast<float2*>(tw);
  float2* lo = hi + N / 64;
  fftf::table_kernel<<<(N / 64 + 64 + 255) / 256, 256, 0, st>>>(hi, lo, N);
  float2* sp = static_cast<float2*>(spec);
  switch (N / fftf::M) {
    case 2: return fftf::spectrum_n1<2>(taps, G, lh, N, hi, lo, sp, st);
    case 4: return fftf::spectrum_n1<4>(taps, G, lh, N, hi, lo, sp, st);
    case 8: return fftf::spectrum_n1<8>(taps, G, lh, N, hi, lo, sp, st);
    case 16: return fftf::spectrum_n1<16>(taps, G, lh, N, hi, lo, sp, st);
    case 32: return fftf::spectrum_n1<32>(taps, G, lh, N, hi, lo, sp, st);
    default: return fail(HY_ERR_UNSUPPORTED, "cached FFT spectra need 2^14 <= N <= 2^18, got N = %d", N);
  }
}

template <typename T>
static int conv_spec(const void* q, const void* k, const void* v, void* y, const void* spec, int B, int C, int L,
                     int gs, int N, int row_block, void* tw, void* x, cudaStream_t st) {
  float2* hi = static_cast<float2*>(tw);
  float2* lo = hi + N / 64;
  fftf::table_kernel<<<(N / 64 + 64 + 255) / 256, 256, 0, st>>>(hi, lo, N);
  const float2* sp = static_cast<const float2*>(spec);
  float2* X = static_cast<float2*>(x);
  switch (N / fftf::M) {
    case 2: return fftf::conv_spec_n1<T, 2>(q, k, v, y, sp, B, C, L, gs, N, row_block, hi, lo, X, st);
    case 4: return fftf::conv_spec_n1<T, 4>(q, k, v, y, sp, B, C, L, gs, N, row_block, hi, lo, X, st);
    case 8: return fftf::conv_spec_n1<T, 8>(q, k, v, y, sp, B, C, L, gs, N, row_block, hi, lo, X, st);
    case 16: return fftf::conv_spec_n1<T, 16>(q, k, v, y, sp, B, C, L, gs, N, row_block, hi, lo, X, st);
    case 32: return fftf::conv_spec_n1<T, 32>(q, k, v, y, sp, B, C, L, gs, N, row_block, hi, lo, X, st);
    default: return fail(HY_ERR_UNSUPPORTED, "cached FFT spectra need 2^14 <= N <= 2^18, got N = %d", N);
  }
}

int fft_fast_conv_spec(const void* q, const void* k, const void* v, void* y, const void* spec, int B, int C, int L,
                       int gs, int dtype, int N, int row_block, void* tw, void* x, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == HY_F32) return conv_spec<float>(q, k, v, y, spec, B, C, L, gs, N, row_block, tw, x, st);
  return conv_spec<__nv_bfloat16>(q, k, v, y, spec, B, C, L, gs, N, row_block, tw, x, st);
}

int fft_fast_run(const void* q, const void* k, const void* v, void* y, const float* taps, int B, int C, int L,
                 int lh, int gs, int dtype, int N, int row_block, void* tw, void* hf, void* x, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == HY_F32) return fftf::run<float>(q, k, v, y, taps, B, C, L, lh, gs, N, row_block, tw, hf, x, st);
  return fftf::run<__nv_bfloat16>(q, k, v, y, taps, B, C, L, lh, gs, N, row_block, tw, hf, x, st);
}

}  // namespace hy
