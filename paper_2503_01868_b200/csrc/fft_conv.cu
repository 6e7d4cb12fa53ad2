// FFT causal convolution fused with the Hyena gates (fft.py:128-145, hyena.py:183-186):
//
//     y[t] = q[t] * (h conv (k * v))[t],  t < L,  h = the row's group taps (lh <= L)
//
// computed as x = IFFT(FFT(pad(k * v)) . FFT(pad(h))) / N over N = next_pow2(L + lh - 1)
// points, the zero-padded circular convolution the reference uses, in fp32 complex
// arithmetic on the CUDA cores (fp32 / bf16 activations; fp64 stays on the exact FIR path).
//
// Four-step decomposition N = N1 * N2 (N2 = min(N, 4096), N1 <= 512), n = N2 n1 + n2,
// k = k1 + N1 k2, every pass one kernel with its transform in shared memory:
//
//   A  (columns)  for each n2: DIF over n1 of the prepped input (k*v or the taps, zero
//                 padded) -> bin k1 at position p = bitrev(k1); times W_N^(n2 k1)
//   R  (rows)     for each p: DIF over n2 -> bin k2 at position bitrev(k2); for the taps
//                 store the spectrum, for data multiply by it and run the inverse DIT back
//                 to natural n2; times W_N^(-n2 k1)
//   A' (columns)  for each n2: inverse DIT over the bit-reversed p -> natural n1; 1/N, the
//                 gate q and the output dtype in the epilogue
//
// The spectrum stays in the transform's own (bit-reversed) order end to end: no
// permutation pass. Twiddles come from one table W_N^j = exp(-2 pi i j / N) computed in
// double precision. Workspace: the table, the spectra of one channel block's groups and
// the transforms of one block of rows (hy_fft_conv_workspace_size).
#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace hy {
namespace fft {

constexpr int MAX_N2 = 4096;   // row transform length (shared memory: 32 KB data + 16 KB twiddles)
constexpr int MAX_N1 = 512;    // column transform length
constexpr int COL_POINTS = 8192;  // points per column-pass CTA: N1 x CC columns (64 KB)
constexpr int ROW_BLOCK = 256; // channels per block (spectra + transforms held in the workspace)
// channels per launch of the fast path (HY_FFT_ROW_BLOCK overrides; probe)
inline int fast_row_block() {
  const char* e = getenv("HY_FFT_ROW_BLOCK");
  const int v = e ? atoi(e) : 0;
  return v > 0 && v <= ROW_BLOCK ? v : ROW_BLOCK;
}
constexpr int THREADS = 256;

struct Plan {
  int N, N1, N2, log1, log2;
};

inline int ilog2(long long n) {
  int l = 0;
  while ((1LL << l) < n) ++l;
  return l;
}

inline Plan make_plan(int L, int lh) {
  Plan p{};
  const long long need = static_cast<long long>(L) + lh - 1;
  int lg = ilog2(need < 1 ? 1 : need);
  if (lg < 4) lg = 4;  // >= 16 points (extra zero padding leaves the causal result unchanged)
  p.N = 1 << lg;
  p.log2 = lg < 12 ? lg : 12;
  p.N2 = 1 << p.log2;
  p.log1 = lg - p.log2;
  p.N1 = 1 << p.log1;
  return p;
}

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // a * conj(b)
  return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ int bitrev(int x, int bits) { return bits ? (__brev(x) >> (32 - bits)) : 0; }

__global__ void twiddle_kernel(float2* tw, int N) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < N) {
    double s, c;
    sincospi(-2.0 * static_cast<double>(j) / static_cast<double>(N), &s, &c);
    tw[j] = make_float2(static_cast<float>(c), static_cast<float>(s));
  }
}

// In-shared-memory transforms of CNT interleaved sequences of length M = 2^lg: element i
// of sequence s at x[i * CNT + s] (CNT = 1: one contiguous sequence). Twiddles per level:
// wl[2^(e-2) + j] = W_(2^e)^j for j < 2^(e-2) (contiguous per stage: conflict-free reads).
// DIF: natural in, bit-reversed out. DIT (inverse, conjugate twiddles): bit-reversed in,
// natural out, unnormalised. Radix-2 stages are fused in pairs (radix 2^2): a thread holds
// the 4 points i0 + {0, q, 2q, 3q} of a 4q-block in registers across both stages, halving
// the shared-memory passes and barriers; an odd leftover stage runs as plain radix 2.
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 mul_negi(float2 a) { return make_float2(a.y, -a.x); }  // a * (-i)
__device__ __forceinline__ float2 mul_posi(float2 a) { return make_float2(-a.y, a.x); }  // a * (+i)

template <int CNT>
__device__ void dif(float2* x, int lg, const float2* wl) {
  const int M = 1 << lg;
  int s = lg;
  for (; s >= 2; s -= 2) {  // stages s (len 4q) and s-1 (len 2q), q = 2^(s-2)
    const int q = 1 << (s - 2);
    for (int b = threadIdx.x; b < CNT * (M / 4); b += blockDim.x) {
      const int seq = b % CNT, r = b / CNT;
      const int j = r & (q - 1), i0 = ((r >> (s - 2)) << s) + j;
      float2* p = x + i0 * CNT + seq;
      const float2 w = wl[q + j], w2 = cmul(w, w);  // W_4q^j, W_2q^j
      const float2 a0 = p[0], a1 = p[q * CNT], a2 = p[2 * q * CNT], a3 = p[3 * q * CNT];
      const float2 b0 = cadd(a0, a2), b2 = cmul(csub(a0, a2), w);
      const float2 b1 = cadd(a1, a3), b3 = mul_negi(cmul(csub(a1, a3), w));
      p[0] = cadd(b0, b1);
      p[q * CNT] = cmul(csub(b0, b1), w2);
      p[2 * q * CNT] = cadd(b2, b3);
      p[3 * q * CNT] = cmul(csub(b2, b3), w2);
    }
    __syncthreads();
  }
  if (s == 1) {  // last radix-2 stage (len 2, twiddle 1)
    for (int b = threadIdx.x; b < CNT * (M / 2); b += blockDim.x) {
      const int seq = b % CNT, r = b / CNT;
      float2* p = x + 2 * r * CNT + seq;
      const float2 a = p[0], c = p[CNT];
      p[0] = cadd(a, c);
      p[CNT] = csub(a, c);
    }
    __syncthreads();
  }
}

template <int CNT>
__device__ void dit_inv(float2* x, int lg, const float2* wl) {
  const int M = 1 << lg;
  int s = 1;
  if (lg & 1) {  // first radix-2 stage (len 2)
    for (int b = threadIdx.x; b < CNT * (M / 2); b += blockDim.x) {
      const int seq = b % CNT, r = b / CNT;
      float2* p = x + 2 * r * CNT + seq;
      const float2 a = p[0], c = p[CNT];
      p[0] = cadd(a, c);
      p[CNT] = csub(a, c);
    }
    __syncthreads();
    s = 2;
  }
  for (; s + 1 <= lg; s += 2) {  // stages s (len 2q) and s+1 (len 4q), q = 2^(s-1)
    const int q = 1 << (s - 1);
    for (int b = threadIdx.x; b < CNT * (M / 4); b += blockDim.x) {
      const int seq = b % CNT, r = b / CNT;
      const int j = r & (q - 1), i0 = ((r >> (s - 1)) << (s + 1)) + j;
      float2* p = x + i0 * CNT + seq;
      const float2 w = wl[q + j], w2 = cmul(w, w);  // W_4q^j, W_2q^j
      const float2 a0 = p[0], a1 = p[q * CNT], a2 = p[2 * q * CNT], a3 = p[3 * q * CNT];
      float2 t = cmulc(a1, w2);
      const float2 b0 = cadd(a0, t), b1 = csub(a0, t);
      t = cmulc(a3, w2);
      const float2 b2 = cadd(a2, t), b3 = csub(a2, t);
      t = cmulc(b2, w);
      p[0] = cadd(b0, t);
      p[2 * q * CNT] = csub(b0, t);
      t = mul_posi(cmulc(b3, w));
      p[q * CNT] = cadd(b1, t);
      p[3 * q * CNT] = csub(b1, t);
    }
    __syncthreads();
  }
}

__device__ void load_local_twiddles(float2* wl, const float2* __restrict__ tw, int lg, int N) {
  const int M = 1 << lg;
  for (int idx = threadIdx.x + 1; idx < M / 2; idx += blockDim.x) {
    const int e2 = 31 - __clz(idx), j = idx - (1 << e2);  // level e = e2 + 2
    wl[idx] = tw[static_cast<size_t>(j) * static_cast<size_t>(N >> (e2 + 2))];
  }
}

template <typename T>
__device__ __forceinline__ float ldf(const T* p) { return Elem<T>::to_a(*p); }

// Pass A: columns [n2_0, n2_0 + COLS) of `rows` rows (blockIdx.y); input row r is
// taps (FILTER: group g0 + r, length lh) or k*v (row r of the block, length L).
template <typename T, bool FILTER, int COLS>
__global__ void __launch_bounds__(THREADS) col_fwd_kernel(float2* __restrict__ X, const float2* __restrict__ tw,
                                                          const T* __restrict__ k, const T* __restrict__ v,
                                                          const float* __restrict__ taps, int row0, int g0,
                                                          int L, int lh, Plan pl) {
  extern __shared__ float2 sm[];
  float2* xs = sm;               // [N1][COLS]
  float2* wl = sm + COL_POINTS;  // column-transform twiddles
  const int r = blockIdx.y, n2_0 = blockIdx.x * COLS;
  load_local_twiddles(wl, tw, pl.log1, pl.N);
  for (int e = threadIdx.x; e < pl.N1 * COLS; e += blockDim.x) {
    const int n1 = e / COLS, col = e % COLS;
    const long long t = static_cast<long long>(pl.N2) * n1 + n2_0 + col;
    float val = 0.f;
    if (FILTER) {
      if (t < lh) val = taps[static_cast<size_t>(g0 + r) * lh + t];
    } else if (t < L) {
      const size_t off = static_cast<size_t>(row0 + r) * L + t;
      val = ldf(v + off);
      if (k) val *= ldf(k + off);
    }
    xs[n1 * COLS + col] = make_float2(val, 0.f);
  }
  __syncthreads();
  dif<COLS>(xs, pl.log1, wl);
  float2* out = X + static_cast<size_t>(r) * pl.N;
  for (int e = threadIdx.x; e < pl.N1 * COLS; e += blockDim.x) {
    const int p = e / COLS, col = e % COLS, n2 = n2_0 + col;
    const int k1 = bitrev(p, pl.log1);
    const float2 w = tw[(static_cast<long long>(n2) * k1) & (pl.N - 1)];  // W_N^(n2 k1)
    out[static_cast<size_t>(p) * pl.N2 + n2] = cmul(xs[p * COLS + col], w);
  }
}

// Pass R: one row p (blockIdx.x) of block row r (blockIdx.y). FILTER: forward transform
// stored as the group spectrum. Else: forward, times the spectrum of the row's group,
// inverse, times W_N^(-n2 k1).
template <bool FILTER>
__global__ void __launch_bounds__(THREADS) row_kernel(float2* X, float2* Hf,
                                                      const float2* __restrict__ tw, int c0, int g0, int gs,
                                                      Plan pl) {
  extern __shared__ float2 sm[];
  float2* xs = sm;               // [N2]
  float2* wl = sm + MAX_N2;      // W_N2^j
  const int p = blockIdx.x, r = blockIdx.y;
  load_local_twiddles(wl, tw, pl.log2, pl.N);
  float2* row = X + static_cast<size_t>(r) * pl.N + static_cast<size_t>(p) * pl.N2;
  for (int i = threadIdx.x; i < pl.N2; i += blockDim.x) xs[i] = row[i];
  __syncthreads();
  dif<1>(xs, pl.log2, wl);
  if (FILTER) {
    float2* h = Hf + static_cast<size_t>(r) * pl.N + static_cast<size_t>(p) * pl.N2;
    for (int i = threadIdx.x; i < pl.N2; i += blockDim.x) h[i] = xs[i];
    return;
  }
  const int g = (c0 + r) / gs - g0;
  const float2* h = Hf + static_cast<size_t>(g) * pl.N + static_cast<size_t>(p) * pl.N2;
  for (int i = threadIdx.x; i < pl.N2; i += blockDim.x) xs[i] = cmul(xs[i], h[i]);
  __syncthreads();
  dit_inv<1>(xs, pl.log2, wl);
  const int k1 = bitrev(p, pl.log1);
  for (int n2 = threadIdx.x; n2 < pl.N2; n2 += blockDim.x)
    row[n2] = cmulc(xs[n2], tw[(static_cast<long long>(n2) * k1) & (pl.N - 1)]);
}

// Pass A': inverse column transforms, then y = q * Re(x) / N for t < L.
template <typename T, int COLS>
__global__ void __launch_bounds__(THREADS) col_inv_kernel(const float2* __restrict__ X,
                                                          const float2* __restrict__ tw,
                                                          const T* __restrict__ q, T* __restrict__ y, int row0,
                                                          int L, Plan pl) {
  extern __shared__ float2 sm[];
  float2* xs = sm;
  float2* wl = sm + COL_POINTS;
  const int r = blockIdx.y, n2_0 = blockIdx.x * COLS;
  load_local_twiddles(wl, tw, pl.log1, pl.N);
  const float2* in = X + static_cast<size_t>(r) * pl.N;
  for (int e = threadIdx.x; e < pl.N1 * COLS; e += blockDim.x) {
    const int p = e / COLS, col = e % COLS;
    xs[p * COLS + col] = in[static_cast<size_t>(p) * pl.N2 + n2_0 + col];
  }
  __syncthreads();
  dit_inv<COLS>(xs, pl.log1, wl);
  const float scale = 1.f / static_cast<float>(pl.N);
  for (int e = threadIdx.x; e < pl.N1 * COLS; e += blockDim.x) {
    const int n1 = e / COLS, col = e % COLS;
    const long long t = static_cast<long long>(pl.N2) * n1 + n2_0 + col;
    if (t < L) {
      const size_t off = static_cast<size_t>(row0 + r) * L + t;
      float val = xs[n1 * COLS + col].x * scale;
      if (q) val *= ldf(q + off);
      y[off] = Elem<T>::from_a(val);
    }
  }
}

constexpr size_t align256(size_t b) { return (b + 255) / 256 * 256; }

struct Layout {
  size_t tw, hf, x, total;
};

inline Layout ws_layout(const Plan& pl, int C, int gs) {
  Layout l{};
  const size_t n = static_cast<size_t>(pl.N) * sizeof(float2);
  const int rows = C < ROW_BLOCK ? C : ROW_BLOCK;
  const int groups = rows / gs + 2;  // a channel block spans at most rows/gs + 2 groups
  l.tw = 0;
  l.hf = align256(n);
  l.x = l.hf + align256(static_cast<size_t>(groups) * n);
  l.total = l.x + align256(static_cast<size_t>(rows) * n);
  return l;
}

template <typename T, int COLS>
int run_cols(const void* q, const void* k, const void* v, void* y, const float* taps, int B, int C, int L, int lh,
             int gs, const Plan& pl, float2* tw, float2* Hf, float2* X, cudaStream_t st) {
  const size_t col_smem = (COL_POINTS + MAX_N1 / 2) * sizeof(float2);
  const size_t row_smem = (MAX_N2 + MAX_N2 / 2) * sizeof(float2);
  ensure_smem_attr(reinterpret_cast<const void*>(col_fwd_kernel<T, true, COLS>), (int)col_smem);
  ensure_smem_attr(reinterpret_cast<const void*>(col_fwd_kernel<T, false, COLS>), (int)col_smem);
  ensure_smem_attr(reinterpret_cast<const void*>(col_inv_kernel<T, COLS>), (int)col_smem);
  ensure_smem_attr(reinterpret_cast<const void*>(row_kernel<true>), (int)row_smem);
  ensure_smem_attr(reinterpret_cast<const void*>(row_kernel<false>), (int)row_smem);
  const int ncol = pl.N2 / COLS;
  for (int c0 = 0; c0 < C; c0 += ROW_BLOCK) {
    const int rows = C - c0 < ROW_BLOCK ? C - c0 : ROW_BLOCK;
    const int g0 = c0 / gs, g1 = (c0 + rows - 1) / gs, ng = g1 - g0 + 1;
    // spectra of this block's groups
    col_fwd_kernel<T, true, COLS><<<dim3(ncol, ng), THREADS, col_smem, st>>>(Hf, tw, nullptr, nullptr, taps, 0, g0,
                                                                            L, lh, pl);
    row_kernel<true><<<dim3(pl.N1, ng), THREADS, row_smem, st>>>(Hf, Hf, tw, 0, g0, gs, pl);
    for (int b = 0; b < B; ++b) {
      const int row0 = b * C + c0;
      col_fwd_kernel<T, false, COLS><<<dim3(ncol, rows), THREADS, col_smem, st>>>(
          X, tw, static_cast<const T*>(k), static_cast<const T*>(v), nullptr, row0, 0, L, lh, pl);
      row_kernel<false><<<dim3(pl.N1, rows), THREADS, row_smem, st>>>(X, Hf, tw, c0, g0, gs, pl);
      col_inv_kernel<T, COLS><<<dim3(ncol, rows), THREADS, col_smem, st>>>(X, tw, static_cast<const T*>(q),
                                                                           static_cast<T*>(y), row0, L, pl);
    }
  }
  return check_launch("fft_conv");
}

template <typename T>
int run(const void* q, const void* k, const void* v, void* y, const float* taps, int B, int C, int L, int lh,
        int gs, void* ws, cudaStream_t st) {
  const Plan pl = make_plan(L, lh);
  const Layout ly = ws_layout(pl, C, gs);
  unsigned char* base = static_cast<unsigned char*>(ws);
  float2* tw = reinterpret_cast<float2*>(base + ly.tw);
  float2* Hf = reinterpret_cast<float2*>(base + ly.hf);
  float2* X = reinterpret_cast<float2*>(base + ly.x);
  if (fft_fast_supported(pl.N) && !getenv("HY_FFT_RADIX4")) {
    const int dt = sizeof(T) == 4 ? HY_F32 : HY_BF16;
    return fft_fast_run(q, k, v, y, taps, B, C, L, lh, gs, dt, pl.N, fast_row_block(), tw, Hf, X, st);
  }
  twiddle_kernel<<<(pl.N + 255) / 256, 256, 0, st>>>(tw, pl.N);
  // widest column block that fits: N1 x COLS <= 8192 points, COLS <= N2
  if (pl.N1 <= 128 && pl.N2 >= 64) return run_cols<T, 64>(q, k, v, y, taps, B, C, L, lh, gs, pl, tw, Hf, X, st);
  if (pl.N1 <= 256 && pl.N2 >= 32) return run_cols<T, 32>(q, k, v, y, taps, B, C, L, lh, gs, pl, tw, Hf, X, st);
  return run_cols<T, 16>(q, k, v, y, taps, B, C, L, lh, gs, pl, tw, Hf, X, st);
}

}  // namespace fft
}  // namespace hy

using namespace hy;

extern "C" HY_API size_t hy_fft_conv_workspace_size(int B, int C, int L, int lh, int gs, int dtype) {
  (void)B;
  if (C < 1 || L < 1 || lh < 1 || gs < 1 || C % gs != 0 || lh > L) return 0;
  if (dtype != HY_F32 && dtype != HY_BF16) return 0;
  const fft::Plan pl = fft::make_plan(L, lh);
  if (pl.N1 > fft::MAX_N1) return 0;
  return fft::ws_layout(pl, C, gs).total;
}

extern "C" HY_API int hy_fft_conv_fwd(const void* q, const void* k, const void* v, void* y, const void* taps, int B,
                                      int C, int L, int lh, int gs, int dtype, void* ws, size_t ws_bytes,
                                      void* stream) {
  if (!v || !y || !taps) return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || lh < 1 || gs < 1)
    return fail(HY_ERR_INVALID, "sizes must be >= 1 (B=%d C=%d L=%d lh=%d gs=%d)", B, C, L, lh, gs);
  if (C % gs != 0) return fail(HY_ERR_INVALID, "group_size %d does not divide channel count %d", gs, C);
  if (lh > L) return fail(HY_ERR_INVALID, "filter length %d exceeds the sequence length %d", lh, L);
  if (dtype != HY_F32 && dtype != HY_BF16)
    return fail(HY_ERR_UNSUPPORTED, "hy_fft_conv_fwd: fp32 / bf16 activations (fp64 uses the exact FIR path)");
  const fft::Plan pl = fft::make_plan(L, lh);
  if (pl.N1 > fft::MAX_N1) return fail(HY_ERR_UNSUPPORTED, "FFT length %d beyond 2^21", pl.N);
  const size_t need = fft::ws_layout(pl, C, gs).total;
  if (!ws || ws_bytes < need) return fail(HY_ERR_INVALID, "workspace %zu bytes, need %zu", ws_bytes, need);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float* h = static_cast<const float*>(taps);
  if (dtype == HY_F32) return fft::run<float>(q, k, v, y, h, B, C, L, lh, gs, ws, st);
  return fft::run<__nv_bfloat16>(q, k, v, y, h, B, C, L, lh, gs, ws, st);
}

// ---------------------------------------------------------------- cached filter spectra
// (register four-step path: 2^14 <= N <= 2^18). The spectrum of each group's zero-padded taps
// is a parameter transform: computed once per filter bank, read by every later call.

extern "C" HY_API size_t hy_fft_spectrum_size(int G, int L, int lh) {
  if (G < 1 || L < 1 || lh < 1 || lh > L) return 0;
  const fft::Plan pl = fft::make_plan(L, lh);
  if (!fft_fast_supported(pl.N)) return 0;
  return static_cast<size_t>(G) * pl.N * 8;
}

extern "C" HY_API int hy_fft_spectrum(const void* taps, int G, int L, int lh, void* spec, void* ws, size_t ws_bytes,
                                      void* stream) {
  if (!taps || !spec) return fail(HY_ERR_INVALID, "null pointer argument");
  if (G < 1 || L < 1 || lh < 1) return fail(HY_ERR_INVALID, "sizes must be >= 1 (G=%d L=%d lh=%d)", G, L, lh);
  if (lh > L) return fail(HY_ERR_INVALID, "filter length %d exceeds the sequence length %d", lh, L);
  const fft::Plan pl = fft::make_plan(L, lh);
  if (!fft_fast_supported(pl.N))
    return fail(HY_ERR_UNSUPPORTED, "cached FFT spectra need 2^14 <= N <= 2^18, got N = %d", pl.N);
  const size_t need = static_cast<size_t>(pl.N / 64 + 64) * 8;
  if (!ws || ws_bytes < need) return fail(HY_ERR_INVALID, "workspace %zu bytes, need %zu", ws_bytes, need);
  return fft_fast_spectrum(static_cast<const float*>(taps), G, lh, pl.N, spec, ws, stream);
}

extern "C" HY_API int hy_fft_conv_spec_fwd(const void* q, const void* k, const void* v, void* y, const void* spec,
                                           int B, int C, int L, int lh, int gs, int dtype, void* ws,
                                           size_t ws_bytes, void* stream) {
  if (!v || !y || !spec) return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || lh < 1 || gs < 1)
    return fail(HY_ERR_INVALID, "sizes must be >= 1 (B=%d C=%d L=%d lh=%d gs=%d)", B, C, L, lh, gs);
  if (C % gs != 0) return fail(HY_ERR_INVALID, "group_size %d does not divide channel count %d", gs, C);
  if (lh > L) return fail(HY_ERR_INVALID, "filter length %d exceeds the sequence length %d", lh, L);
  if (dtype != HY_F32 && dtype != HY_BF16)
    return fail(HY_ERR_UNSUPPORTED, "hy_fft_conv_spec_fwd: fp32 / bf16 activations");
  const fft::Plan pl = fft::make_plan(L, lh);
  if (!fft_fast_supported(pl.N))
    return fail(HY_ERR_UNSUPPORTED, "cached FFT spectra need 2^14 <= N <= 2^18, got N = %d", pl.N);
  const fft::Layout ly = fft::ws_layout(pl, C, gs);
  if (!ws || ws_bytes < ly.total) return fail(HY_ERR_INVALID, "workspace %zu bytes, need %zu", ws_bytes, ly.total);
  unsigned char* base = static_cast<unsigned char*>(ws);
  return fft_fast_conv_spec(q, k, v, y, spec, B, C, L, gs, dtype, pl.N, fft::fast_row_block(), base + ly.tw, base + ly.x,
                            stream);
}
