// Hyena-LI filter-parameter gradients without materialising the length-L tap gradient.
//
// The reference forms dtaps[t] = sum_s dc[s] u[s-t] for every lag t < L (core.py:255-268) and
// pulls it back to the implicit filter h_t = sum_n R_n lam_n^t (hyena.py:193-211):
//   d_res[n]  = sum_t lam_n^t dtaps[t]              = sum_s dc[s] S_n[s]
//   d_pole[n] = R_n sum_t t lam_n^(t-1) dtaps[t]    = R_n sum_s dc[s] P_n[s]
// with the per-mode states S_n[s] = lam_n S_n[s-1] + u[s] and P_n = dS_n/dlam_n,
// P_n[s] = lam_n P_n[s-1] + S_n[s-1] (S, P zero before t = 0). Exact, O(L * modes).
//
#include "common.cuh"
#include "sm100.cuh"

namespace hy {

constexpr int kLiModes = 8;
constexpr int kLiRows = 16;                        // rows per CTA
constexpr int kLiThreads = kLiRows * kLiModes / 2;  // 4 threads per row, 2 modes each (64)

__device__ __forceinline__ float2 lg_ffma2(float2 a, float2 b, float2 c) {
  unsigned long long x, y, z, r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(z) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(y), "l"(z));
  float2 o;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
  return o;
}

template <typename T>
__device__ __forceinline__ float2 lg_pair(const T* p) {  // steps (s, s+1)
  if constexpr (sizeof(T) == 4) {
    return *reinterpret_cast<const float2*>(p);
  } else {
    const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(p);
    return __bfloat1622float2(v);
  }
}

// li_param_grad_kernel: one CTA per 16 (batch, channel) rows; thread (row, pair p) scans the
// whole row in time order for modes 2p, 2p+1 with packed fp32 FMAs (no chunk summaries, no
// combine): S = lam S + u, P = lam P + S_prev, a0 += dc S, a1 += dc P. The rows stream through
// a 2-deep shared ring of TS-step tiles filled by 1-D bulk copies (one per row and operand,
// issued by thread 0; rows padded by 16 B so the 4 rows of a warp hit distinct banks). Tile
// sums of a0 / a1 are added into fp64 accumulators.
template <typename T>
__global__ void __launch_bounds__(kLiThreads)
li_param_grad_kernel(const T* __restrict__ dc, const T* __restrict__ u, const float* __restrict__ poles,
                     int npoles, int rows, int C, int L, int gs, double* __restrict__ part) {
  using namespace sm100;
  constexpr int TS = sizeof(T) == 2 ? 256 : 128;           // steps per tile (34 KB ring)
  constexpr int RB = TS * static_cast<int>(sizeof(T)) + 16;  // padded row bytes
  __shared__ __align__(128) unsigned char ring[2][2][kLiRows * RB];  // [stage][dc, u][row]
  __shared__ uint64_t bars[2];
  const int r0 = blockIdx.x * kLiRows;
  const int nr = min(kLiRows, rows - r0);
  const int lr = threadIdx.x >> 2, pr = threadIdx.x & 3;
  const int row = r0 + lr;
  const int c = row % C;
  float2 lam = make_float2(0.f, 0.f);
  if (lr < nr) {
    const float* pp = poles + static_cast<size_t>(c / gs) * npoles;
    lam.x = 2 * pr < npoles ? pp[2 * pr] : 0.f;
    lam.y = 2 * pr + 1 < npoles ? pp[2 * pr + 1] : 0.f;
  }
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int ntile = (L + TS - 1) / TS;
  auto issue = [&](int tile) {  // thread 0
    const int st = tile & 1;
    const int t0 = tile * TS, cnt = min(TS, L - t0);
    const uint32_t bytes = static_cast<uint32_t>(cnt * sizeof(T));
    fence_proxy_async();
    mbar_arrive_expect_tx(&bars[st], 2 * nr * bytes);
    for (int i = 0; i < nr; ++i) {
      const size_t off = static_cast<size_t>(r0 + i) * L + t0;
      bulk_g2s(ring[st][0] + i * RB, dc + off, bytes, &bars[st]);
      bulk_g2s(ring[st][1] + i * RB, u + off, bytes, &bars[st]);
    }
  };
  if (threadIdx.x == 0) {
    issue(0);
    if (ntile > 1) issue(1);
  }
  float2 S = make_float2(0.f, 0.f), P = S;
  double A0x = 0.0, A0y = 0.0, A1x = 0.0, A1y = 0.0;
  for (int tile = 0; tile < ntile; ++tile) {
    const int st = tile & 1;
    mbar_wait(&bars[st], (tile >> 1) & 1);
    const int cnt = min(TS, L - tile * TS);  // even (L % 8 == 0)
    const T* dr = reinterpret_cast<const T*>(ring[st][0] + lr * RB);
    const T* ur = reinterpret_cast<const T*>(ring[st][1] + lr * RB);
    float2 a0 = make_float2(0.f, 0.f), a1 = a0;
    if (lr < nr) {
#pragma unroll 4
      for (int s = 0; s < cnt; s += 2) {
        const float2 d = lg_pair<T>(dr + s), x = lg_pair<T>(ur + s);
        float2 Sn = lg_ffma2(lam, S, make_float2(x.x, x.x));   // S[s]
        P = lg_ffma2(lam, P, S);                                // P[s] = lam P[s-1] + S[s-1]
        a0 = lg_ffma2(make_float2(d.x, d.x), Sn, a0);
        a1 = lg_ffma2(make_float2(d.x, d.x), P, a1);
        S = lg_ffma2(lam, Sn, make_float2(x.y, x.y));           // S[s+1]
        P = lg_ffma2(lam, P, Sn);
        a0 = lg_ffma2(make_float2(d.y, d.y), S, a0);
        a1 = lg_ffma2(make_float2(d.y, d.y), P, a1);
      }
    }
    A0x += a0.x, A0y += a0.y, A1x += a1.x, A1y += a1.y;
    __syncthreads();  // every thread is done with this stage
    if (threadIdx.x == 0 && tile + 2 < ntile) issue(tile + 2);
  }
  if (lr < nr) {
    double* pp = part + static_cast<size_t>(row) * kLiModes * 2;
    pp[(2 * pr) * 2 + 0] = A0x;
    pp[(2 * pr) * 2 + 1] = A1x;
    pp[(2 * pr + 1) * 2 + 0] = A0y;
    pp[(2 * pr + 1) * 2 + 1] = A1y;
  }
}

// d_res[g][n] = sum_{b, c in g} A0; d_pole[g][n] = R_n sum_{b, c in g} A1.
__global__ void li_param_reduce_kernel(const double* __restrict__ part, const float* __restrict__ residues,
                                       float* __restrict__ d_res, float* __restrict__ d_pole, int npoles, int B,
                                       int C, int gs) {
  const int g = blockIdx.x, m = threadIdx.x;
  if (m >= npoles) return;
  double s0 = 0.0, s1 = 0.0;
  for (int b = 0; b < B; ++b)
    for (int c = g * gs; c < (g + 1) * gs; ++c) {
      const double* p = part + ((static_cast<size_t>(b) * C + c) * kLiModes + m) * 2;
      s0 += p[0];
      s1 += p[1];
    }
  d_res[static_cast<size_t>(g) * npoles + m] = static_cast<float>(s0);
  d_pole[static_cast<size_t>(g) * npoles + m] =
      static_cast<float>(s1 * static_cast<double>(residues[static_cast<size_t>(g) * npoles + m]));
}

}  // namespace hy

using namespace hy;

extern "C" {

size_t hy_li_param_grad_workspace_size(int B, int C) {
  if (B < 1 || C < 1) return 0;
  return static_cast<size_t>(B) * C * kLiModes * 2 * sizeof(double);
}

int hy_li_param_grad(const void* dc, const void* u, const float* residues, const float* poles, int npoles, int gs,
                     int B, int C, int L, int dtype, float* d_res, float* d_pole, void* ws, size_t ws_bytes,
                     void* stream) {
  if (!dc || !u || !residues || !poles || !d_res || !d_pole || !ws)
    return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || gs < 1 || npoles < 1)
    return fail(HY_ERR_INVALID, "sizes must be >= 1 (B=%d C=%d L=%d gs=%d npoles=%d)", B, C, L, gs, npoles);
  if (npoles > kLiModes) return fail(HY_ERR_UNSUPPORTED, "li_param_grad: %d poles > %d", npoles, kLiModes);
  if (C % gs != 0) return fail(HY_ERR_INVALID, "group_size %d does not divide channel count %d", gs, C);
  if (static_cast<long long>(B) * C > 0x7fffffffLL) return fail(HY_ERR_UNSUPPORTED, "too many rows");
  if (ws_bytes < hy_li_param_grad_workspace_size(B, C)) return fail(HY_ERR_INVALID, "workspace too small");
  if (L % 8 != 0 || !aligned16(dc) || !aligned16(u))
    return fail(HY_ERR_UNSUPPORTED, "li_param_grad needs L %% 8 == 0 and 16-byte aligned rows");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* part = static_cast<double*>(ws);
  const int rows = B * C;
  const int grid = (rows + kLiRows - 1) / kLiRows;
  if (dtype == HY_F32) {
    li_param_grad_kernel<float><<<grid, kLiThreads, 0, st>>>(static_cast<const float*>(dc),
                                                              static_cast<const float*>(u), poles, npoles, rows, C, L,
                                                              gs, part);
  } else if (dtype == HY_BF16) {
    li_param_grad_kernel<__nv_bfloat16><<<grid, kLiThreads, 0, st>>>(static_cast<const __nv_bfloat16*>(dc),
                                                                      static_cast<const __nv_bfloat16*>(u), poles,
                                                                      npoles, rows, C, L, gs, part);
  } else {
    return fail(HY_ERR_UNSUPPORTED, "li_param_grad: fp32 / bf16 only");
  }
  int s = check_launch("li_param_grad_kernel");
  if (s != HY_OK) return s;
  li_param_reduce_kernel<<<C / gs, kLiModes, 0, st>>>(part, residues, d_res, d_pole, npoles, B, C, gs);
  return check_launch("li_param_reduce_kernel");
}

}  // extern "C"
