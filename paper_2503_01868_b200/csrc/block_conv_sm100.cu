// K-block causal convolution on 5th-gen tensor cores (sm_100a): filters longer than one spill
// factor, 129 < lh <= 513.
//
// Restates blockconv.py:103-121 (block_conv: Y_n = sum_{k=0..K} B_k U_{n-k}, K = ceil((lh-1)/lb))
// at the kernel's own block length LB = 128 (any block size gives the same causal sum), bf16 in /
// fp32 accumulate, with the optional gates of two_stage_forward (y = q * conv(k * v)) and the
// regularisation decay applied in-kernel (core.py:144-146):
//
//     D[t_out][chunk] = sum_{k=0..K} T_k[t_out][:] . U_{chunk-k}[:]        (K + 1) x 8 MMAs per tile
//     T_k[m][j] = h[128 k + m - j]   (Toeplitz factors, A operand in TMEM, built in-kernel)
//
// Tile = NCH = 32 consecutive 128-step chunks of one sequence. The shifted operands U_{n-k} are
// NOT copies: the U buffer holds the tile's chunks plus the K chunks before them as rows of one
// SW128 K-major matrix (row r = chunk r - HROWS), and the MMA for factor k reads it through a
// descriptor starting k rows earlier (a 128-byte row offset inside the swizzle atom).
//
// Warp roles (576 threads, 1 CTA per SM, persistent over a contiguous tile range):
//   warps 0-7   converter: staged raw v (and k) window -> u = k * v -> bf16 swizzled U rows
//   warps 8-11  epilogue : TMEM acc -> y = q * acc (q read from HBM) -> coalesced stores
//   warps 12-15 factor builder: T_0..T_K of each filter group into TMEM once the last MMA of the
//                          previous group retired (the next group's taps are prefetched)
//   warp 16     MMA      : TMEM alloc (512 cols); one lane issues the (K+1) x 8 MMAs of each tile
//   warp 17     producer : 1-D bulk copies (cp.async.bulk) of the v / k windows into a 4-stage ring
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace hy {
namespace kb {

using bf16 = __nv_bfloat16;
using namespace sm100;

constexpr int LB = 128;
constexpr int NCH = 32;
constexpr int TILE_T = NCH * LB;
constexpr int KMAX = 4;                  // spill factors: lh <= KMAX * LB + 1
constexpr int HROWS = 8;                 // U rows before the tile's first chunk (>= KMAX)
constexpr int UROWS = NCH + HROWS;       // 40 rows: 5 groups of 8
constexpr int WIN = TILE_T + KMAX * LB;  // staged window per tensor: the tile + KMAX chunks before
constexpr int STAGES = 4;
constexpr int NBUF = 3;
constexpr int N_CONV_WARPS = 8, N_EPI_WARPS = 4, N_TB_WARPS = 4;
constexpr int W_CONV0 = 0, W_EPI0 = 8, W_TB0 = 12, W_MMA = 16, W_PROD = 17, THREADS = 18 * 32;
constexpr int CONV_THREADS = N_CONV_WARPS * 32, TB_THREADS = N_TB_WARPS * 32;
constexpr uint32_t BAR_CONV = 1, BAR_TB = 2;
constexpr uint32_t TM_ACC = 0, TM_F = 128;  // accumulators [NBUF] x 32; factor k at TM_F + 64 k
static_assert(NBUF * NCH <= static_cast<int>(TM_F) && TM_F + 64 * (KMAX + 1) <= 512, "TMEM budget");
static_assert(HROWS >= KMAX && UROWS % 8 == 0, "U rows");

constexpr int round_up(int a, int m) { return (a + m - 1) / m * m; }
constexpr int WIN_BYTES = WIN * 2;
constexpr int STAGE_BYTES = 2 * WIN_BYTES;           // v, k windows
constexpr int U_ATOM = UROWS * 128;                  // one 64-element K atom of the U matrix
constexpr int U_BYTES = 2 * U_ATOM;
constexpr int OFF_ST = 0;
constexpr int OFF_U = round_up(STAGES * STAGE_BYTES, 1024);
constexpr int HP_N = 1024;                           // hpad[i + 128] = h[i], i in [-128, 896)
constexpr int OFF_HP = OFF_U + NBUF * U_BYTES;       // two buffers (current / next group)
constexpr int OFF_BAR = OFF_HP + 2 * HP_N * 2;
constexpr int N_BARS = 2 * STAGES + 4 * NBUF + 2;
constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
constexpr int SMEM_BYTES = OFF_TMEM + 16 + 1024;
static_assert(SMEM_BYTES <= 232448, "shared memory budget");

struct Params {
  const bf16* q;
  const bf16* k;
  const bf16* v;
  bf16* y;
  const float* taps_hat;  // (n_groups, lh)
  const float* decay;     // (n_groups) rate * log2(base), or null
  int B, C, L, lh, K, gs;
  int tiles_per_seq, total_tiles;
  int base_off;           // 1: set the descriptor base-offset field for row-shifted starts
};

struct Tile {
  int c, b, j, t0;
  __device__ __forceinline__ void init(int tile, const Params& p) {
    j = tile % p.tiles_per_seq;
    const int r = tile / p.tiles_per_seq;
    b = r % p.B;
    c = r / p.B;
    t0 = j * TILE_T;
  }
  __device__ __forceinline__ void next(const Params& p) {
    if (++j == p.tiles_per_seq) {
      j = 0;
      if (++b == p.B) {
        b = 0;
        ++c;
      }
    }
    t0 = j * TILE_T;
  }
  __device__ __forceinline__ bool last_of_channel(const Params& p) const {
    return j == p.tiles_per_seq - 1 && b == p.B - 1;
  }
};

__device__ __forceinline__ uint32_t sw_off(int row, int j) {  // 16-byte unit j (0..15) of U row `row`
  return (j >> 3) * U_ATOM + row * 128 + (((j & 7) ^ (row & 7)) << 4);
}

template <bool GK, bool GQ>
__global__ void __launch_bounds__(THREADS, 1) block_conv_kernel(const Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* ufull = bars + 2 * STAGES;
  uint64_t* uempty = ufull + NBUF;
  uint64_t* tfull = uempty + NBUF;
  uint64_t* tempty = tfull + NBUF;
  uint64_t* tready = tempty + NBUF;  // builder -> MMA: the group's factors are in TMEM
  uint64_t* tfree = tready + 1;      // MMA commit: the last MMA reading the factors retired
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tb = static_cast<int>((static_cast<long long>(blockIdx.x) * p.total_tiles) / gridDim.x);
  const int te = static_cast<int>((static_cast<long long>(blockIdx.x + 1) * p.total_tiles) / gridDim.x);
  const int ntiles = te - tb;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&ufull[i], 1);
      mbar_init(&uempty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], N_EPI_WARPS);
    }
    mbar_init(tready, 1);
    mbar_init(tfree, 1);
    fence_mbar_init();
  }
  if (warp == W_MMA) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == W_PROD) {
    // ------------------------------------------------------------ producer
    Tile t;
    t.init(tb, p);
    for (int it = 0; it < ntiles; ++it, t.next(p)) {
      const int s = it % STAGES;
      mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
      unsigned char* st = smem + OFF_ST + s * STAGE_BYTES;
      bf16* vbuf = reinterpret_cast<bf16*>(st);
      bf16* kbuf = reinterpret_cast<bf16*>(st + WIN_BYTES);
      const int ws = t.t0 - KMAX * LB, we = t.t0 + TILE_T;
      const int vs = max(ws, 0), ve = min(we, p.L);
      if (vs != ws || ve != we) {  // zero the window outside [0, L) (whole 16-byte units)
        const int4 z = make_int4(0, 0, 0, 0);
        for (int i = lane * 8; i < vs - ws; i += 256) {
          *reinterpret_cast<int4*>(vbuf + i) = z;
          if (GK) *reinterpret_cast<int4*>(kbuf + i) = z;
        }
        for (int i = (ve - ws) + lane * 8; i < WIN; i += 256) {
          *reinterpret_cast<int4*>(vbuf + i) = z;
          if (GK) *reinterpret_cast<int4*>(kbuf + i) = z;
        }
        fence_proxy_async();
      }
      __syncwarp();
      if (elect_one()) {
        const uint32_t bytes = static_cast<uint32_t>(ve - vs) * 2;
        const size_t row = static_cast<size_t>(t.b * p.C + t.c) * p.L;
        mbar_arrive_expect_tx(&full[s], bytes * (GK ? 2 : 1));
        bulk_g2s(vbuf + (vs - ws), p.v + row + vs, bytes, &full[s]);
        if (GK) bulk_g2s(kbuf + (vs - ws), p.k + row + vs, bytes, &full[s]);
      }
      __syncwarp();
    }
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32<LB, NCH>();
    int gi = -1, g_prev = -1;
    Tile t;
    t.init(tb, p);
    for (int j = 0; j < ntiles; ++j, t.next(p)) {
      const int u = j % NBUF;
      const int g = t.c / p.gs;
      const bool first = g != g_prev;
      const bool last = j + 1 < ntiles && t.last_of_channel(p) && (t.c + 1) / p.gs != g;
      if (first) ++gi;
      g_prev = g;
      mbar_wait(&ufull[u], (j / NBUF) & 1);  // U written and accumulator u drained
      if (first) mbar_wait(tready, gi & 1);
      tc_fence_after();
      const uint32_t d = tmem_base + TM_ACC + u * NCH;
      const uint32_t ub = smem_u32(smem + OFF_U + u * U_BYTES);
      if (elect_one()) {
        for (int k = 0; k <= p.K; ++k) {
#pragma unroll
          for (int ks = 0; ks < LB / 16; ++ks) {
            const uint32_t a = ub + (ks >> 2) * U_ATOM + (HROWS - k) * 128 + (ks & 3) * 32;
            uint64_t bd = desc_sw128(a);
            if (p.base_off) bd |= static_cast<uint64_t>((a >> 7) & 7) << 49;
            mma_bf16_ts(d, tmem_base + TM_F + 64 * k + ks * 8, bd, idesc, (k | ks) ? 1u : 0u);
          }
        }
        mma_commit(&uempty[u]);
        mma_commit(&tfull[u]);
        if (last) mma_commit(tfree);
      }
      __syncwarp();
    }
  } else if (warp < W_EPI0) {
    // ------------------------------------------------------------ converters
    const int ctid = threadIdx.x - W_CONV0 * 32;
    Tile t;
    t.init(tb, p);
    for (int it = 0; it < ntiles; ++it, t.next(p)) {
      const int s = it % STAGES, u = it % NBUF;
      const uint32_t uph = (it / NBUF) & 1;
      mbar_wait(&full[s], (it / STAGES) & 1);
      mbar_wait(&uempty[u], uph ^ 1);
      const unsigned char* st = smem + OFF_ST + s * STAGE_BYTES;
      unsigned char* ub = smem + OFF_U + u * U_BYTES;
      // U rows HROWS - K .. UROWS - 1 = chunks -K .. NCH - 1 of the tile (rows above are unread)
      const int r0 = HROWS - p.K;
      const int nunits = (UROWS - r0) * 16;
      for (int i = ctid; i < nunits; i += CONV_THREADS) {
        const int row = r0 + (i >> 4), jj = i & 15;
        const int off = (row - HROWS + KMAX) * LB + jj * 8;  // element offset in the window
        int4 vv = *reinterpret_cast<const int4*>(st + off * 2);
        if (GK) {
          const int4 kk = *reinterpret_cast<const int4*>(st + WIN_BYTES + off * 2);
          __nv_bfloat162* a = reinterpret_cast<__nv_bfloat162*>(&vv);
          const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&kk);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 x = __bfloat1622float2(a[e]), y = __bfloat1622float2(b[e]);
            a[e] = __floats2bfloat162_rn(x.x * y.x, x.y * y.y);
          }
        }
        *reinterpret_cast<int4*>(ub + sw_off(row, jj)) = vv;
      }
      fence_proxy_async();
      named_bar_sync(BAR_CONV, CONV_THREADS);
      if (ctid == 0) {
        mbar_arrive(&empty[s]);
        mbar_wait(&tempty[u], uph ^ 1);  // accumulator u drained by the epilogue
        mbar_arrive(&ufull[u]);
      }
    }
  } else if (warp < W_TB0) {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;
    const int tout = quarter * 32 + lane;
    Tile t;
    t.init(tb, p);
    for (int it = 0; it < ntiles; ++it, t.next(p)) {
      const int a = it % NBUF;
      const size_t row = static_cast<size_t>(t.b * p.C + t.c) * p.L + t.t0;
      const int nt = min(TILE_T, p.L - t.t0);
      float qv[NCH];
      if (GQ) {  // gate loads in flight while the MMAs run
#pragma unroll
        for (int n = 0; n < NCH; ++n) {
          const int tt = n * LB + tout;
          qv[n] = tt < nt ? __bfloat162float(p.q[row + tt]) : 0.f;
        }
      }
      mbar_wait(&tfull[a], (it / NBUF) & 1);
      tc_fence_after();
      float acc[NCH];
      tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + TM_ACC + a * NCH, acc);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
      bf16* yrow = p.y + row;
#pragma unroll
      for (int n = 0; n < NCH; ++n) {
        const int tt = n * LB + tout;
        float val = acc[n];
        if (GQ) val *= qv[n];
        if (tt < nt) yrow[tt] = __float2bfloat16_rn(val);
      }
    }
  } else if (warp < W_MMA) {
    // ------------------------------------------------------------ factor builder
    const int bt = threadIdx.x - W_TB0 * 32;
    constexpr int PER = HP_N / TB_THREADS;  // hpad entries per thread
    bf16* hpad = reinterpret_cast<bf16*>(smem + OFF_HP);
    const int quarter = warp & 3;
    const int mrow = quarter * 32 + lane;
    const uint32_t trow = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
    // hpad[b][i + 128] = h[i] (decay applied), zero outside [0, lh)
    auto fill = [&](int g, bf16* hb) {
      const float dec = p.decay ? p.decay[g] : 0.f;
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int tt = bt + r * TB_THREADS - 128;
        const float h = (tt >= 0 && tt < p.lh)
                            ? p.taps_hat[static_cast<size_t>(g) * p.lh + tt] * exp2f(-dec * static_cast<float>(tt))
                            : 0.f;
        hb[bt + r * TB_THREADS] = __float2bfloat16_rn(h);
      }
    };
    // factor f into TMEM: lane m = output row, column c = packed pair (T_f[m][2c], T_f[m][2c+1])
    // = (h[128 f + m - 2c], h[128 f + m - 2c - 1]), read as 32-bit words of hpad (one byte
    // permute per pair; for odd p0 both halves sit in one word, for even p0 they straddle two)
    auto build = [&](int fct, const bf16* hbuf) {
      const int p0 = 128 + fct * 128 + mrow;
      const uint32_t* hw = reinterpret_cast<const uint32_t*>(hbuf);
      const uint32_t sel = (p0 & 1) ? 0x1032u : 0x7610u;
      uint32_t wa = hw[p0 >> 1];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t w[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const uint32_t wb = hw[(p0 >> 1) - (half * 32 + c) - 1];
          w[c] = __byte_perm(wa, wb, sel);
          wa = wb;
        }
        tmem_st_32x32b_x32(trow + TM_F + 64 * fct + half * 32, w);
      }
    };
    int gi = 0, g_prev = -1;
    Tile t;
    t.init(tb, p);
    const int g_end = ntiles > 0 ? ((te - 1) / (p.tiles_per_seq * p.B)) / p.gs : -1;
    if (ntiles > 0) fill(t.c / p.gs, hpad);
    named_bar_sync(BAR_TB, TB_THREADS);
    for (int j = 0; j < ntiles; ++j, t.next(p)) {
      const int g = t.c / p.gs;
      if (g == g_prev) continue;
      g_prev = g;
      const bf16* hb = hpad + HP_N * (gi & 1);
      if (gi > 0) mbar_wait(tfree, (gi - 1) & 1);  // the previous group's last MMA retired
      tc_fence_after();
      for (int f = 0; f <= p.K; ++f) build(f, hb);
      tmem_wait_st();
      tc_fence_before();
      named_bar_sync(BAR_TB, TB_THREADS);
      if (bt == 0) mbar_arrive(tready);
      if (g < g_end) fill(g + 1, hpad + HP_N * ((gi + 1) & 1));  // next group's taps, ahead
      named_bar_sync(BAR_TB, TB_THREADS);
      ++gi;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == W_MMA) tmem_dealloc<512>(tmem_base);
}

template <bool GK, bool GQ>
static int launch(const Params& p, cudaStream_t st) {
  auto kern = block_conv_kernel<GK, GQ>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), SMEM_BYTES);
  if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = p.total_tiles < sms ? p.total_tiles : sms;
  kern<<<grid, THREADS, SMEM_BYTES, st>>>(p);
  return check_launch("block_conv_kernel");
}

}  // namespace kb
}  // namespace hy

using namespace hy;

// K-block causal conv (blockconv.py:103-121), optionally gated as two_stage_forward
// (blockconv.py:182-220) and with the MR decay: bf16, 1 <= lh <= 513, L % 8 == 0.
extern "C" HY_API int hy_block_conv_fwd(const void* q, const void* k, const void* v, void* y, const float* taps_hat,
                                        const float* decay, int B, int C, int L, int lh, int gs, int dtype,
                                        void* stream) {
  if (dtype != HY_BF16) return fail(HY_ERR_UNSUPPORTED, "hy_block_conv_fwd: tcgen05 path is bf16 only");
  if (!v || !y || !taps_hat) return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || lh < 1 || gs < 1)
    return fail(HY_ERR_INVALID, "sizes must be >= 1 (B=%d C=%d L=%d lh=%d gs=%d)", B, C, L, lh, gs);
  if (C % gs != 0) return fail(HY_ERR_INVALID, "group_size %d does not divide channel count %d", gs, C);
  if (lh > kb::KMAX * kb::LB + 1)
    return fail(HY_ERR_UNSUPPORTED, "K-block tcgen05 conv supports filter_len <= %d (got %d)", kb::KMAX * kb::LB + 1,
                lh);
  if (L % 8 != 0) return fail(HY_ERR_UNSUPPORTED, "tcgen05 K-block path needs L %% 8 == 0 (L=%d)", L);
  if (!aligned16(v) || !aligned16(y) || (k && !aligned16(k)))
    return fail(HY_ERR_UNSUPPORTED, "tcgen05 K-block path needs 16-byte aligned tensors");
  kb::Params p{};
  p.q = static_cast<const kb::bf16*>(q);
  p.k = static_cast<const kb::bf16*>(k);
  p.v = static_cast<const kb::bf16*>(v);
  p.y = static_cast<kb::bf16*>(y);
  p.taps_hat = taps_hat;
  p.decay = decay;
  p.B = B, p.C = C, p.L = L, p.lh = lh, p.gs = gs;
  p.K = (lh - 1 + kb::LB - 1) / kb::LB;
  p.tiles_per_seq = (L + kb::TILE_T - 1) / kb::TILE_T;
  p.total_tiles = p.tiles_per_seq * B * C;
  static const int bo = [] { const char* e = getenv("HY_KB_BASE_OFFSET"); return e ? atoi(e) : 0; }();
  p.base_off = bo;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (q && k) return kb::launch<true, true>(p, st);
  if (k) return kb::launch<true, false>(p, st);
  if (q) return kb::launch<false, true>(p, st);
  return kb::launch<false, false>(p, st);
}
