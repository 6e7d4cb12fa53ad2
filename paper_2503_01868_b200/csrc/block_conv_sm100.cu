// Blocked causal convolutions on 5th-gen tensor cores (sm_100a) from staged rows: the K-block
// conv for filters longer than one spill factor, and the implicit-filter (Hyena-LI) long conv.
//
// Explicit mode restates blockconv.py:103-121 (block_conv: Y_n = sum_{k=0..K} B_k U_{n-k},
// K = ceil((lh-1)/lb)) at the kernel's own block length LB = 128 (any block size gives the same
// causal sum), 1 <= lh <= 513, with the optional gates of two_stage_forward (y = q * conv(k * v),
// blockconv.py:182-220) and the regularisation decay applied in-kernel (core.py:144-146):
//
//     D[t_out][chunk] = sum_{k=0..K} T_k[t_out][:] . U_{chunk-k}[:]        (K + 1) x 8 MMAs per tile
//     T_k[m][j] = h[128 k + m - j]   (Toeplitz factors, A operand in TMEM, built in-kernel)
//
// Implicit mode (IMPL) computes the long conv with h_t = sum_n R_n lam_n^t (core.py:147-151, the
// conv of fft.py:128-145) exactly, without the filter or an FFT: the intra-chunk part is T_0 . U,
// every longer lag goes through the per-mode states s_n[t] = lam_n s_n[t-1] + u[t]:
//     E[n][chunk] = sum_t lam_n^(127-t) U[chunk][t]          (Lam . U, one more MMA per K-step)
//     S_c = lam^128 S_{c-1} + E_{c-1}                        (scan warp, carried tile to tile)
//     D[t_out][chunk] += sum_n R_n lam_n^(t_out+1) S_c[n]     (P . S_prev, one tf32 MMA)
//
// Tile = NCH = 64 consecutive 128-step chunks of one sequence (MMA N = 64: half the MMA issues
// per byte of a 32-chunk tile). The shifted operands U_{n-k} are NOT copies: the U buffer holds
// the tile's chunks plus the K chunks before them as rows of one SW128 K-major matrix (row r =
// chunk r - HROWS), and the MMA for factor k reads it through a descriptor starting k rows
// earlier (a 128-byte row offset inside the swizzle atom: the swizzle is a function of the
// address, so the view is exact). Rows arrive by 1-D bulk copies into a ring sized so that
// ~130 KB per SM are in flight (8 stages ungated, 4 gated).
//
// Warp roles (608 threads, 1 CTA per SM, persistent over a contiguous tile range; IMPL ranges
// hold whole sequences, whose modal state is carried tile to tile):
//   warps 0-3   converter: staged raw v (and k) -> u = k * v -> bf16 swizzled U rows
//   warps 4-11  epilogue : TMEM acc -> y = q * acc (q read from HBM) -> coalesced stores
//                          (two warps per TMEM lane quarter, 32 of the 64 columns each)
//   warps 12-15 factor builder: the filter group's factors (T_0..T_K; IMPL: T_0, Lam, P) into
//                          TMEM / SMEM, double-buffered where TMEM allows (IMPL), else once the
//                          last MMA of the previous group retired (the next group's taps are
//                          prefetched into a second tap buffer)
//   warp 16     scan     : IMPL only — E from TMEM, the chunk recurrence, S_prev -> SMEM, and
//                          the P . S_prev tf32 MMA that completes the tile
//   warp 17     MMA      : TMEM alloc (512 cols); one lane issues the tile's MMAs
//   warp 18     producer : bulk copies of the v / k windows into the ring
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace hy {
namespace kb {

using bf16 = __nv_bfloat16;
using namespace sm100;

constexpr int LB = 128;
constexpr int NCH = 64;
constexpr int TILE_T = NCH * LB;
constexpr int KMAX = 4;                   // spill factors: lh <= KMAX * LB + 1
constexpr int HROWS = 8;                  // U rows before the tile's first chunk (>= KMAX)
constexpr int UROWS = NCH + HROWS;        // 72 rows: 9 groups of 8
constexpr int NPOLE = 8;                  // IMPL: modes per group (zero padded)
constexpr int NBUF = 3;
constexpr int N_EPI_WARPS = 8, N_TB_WARPS = 4;
constexpr int TB_THREADS = N_TB_WARPS * 32;
// Warp roles; FEAT (the fused mixers: featurizer FIRs on the converter warps) doubles the
// converter warps
template <bool FEAT>
struct Roles {
  static constexpr int N_CONV = FEAT ? 8 : 4;
  static constexpr int W_EPI0 = N_CONV, W_TB0 = W_EPI0 + N_EPI_WARPS, W_SCAN = W_TB0 + N_TB_WARPS,
                       W_MMA = W_SCAN + 1, W_PROD = W_MMA + 1, THREADS = (W_PROD + 1) * 32,
                       CONV_THREADS = N_CONV * 32;
};
constexpr uint32_t BAR_CONV = 1, BAR_TB = 2;
// TMEM columns: accumulators [NBUF] x 64; explicit factors T_k at TM_F + 64 k; IMPL: T_0 of
// group buffer b at TM_F + 64 b, mode inputs E [2] x 64 at TM_E
constexpr uint32_t TM_ACC = 0, TM_F = NBUF * NCH, TM_E = TM_F + 128;
static_assert(TM_F + 64 * (KMAX + 1) <= 512 && TM_E + 2 * NCH <= 512, "TMEM budget");
static_assert(HROWS >= KMAX && UROWS % 8 == 0, "U rows");

constexpr int round_up(int a, int m) { return (a + m - 1) / m * m; }
constexpr int FH = 8;                                      // FEAT: featurizer history steps
constexpr int RING_BYTES = 8 * (TILE_T + KMAX * LB) * 2;  // 139264: 8 ungated / 4 gated windows
// FEAT: 2 stages of q / k / v windows, then the featurized q of each accumulator buffer
constexpr int FQ_BYTES = TILE_T * 2;
constexpr int U_ATOM = UROWS * 128;                        // one 64-element K atom of the U matrix
constexpr int U_BYTES = 2 * U_ATOM;
constexpr int OFF_ST = 0;
// FEAT stages hold one chunk of explicit history at most (the fused MR mixer, K <= 1)
constexpr int OFF_U = round_up(2 * 3 * (TILE_T + LB + FH) * 2 + NBUF * FQ_BYTES, 1024);
static_assert(OFF_U >= RING_BYTES, "ring");
constexpr int HP_N = 1024;                                 // hpad[i + 128] = h[i], i in [-128, 896)
constexpr int OFF_HP = OFF_U + NBUF * U_BYTES;             // two tap buffers (this group / next)
constexpr int OFF_L = round_up(OFF_HP + 2 * HP_N * 2, 1024);  // IMPL: Lam[2] (bf16 SW128, 8 rows)
constexpr int OFF_P = OFF_L + 2 * 2048;                    // IMPL: P[2] (tf32, 128 x 8)
constexpr int OFF_S = OFF_P + 2 * 4096;                    // IMPL: S_prev[NBUF] (tf32, 64 x 8)
constexpr int OFF_BAR = OFF_S + NBUF * NCH * NPOLE * 4;
constexpr int N_BARS = 2 * 8 + 5 * NBUF + 10;
constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
constexpr int SMEM_BYTES = OFF_TMEM + 16 + 1024;
static_assert(SMEM_BYTES <= 232448, "shared memory budget");

struct Params {
  const bf16* proj;       // FEAT: (B, 3C, L) projections [q; k; v]
  const float* feat;      // FEAT: (3, C, lhf) featurizer taps, lhf <= 8
  const bf16* q;
  const bf16* k;
  const bf16* v;
  bf16* y;
  const float* taps_hat;  // explicit: (n_groups, lh)
  const float* decay;     // explicit: (n_groups) rate * log2(base), or null
  const float* poles;     // IMPL: (n_groups, npoles)
  const float* residues;
  int npoles;
  int B, C, L, lh, K, gs, lhf;
  int tiles_per_seq, total_tiles;
  // rows stored as L / seg_len time segments: element (row, t) at row * seg_len +
  // (t / seg_len) * seg_stride + t % seg_len (the rank-major all-to-all buffer); 0 = plain rows
  int seg_len;
  long long seg_stride;
};

__device__ __forceinline__ size_t elem_off(const Params& p, int row, int t) {
  if (p.seg_len == 0) return static_cast<size_t>(row) * p.L + t;
  const int sg = t / p.seg_len;
  return static_cast<size_t>(row) * p.seg_len + static_cast<size_t>(sg) * p.seg_stride + (t - sg * p.seg_len);
}

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

__device__ __forceinline__ int4 pack8(const float* in) {
  int4 raw;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(in[2 * i], in[2 * i + 1]);
  return raw;
}

// Featurizer FIR (hyena.py:122-126, taps zero padded to 8) of the 8 steps at window offset off:
// out[e] = sum_j h[j] w[off + e - j], from the unit before (history) and the unit itself, as
// packed FFMA2 on output pairs (the odd-aligned input pairs are formed once)
__device__ __forceinline__ void feat_unit(const unsigned char* win, int off, const float* h, float* out) {
  const int4 a = *reinterpret_cast<const int4*>(win + (off - 8) * 2);
  const int4 b = *reinterpret_cast<const int4*>(win + off * 2);
  float2 ev[8];  // ev[i] = (w[off - 8 + 2i], w[off - 7 + 2i])
  const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    ev[i] = __bfloat1622float2(pa[i]);
    ev[4 + i] = __bfloat1622float2(pb[i]);
  }
  float2 od[7];  // od[i] = (w[off - 7 + 2i], w[off - 6 + 2i])
#pragma unroll
  for (int i = 0; i < 7; ++i) od[i] = make_float2(ev[i].y, ev[i + 1].x);
#pragma unroll
  for (int e = 0; e < 8; e += 2) {
    float2 acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i0 = 8 + e - j;  // window index (relative to off - 8) of the pair's first input
      const float2 x = (i0 & 1) ? od[(i0 - 1) >> 1] : ev[i0 >> 1];
      acc = __ffma2_rn(make_float2(h[j], h[j]), x, acc);
    }
    out[e] = acc.x;
    out[e + 1] = acc.y;
  }
}

// No-swizzle K-major descriptor with explicit leading / stride byte offsets.
__device__ __forceinline__ uint64_t desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (static_cast<uint64_t>((saddr >> 4) & 0x3FFF)) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(sbo >> 4) << 32) | (static_cast<uint64_t>(1) << 46);
}

template <bool GK, bool GQ, bool IMPL, bool FEAT>
__global__ void __launch_bounds__(Roles<FEAT>::THREADS, 1) block_conv_kernel(const Params p) {
  using R = Roles<FEAT>;
  constexpr int W_EPI0 = R::W_EPI0, W_TB0 = R::W_TB0, W_SCAN = R::W_SCAN, W_MMA = R::W_MMA, W_PROD = R::W_PROD;
  constexpr int CONV_THREADS = R::CONV_THREADS;
  constexpr int KH = IMPL ? 0 : (FEAT ? 1 : KMAX);  // history chunks staged before the tile
  constexpr int HS = KH * LB + (FEAT ? FH : 0); // history steps staged before the tile
  constexpr int WIN = TILE_T + HS;              // staged window per tensor (steps)
  constexpr int WIN_BYTES = WIN * 2;
  constexpr int NWIN = FEAT ? 3 : (GK ? 2 : 1); // windows per stage: [v, k] or FEAT [v, k, q]
  constexpr int STAGE_BYTES = NWIN * WIN_BYTES;
  constexpr int STAGES = FEAT ? 2 : RING_BYTES / STAGE_BYTES;
  constexpr int OFF_FQ = STAGES * STAGE_BYTES;  // FEAT: featurized q [NBUF]
  static_assert(FEAT || (STAGES >= 4 && STAGES <= 8), "ring depth");
  static_assert(!FEAT || OFF_FQ + NBUF * FQ_BYTES <= OFF_U, "FEAT ring");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* full = bars;           // [STAGES]
  uint64_t* empty = bars + 8;      // [STAGES]
  uint64_t* ufull = bars + 16;     // [NBUF] converter -> MMA (U written, accumulator drained)
  uint64_t* uempty = ufull + NBUF; // [NBUF] MMA commit -> converter
  uint64_t* tfull = uempty + NBUF; // [NBUF] MMA / scan commit -> epilogue
  uint64_t* tempty = tfull + NBUF; // [NBUF] epilogue warps -> converter
  uint64_t* tready = tempty + NBUF;  // [2] builder -> MMA: group factors of buffer b
  uint64_t* tfree = tready + 2;      // [2] MMA commit: last T . U (and Lam . U) of buffer b retired
  uint64_t* tfreep = tfree + 2;      // [2] IMPL scan commit: last P . S_prev of buffer b retired
  uint64_t* efull = tfreep + 2;      // [2] IMPL: MMA commit -> scan (E in TMEM)
  uint64_t* eempty = efull + 2;      // [2] IMPL: scan -> converter (E drained)
  uint64_t* qfull = eempty + 2;      // [NBUF] FEAT: converter -> epilogue (featurized q in SMEM)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int units = IMPL ? p.total_tiles / p.tiles_per_seq : p.total_tiles;
  const int per = IMPL ? p.tiles_per_seq : 1;
  const int tb = per * static_cast<int>((static_cast<long long>(blockIdx.x) * units) / gridDim.x);
  const int te = per * static_cast<int>((static_cast<long long>(blockIdx.x + 1) * units) / gridDim.x);
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
      mbar_init(&qfull[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tready[i], 1);
      mbar_init(&tfree[i], 1);
      mbar_init(&tfreep[i], 1);
      mbar_init(&efull[i], 1);
      mbar_init(&eempty[i], 1);
    }
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
      const int ws = t.t0 - HS, we = t.t0 + TILE_T;
      const int vs = max(ws, 0), ve = min(we, p.L);
      if (vs != ws || ve != we) {  // zero the windows outside [0, L) (whole 16-byte units)
        const int4 z = make_int4(0, 0, 0, 0);
#pragma unroll
        for (int x = 0; x < NWIN; ++x) {
          bf16* wb = reinterpret_cast<bf16*>(st + x * WIN_BYTES);
          for (int i = lane * 8; i < vs - ws; i += 256) *reinterpret_cast<int4*>(wb + i) = z;
          for (int i = (ve - ws) + lane * 8; i < WIN; i += 256) *reinterpret_cast<int4*>(wb + i) = z;
        }
        fence_proxy_async();
      }
      __syncwarp();
      if (elect_one()) {
        // a window never crosses a segment of the segmented layout (seg_len % TILE_T == 0, and
        // the explicit history is used with plain rows only)
        const uint32_t bytes = static_cast<uint32_t>(ve - vs) * 2;
        mbar_arrive_expect_tx(&full[s], bytes * NWIN);
        if (FEAT) {
          const size_t r0 = (static_cast<size_t>(t.b) * 3 * p.C + t.c) * p.L + vs;  // q row
          const size_t cl = static_cast<size_t>(p.C) * p.L;
          bulk_g2s(st + (vs - ws) * 2, p.proj + r0 + 2 * cl, bytes, &full[s]);                  // v
          bulk_g2s(st + WIN_BYTES + (vs - ws) * 2, p.proj + r0 + cl, bytes, &full[s]);          // k
          bulk_g2s(st + 2 * WIN_BYTES + (vs - ws) * 2, p.proj + r0, bytes, &full[s]);           // q
        } else {
          const size_t off = elem_off(p, t.b * p.C + t.c, vs);
          bulk_g2s(st + (vs - ws) * 2, p.v + off, bytes, &full[s]);
          if (GK) bulk_g2s(st + WIN_BYTES + (vs - ws) * 2, p.k + off, bytes, &full[s]);
        }
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
      const int fb = IMPL ? (gi & 1) : 0;  // factor buffer of this group
      mbar_wait(&ufull[u], (j / NBUF) & 1);  // U written, accumulator (and E) buffer drained
      if (first) mbar_wait(&tready[fb], IMPL ? ((gi >> 1) & 1) : (gi & 1));
      tc_fence_after();
      const uint32_t d = tmem_base + TM_ACC + u * NCH;
      const uint32_t ub = smem_u32(smem + OFF_U + u * U_BYTES);
      if (elect_one()) {
        if (IMPL) {
          const uint32_t ta = tmem_base + TM_F + 64 * fb;
          const uint32_t la = smem_u32(smem + OFF_L + fb * 2048);
          const uint32_t de = tmem_base + TM_E + (j & 1) * NCH;
#pragma unroll
          for (int ks = 0; ks < LB / 16; ++ks) {
            const uint32_t a = ub + (ks >> 2) * U_ATOM + HROWS * 128 + (ks & 3) * 32;
            mma_bf16_ts(d, ta + ks * 8, desc_sw128(a), idesc, ks > 0 ? 1u : 0u);
          }
#pragma unroll
          for (int ks = 0; ks < LB / 16; ++ks) {
            const uint32_t a = ub + (ks >> 2) * U_ATOM + HROWS * 128 + (ks & 3) * 32;
            mma_bf16(de, desc_sw128_sbo(la + (ks >> 2) * 1024 + (ks & 3) * 32, 0), desc_sw128(a),
                     idesc_bf16_f32<64, NCH>(), ks > 0 ? 1u : 0u);  // M = 64: half the Lam re-reads
          }
          mma_commit(&efull[j & 1]);
          mma_commit(&uempty[u]);
          if (last) mma_commit(&tfree[fb]);
        } else {
          for (int k = 0; k <= p.K; ++k) {
#pragma unroll
            for (int ks = 0; ks < LB / 16; ++ks) {
              const uint32_t a = ub + (ks >> 2) * U_ATOM + (HROWS - k) * 128 + (ks & 3) * 32;
              mma_bf16_ts(d, tmem_base + TM_F + 64 * k + ks * 8, desc_sw128(a), idesc, (k | ks) ? 1u : 0u);
            }
          }
          mma_commit(&uempty[u]);
          mma_commit(&tfull[u]);
          if (last) mma_commit(&tfree[0]);
        }
      }
      __syncwarp();
    }
  } else if (warp < W_EPI0) {
    // ------------------------------------------------------------ converters
    const int ctid = threadIdx.x;
    Tile t;
    t.init(tb, p);
    int fc = -1;
    float fh[3][8];  // FEAT: [q, k, v] featurizer taps of the tile's channel
    for (int it = 0; it < ntiles; ++it, t.next(p)) {
      const int s = it % STAGES, u = it % NBUF;
      const uint32_t uph = (it / NBUF) & 1;
      if (FEAT && t.c != fc) {
        fc = t.c;
#pragma unroll
        for (int x = 0; x < 3; ++x)
#pragma unroll
          for (int j = 0; j < 8; ++j)
            fh[x][j] = j < p.lhf ? p.feat[(static_cast<size_t>(x) * p.C + t.c) * p.lhf + j] : 0.f;
      }
      mbar_wait(&full[s], (it / STAGES) & 1);
      mbar_wait(&uempty[u], uph ^ 1);
      const unsigned char* st = smem + OFF_ST + s * STAGE_BYTES;
      unsigned char* ub = smem + OFF_U + u * U_BYTES;
      // U rows HROWS - K .. UROWS - 1 = chunks -K .. NCH - 1 of the tile (rows above are unread)
      const int r0 = HROWS - (IMPL ? 0 : p.K);
      const int nunits = (UROWS - r0) * 16;
      if (FEAT) {
        // u = Fk(pk) * Fv(pv) per 8-step unit from the raw windows (8 steps of history each)
        for (int i = ctid; i < nunits; i += CONV_THREADS) {
          const int row = r0 + (i >> 4), jj = i & 15;
          const int off = (row - HROWS) * LB + KH * LB + FH + jj * 8;  // window offset of the unit
          float fv[8], fk[8];
          feat_unit(st, off, fh[2], fv);
          feat_unit(st + WIN_BYTES, off, fh[1], fk);
#pragma unroll
          for (int e = 0; e < 8; ++e) fv[e] *= fk[e];
          *reinterpret_cast<int4*>(ub + sw_off(row, jj)) = pack8(fv);
        }
        // featurized q of the tile -> FQ[u] (natural order), once the epilogue drained buffer u
        if (ctid == 0) mbar_wait(&tempty[u], uph ^ 1);
        named_bar_sync(BAR_CONV, CONV_THREADS);
        bf16* fqb = reinterpret_cast<bf16*>(smem + OFF_FQ + u * FQ_BYTES);
        for (int i = ctid; i < TILE_T / 8; i += CONV_THREADS) {
          float fq[8];
          feat_unit(st + 2 * WIN_BYTES, KH * LB + FH + i * 8, fh[0], fq);
          *reinterpret_cast<int4*>(fqb + i * 8) = pack8(fq);
        }
        named_bar_sync(BAR_CONV, CONV_THREADS);
        if (ctid == 0) mbar_arrive(&qfull[u]);
      }
      for (int i = FEAT ? nunits : ctid; i < nunits; i += CONV_THREADS) {
        const int row = r0 + (i >> 4), jj = i & 15;
        const int off = (row - HROWS + KH) * LB + jj * 8;  // element offset in the window
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
        if (!FEAT) mbar_wait(&tempty[u], uph ^ 1);                  // accumulator u drained
        if (IMPL) mbar_wait(&eempty[it & 1], ((it >> 1) & 1) ^ 1);  // E buffer drained by the scan
        mbar_arrive(&ufull[u]);
      }
    }
  } else if (warp < W_TB0) {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;
    const int colh = (warp - W_EPI0) >> 2;  // which 32 of the 64 chunk columns
    const int tout = quarter * 32 + lane;
    Tile t;
    t.init(tb, p);
    for (int it = 0; it < ntiles; ++it, t.next(p)) {
      const int a = it % NBUF;
      const int row = t.b * p.C + t.c;
      const int nt = min(TILE_T, p.L - t.t0);
      const size_t roff = elem_off(p, row, t.t0);  // a tile never crosses a segment
      float qv[32];
      if (GQ && !FEAT) {  // gate loads in flight while the MMAs run
#pragma unroll
        for (int n = 0; n < 32; ++n) {
          const int tt = (colh * 32 + n) * LB + tout;
          qv[n] = tt < nt ? __bfloat162float(p.q[roff + tt]) : 0.f;
        }
      }
      mbar_wait(&tfull[a], (it / NBUF) & 1);
      tc_fence_after();
      float acc[32];
      tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + TM_ACC + a * NCH + colh * 32,
                         acc);
      tc_fence_before();
      __syncwarp();
      if (!FEAT && lane == 0) mbar_arrive(&tempty[a]);
      bf16* yrow = p.y + roff;
      if (FEAT) {  // gate with the featurized q the converters left in FQ[a]
        mbar_wait(&qfull[a], (it / NBUF) & 1);
        const bf16* fqb = reinterpret_cast<const bf16*>(smem + OFF_FQ + a * FQ_BYTES);
#pragma unroll
        for (int n = 0; n < 32; ++n) qv[n] = __bfloat162float(fqb[(colh * 32 + n) * LB + tout]);
      }
#pragma unroll
      for (int n = 0; n < 32; ++n) {
        const int tt = (colh * 32 + n) * LB + tout;
        float val = acc[n];
        if (GQ || FEAT) val *= qv[n];
        if (tt < nt) yrow[tt] = __float2bfloat16_rn(val);
      }
      if (FEAT) {  // accumulator and FQ[a] both free
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[a]);
      }
    }
  } else if (warp < W_SCAN) {
    // ------------------------------------------------------------ factor builder
    const int bt = threadIdx.x - W_TB0 * 32;
    constexpr int PER = HP_N / TB_THREADS;  // hpad entries per thread
    bf16* hpad = reinterpret_cast<bf16*>(smem + OFF_HP);
    const int quarter = warp & 3;
    const int mrow = quarter * 32 + lane;
    const uint32_t trow = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
    // explicit: hpad[b][i + 128] = h[i] (decay applied), zero outside [0, lh)
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
    // factor f into TMEM columns tcol: lane m = output row, column c = packed pair
    // (T_f[m][2c], T_f[m][2c+1]) = (h[128 f + m - 2c], h[128 f + m - 2c - 1]), read as 32-bit
    // words of hpad (one byte permute per pair; consecutive columns share a word)
    auto build = [&](int fct, uint32_t tcol, const bf16* hbuf) {
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
        tmem_st_32x32b_x32(trow + tcol + half * 32, w);
      }
    };
    Tile t;
    t.init(tb, p);
    const int g_end = ntiles > 0 ? ((te - 1) / (p.tiles_per_seq * p.B)) / p.gs : -1;
    if (IMPL) {
      // group gb's factors into buffer gb & 1, one group ahead, once group gb - 2's readers
      // retired: T_0 from h[t] = sum_n R_n lam_n^t (t < 128) in TMEM; P[m][n] = R_n lam_n^(m+1)
      // (tf32 A operand, element (m, n) at (m%8)*16 + (m/8)*256 + (n%4)*4 + (n/4)*128 bytes);
      // Lam[n][t] = lam_n^(127 - t) (bf16, SW128 K-major, 8 rows)
      auto build_impl = [&](int gb, int g) {
        const int b = gb & 1;
        if (gb >= 2) {
          mbar_wait(&tfree[b], ((gb - 2) >> 1) & 1);
          mbar_wait(&tfreep[b], ((gb - 2) >> 1) & 1);
        }
        float hv = 0.f, pm[NPOLE];
        unsigned char* lrow = smem + OFF_L + b * 2048 + (bt >> 6) * 1024 + (bt & 7) * 2;
#pragma unroll
        for (int n = 0; n < NPOLE; ++n) {
          const bool ok = n < p.npoles;
          const float lam = ok ? p.poles[static_cast<size_t>(g) * p.npoles + n] : 0.f;
          const float res = ok ? p.residues[static_cast<size_t>(g) * p.npoles + n] : 0.f;
          const float la = log2f(fabsf(lam));
          // lam^e for integer e as exp2(e log2|lam|) with the sign of lam^e (0^0 = 1)
          auto ipow = [&](int e) {
            if (e == 0) return 1.f;
            if (lam == 0.f) return 0.f;
            const float m = exp2f(static_cast<float>(e) * la);
            return (lam < 0.f && (e & 1)) ? -m : m;
          };
          const float lt = ipow(bt);
          hv = fmaf(res, lt, hv);
          pm[n] = res * lt * lam;
          const int jj = (bt >> 3) & 7;
          *reinterpret_cast<bf16*>(lrow + n * 128 + ((jj ^ n) << 4)) = __float2bfloat16_rn(ipow(127 - bt));
        }
        bf16* hb = hpad + HP_N * b;
        hb[bt] = __float2bfloat16_rn(0.f);
        hb[128 + bt] = __float2bfloat16_rn(hv);
        float* pa = reinterpret_cast<float*>(smem + OFF_P + b * 4096 + (bt & 7) * 16 + (bt >> 3) * 256);
        *reinterpret_cast<float4*>(pa) = make_float4(pm[0], pm[1], pm[2], pm[3]);
        *reinterpret_cast<float4*>(pa + 32) = make_float4(pm[4], pm[5], pm[6], pm[7]);
        fence_proxy_async();
        named_bar_sync(BAR_TB, TB_THREADS);
        tc_fence_after();
        build(0, TM_F + 64 * b, hb);
        tmem_wait_st();
        tc_fence_before();
        named_bar_sync(BAR_TB, TB_THREADS);
        if (bt == 0) mbar_arrive(&tready[b]);
      };
      int gi = 0, g_prev = -1;
      for (int j = 0; j < ntiles; ++j, t.next(p)) {
        const int g = t.c / p.gs;
        if (g == g_prev) continue;
        g_prev = g;
        if (gi == 0) build_impl(0, g);
        if (g < g_end) build_impl(gi + 1, g + 1);  // the next group, into the other buffer
        ++gi;
      }
    } else {
      int gi = 0, g_prev = -1;
      if (ntiles > 0) fill(t.c / p.gs, hpad);
      named_bar_sync(BAR_TB, TB_THREADS);
      for (int j = 0; j < ntiles; ++j, t.next(p)) {
        const int g = t.c / p.gs;
        if (g == g_prev) continue;
        g_prev = g;
        const bf16* hb = hpad + HP_N * (gi & 1);
        if (gi > 0) mbar_wait(&tfree[0], (gi - 1) & 1);  // the previous group's last MMA retired
        tc_fence_after();
        for (int f = 0; f <= p.K; ++f) build(f, TM_F + 64 * f, hb);
        tmem_wait_st();
        tc_fence_before();
        named_bar_sync(BAR_TB, TB_THREADS);
        if (bt == 0) mbar_arrive(&tready[0]);
        if (g < g_end) fill(g + 1, hpad + HP_N * ((gi + 1) & 1));  // next group's taps, ahead
        named_bar_sync(BAR_TB, TB_THREADS);
        ++gi;
      }
    }
  } else if (warp == W_SCAN) {
    // ------------------------------------------------------------ IMPL state scan
    // lane n < NPOLE = mode n: E[n][chunk] from TMEM, S_c = lam^128 S_{c-1} + E_{c-1} over the
    // tile's chunks (carried to the next tile of the sequence), S_prev[c][n] as the tf32 B operand
    // (element (c, n) at (c%8)*16 + (c/8)*256 + (n%4)*4 + (n/4)*128 bytes), then D += P . S_prev
    if (IMPL) {
      constexpr uint32_t idesc_tf32 = idesc_tf32_f32<LB, NCH>();
      const int g_end = ntiles > 0 ? ((te - 1) / (p.tiles_per_seq * p.B)) / p.gs : -1;
      auto pole = [&](int g) {
        return (lane < NPOLE && lane < p.npoles) ? p.poles[static_cast<size_t>(g) * p.npoles + lane] : 0.f;
      };
      float lam128 = 0.f, carry = 0.f;
      int gi = -1, g_prev = -1;
      Tile t;
      t.init(tb, p);
      float pf = ntiles > 0 ? pole(t.c / p.gs) : 0.f;
      for (int j = 0; j < ntiles; ++j, t.next(p)) {
        const int g = t.c / p.gs;
        const bool lst = j + 1 < ntiles && t.last_of_channel(p) && (t.c + 1) / p.gs != g;
        if (g != g_prev) {
          g_prev = g;
          ++gi;
          lam128 = powf(pf, 128.f);
          if (g < g_end) pf = pole(g + 1);
        }
        const int fb = gi & 1, eb = j & 1, a = j % NBUF;
        mbar_wait(&efull[eb], (j >> 1) & 1);
        tc_fence_after();
        float ev[NCH];
        tmem_ld_32x32b_x32(tmem_base + TM_E + eb * NCH, *reinterpret_cast<float(*)[32]>(ev));
        tmem_ld_32x32b_x32(tmem_base + TM_E + eb * NCH + 32, *reinterpret_cast<float(*)[32]>(ev + 32));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&eempty[eb]);
        float* sp = reinterpret_cast<float*>(smem + OFF_S + a * NCH * NPOLE * 4);
        float st = t.t0 == 0 ? 0.f : carry;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          if (lane < NPOLE) sp[((c & 7) * 16 + (c >> 3) * 256 + (lane & 3) * 4 + (lane >> 2) * 128) / 4] = st;
          st = fmaf(lam128, st, ev[c]);
        }
        carry = st;
        fence_proxy_async();
        __syncwarp();
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(sp);
          mma_tf32(tmem_base + TM_ACC + a * NCH, desc_noswz(smem_u32(smem + OFF_P + fb * 4096), 128, 256),
                   desc_noswz(sa, 128, 256), idesc_tf32, 1u);
          if (lst) mma_commit(&tfreep[fb]);
          mma_commit(&tfull[a]);
        }
        __syncwarp();
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == W_MMA) tmem_dealloc<512>(tmem_base);
}

template <bool GK, bool GQ, bool IMPL, bool FEAT = false>
static int launch(const Params& p, cudaStream_t st) {
  auto kern = block_conv_kernel<GK, GQ, IMPL, FEAT>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), SMEM_BYTES);
  if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = IMPL ? p.total_tiles / p.tiles_per_seq : p.total_tiles;  // IMPL: whole sequences
  const int grid = units < sms ? units : sms;
  kern<<<grid, Roles<FEAT>::THREADS, SMEM_BYTES, st>>>(p);
  return check_launch("block_conv_kernel");
}

template <bool IMPL>
static int dispatch(const Params& p, bool q, bool k, cudaStream_t st) {
  if (q && k) return launch<true, true, IMPL>(p, st);
  if (k) return launch<true, false, IMPL>(p, st);
  if (q) return launch<false, true, IMPL>(p, st);
  return launch<false, false, IMPL>(p, st);
}

}  // namespace kb

// Fused mixers on the staged-row kernel (FEAT): featurizers (lhf <= 8) on the converter warps,
// u = k * v, the long conv (implicit filter when residues / poles are given, else the K-block
// explicit conv with the MR decay), q gate -- from the (B, 3C, L) projections, one pass.
int mixer_tc_fwd(const void* proj, void* y, const float* feat_taps, int lhf, const float* taps_hat,
                 const float* decay, int lh, const float* residues, const float* poles, int npoles, int gs, int B,
                 int C, int L, void* stream) {
  kb::Params p{};
  p.proj = static_cast<const kb::bf16*>(proj);
  p.feat = feat_taps;
  p.lhf = lhf;
  p.y = static_cast<kb::bf16*>(y);
  p.taps_hat = taps_hat;
  p.decay = decay;
  p.poles = poles;
  p.residues = residues;
  p.npoles = npoles;
  p.B = B, p.C = C, p.L = L, p.gs = gs;
  p.lh = residues ? 1 : lh;
  p.K = residues ? 0 : (lh - 1 + kb::LB - 1) / kb::LB;
  if (p.K > 1) return fail(HY_ERR_UNSUPPORTED, "fused staged-row mixer holds one spill factor (lh <= 129)");
  p.tiles_per_seq = (L + kb::TILE_T - 1) / kb::TILE_T;
  p.total_tiles = p.tiles_per_seq * B * C;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (residues) return kb::launch<true, true, true, true>(p, st);
  return kb::launch<true, true, false, true>(p, st);
}

// Implicit-filter long conv on the staged-row tcgen05 kernel (two_stage_sm100.cu's li_conv
// entry points route here): plain rows (seg_len = 0) or the segmented all-to-all layout.
int li_conv_tc_fwd(const void* q, const void* k, const void* v, void* y, const float* residues, const float* poles,
                   int npoles, int gs, int B, int C, int L, int seg_len, long long seg_stride, void* stream) {
  kb::Params p{};
  p.q = static_cast<const kb::bf16*>(q);
  p.k = static_cast<const kb::bf16*>(k);
  p.v = static_cast<const kb::bf16*>(v);
  p.y = static_cast<kb::bf16*>(y);
  p.poles = poles;
  p.residues = residues;
  p.npoles = npoles;
  p.B = B, p.C = C, p.L = L, p.lh = 1, p.K = 0, p.gs = gs;
  p.seg_len = seg_len;
  p.seg_stride = seg_stride;
  p.tiles_per_seq = (L + kb::TILE_T - 1) / kb::TILE_T;
  p.total_tiles = p.tiles_per_seq * B * C;
  return kb::dispatch<true>(p, q != nullptr, k != nullptr, static_cast<cudaStream_t>(stream));
}

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
  return kb::dispatch<false>(p, q != nullptr, k != nullptr, static_cast<cudaStream_t>(stream));
}
