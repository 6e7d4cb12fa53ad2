// Two-stage blocked causal convolution on 5th-gen tensor cores (sm_100a).
//
// Restates blockconv.py:160-220 (two_stage_forward / _two_stage_core) and, in
// the fused form, hyena.py:162-186 (featurizers + gates), bf16 in / fp32 accumulate:
//
//     k, v, q = featurizer FIRs of the raw rows     (tcgen05, overlapping windows)
//     u = k * v                                      (CUDA cores, TMEM -> SMEM)
//     Y_n = T0 . U_n + T1 . U_{n-1}                  (tcgen05, 128-step chunks)
//     y = q * Y                                      (CUDA cores, TMEM -> HBM)
//
// Main GEMM per tile (one sequence (b, c), NCH = 32 consecutive 128-step chunks):
//   D[t_out][chunk] = T0[t_out][:] . U[chunk][:] + T1[t_out][:] . U_prev[chunk][:]
//   M = 128, N = 32, K = 128; A = T0/T1 built in SMEM from taps_hat with the
//   regularisation decay exp2(-rate*log2(base)*t) applied in-kernel (SW128 K-major),
//   B = U / U_prev written by the converter warps (SW128 K-major), D in TMEM.
//
// Featurizer GEMMs (short FIR of <= 16 taps, on the raw staged rows): the staged
// row p is read as overlapping 8-step windows, A[m][k] = p[8m + k] — the
// no-swizzle K-major canonical layout with LBO = 16 B and SBO = 128 B — so that
//   D[m][n] = sum_k A[m][k] F[n][k] = feat(8m + 8*KS + n),  F[n][k] = h[8*KS + n - k],
// M = 128 windows (1024 outputs) per MMA, N = 16 (8 used), K = 16*KS. Each TMEM
// lane then holds 8 consecutive featurized samples: exactly one 16-byte unit of
// the U operand.
//
// Warp roles (608 threads, 1 CTA per SM, persistent over a contiguous tile range):
//   warps 0-7   converter: TMEM feat -> u = k*v -> bf16 swizzled U / U_prev and
//                          featurized q -> SMEM
//   warps 8-11  epilogue : TMEM acc -> y = q * acc -> 64-byte coalesced stores
//   warps 12-15 T builder: Toeplitz factors T0 / T1 of the next filter group, each
//                          rebuilt as soon as the last MMA reading the old one retires
//                          (tcgen05.commit after that tile's T0 / T1 MMAs)
//   (IMPL)      scan     : per-mode state recurrence over each tile's chunks + the P . S_prev
//                          tf32 MMA (one extra warp; the ids below shift by one)
//   warp 16     feat MMA : one lane issues the featurizer MMAs of each tile, then frees
//                          the stage (tcgen05.commit -> empty barrier)
//   warp 17     MMA      : TMEM alloc (512 cols); one lane issues the 16 main MMAs per tile
//   warp 18     producer : 1-D bulk copies (cp.async.bulk) of raw k/v/q windows into a
//                          4-deep SMEM ring + the per-channel featurizer matrices F
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace hy {
namespace ts {

using bf16 = __nv_bfloat16;
using namespace sm100;

constexpr int LB = 128;            // chunk length (= main MMA M = K)
constexpr int NCH = 32;            // chunks per tile (= main MMA N)
constexpr int TILE_T = NCH * LB;   // time steps per tile
constexpr int HALO = 16;           // featurizer history staged before each window
constexpr int KV_LEN = (NCH + 1) * LB + HALO;  // staged k / v: prev chunk + tile + halo
constexpr int Q_LEN = NCH * LB + HALO;
constexpr int KV_WIN = (NCH + 1) * LB / 8;     // 528 featurizer windows for k / v
constexpr int KV_MB = (KV_WIN + 127) / 128;    // 5 M-blocks
constexpr int Q_WIN = NCH * LB / 8;            // 512 windows for q
constexpr int Q_MB = Q_WIN / 128;              // 4 M-blocks
constexpr int MAX_LHF = 16;
constexpr int NPOLE = 8;  // implicit-filter modes per group (ImplicitFilter poles), zero padded
// Context parallel: history of the raw projections before t = 0 (the predecessor rank's
// last steps) that the first tile of each sequence reads instead of zeros.
constexpr int HIST = LB + HALO;  // 144 = HY_MIXER_HISTORY
static_assert(HIST == 144, "keep in sync with include/hyena_b200.h");

// The warp scheduler favours higher warp ids, so the latency-critical single-lane
// roles (producer, MMA issuers) take the top ids and the bulk CUDA-core roles the bottom.
constexpr int N_CONV_WARPS = 8, N_EPI_WARPS = 4, N_TB_WARPS = 4;
constexpr int W_CONV0 = 0, W_EPI0 = W_CONV0 + N_CONV_WARPS, W_TB0 = W_EPI0 + N_EPI_WARPS;
// Two producer warps alternate tiles (each owns every other stage of the ring).
constexpr int N_PROD_WARPS = 2;
// IMPL adds one warp for the per-mode state scan (21 warps, <= 80 registers); the explicit
// modes keep 20 warps and their 96-register budget
template <bool IMPL>
struct Warps {
  static constexpr int SCAN = IMPL ? W_TB0 + N_TB_WARPS : -1;
  static constexpr int FMMA = W_TB0 + N_TB_WARPS + (IMPL ? 1 : 0), MMA = FMMA + 1, PROD = MMA + 1;
  static constexpr int THREADS = (PROD + N_PROD_WARPS) * 32;
};
constexpr int CONV_THREADS = N_CONV_WARPS * 32, TB_THREADS = N_TB_WARPS * 32;
constexpr uint32_t BAR_CONV = 1, BAR_TB = 2, BAR_EPI = 3;

// Ring depth of the per-tile buffers between converter, main MMA and epilogue
// (U / U_prev / featurized q in SMEM, accumulators in TMEM).
constexpr int NBUF = 3;

// TMEM columns (512 allocated): main accumulators [NBUF] x 32, Toeplitz factors T0 / T1
// (A operand of the main MMA, 128 lanes x 64 columns of packed bf16 pairs each), one
// featurizer buffer (k / v / q outputs; drained to registers right after it lands).
constexpr uint32_t TM_ACC = 0, TM_T0 = NBUF * NCH, TM_T1 = TM_T0 + 64, TM_FEAT = TM_T1 + 64;
constexpr uint32_t TM_K = 0, TM_V = 16 * KV_MB, TM_Q = 32 * KV_MB;
// implicit mode has no T1: its columns hold the mode-input accumulators E[2] x 32
constexpr uint32_t TM_E = TM_T1;
// implicit mode double-buffers its group factors: T0 of odd groups in the last 64 columns
constexpr uint32_t TM_T0B = 448;
static_assert(TM_FEAT + TM_Q + 16 * Q_MB <= TM_T0B && TM_T0B + 64 <= 512, "TMEM budget");

constexpr int round_up(int a, int m) { return (a + m - 1) / m * m; }
constexpr int KV_BYTES = round_up(KV_LEN * 2, 128);
constexpr int Q_BYTES = round_up(Q_LEN * 2, 128);
constexpr int F_BYTES = 512;  // one 16x16 bf16 featurizer matrix (no-swizzle K-major)
template <int KS>
struct Layout {
  static constexpr int STAGES = 4;  // even: stage s is always filled by producer s % 2
  static constexpr int F_SET = 3 * KS * F_BYTES;  // q, k, v featurizer matrices
  static constexpr int STAGE_BYTES = 2 * KV_BYTES + Q_BYTES + F_SET;
  static constexpr int OFF_ST = 0;  // stages first: window over-reads stay inside SMEM
  static constexpr int OFF_U = round_up(OFF_ST + STAGES * STAGE_BYTES, 1024);  // U[NBUF]
  // explicit modes: U holds chunks -1 .. NCH-1 as rows 0 .. NCH (UROWS_X rows, 5 groups of 8), and
  // T1 . U_prev reads it through a descriptor one row (128 B) earlier than T0 . U -- a shifted
  // view, not a copy (the swizzle is a function of the address). It spills into the U_prev
  // region below, which only the implicit mode uses (for its P / Lam double buffers)
  static constexpr int UROWS_X = NCH + 8;
  static constexpr int OFF_UP = OFF_U + NBUF * NCH * LB * 2;   // IMPL: P / Lam buffers
  static_assert(NBUF * UROWS_X * LB * 2 <= 2 * NBUF * NCH * LB * 2, "explicit U buffers");
  static constexpr int OFF_FQ = OFF_UP + NBUF * NCH * LB * 2;  // featurized q, bf16 [NBUF]
  static constexpr int OFF_HP = OFF_FQ + NBUF * NCH * LB * 2;  // padded taps, bf16 [512]
  // implicit (LI) mode: P[m][n] = R_n lam_n^(m+1) (tf32 A operand, 128 x 8), per-chunk mode
  // inputs E[chunk][n], carried states S_prev[chunk][n] (tf32 B operand, [NBUF] x 32 x 8)
  static constexpr int OFF_P = OFF_HP + 2048;  // hpad[2]: the explicit modes prebuild the next group
  static constexpr int OFF_E = OFF_P + 128 * NPOLE * 4;
  static constexpr int OFF_S = OFF_E + NCH * NPOLE * 4;
  // implicit mode: Lam[n][t] = lam_n^(127 - t), the bf16 A operand of the mode-input MMA
  // E[n][chunk] = Lam . U (SW128 K-major, 8 rows, two 64-element K atoms; the descriptor's
  // zero group stride lets the M = 128 MMA re-read these rows for every 8-row group)
  static constexpr int OFF_L = round_up(OFF_S + NBUF * NCH * NPOLE * 4, 1024);
  // implicit mode keeps two sets (P, Lam) for group double-buffering in the U_prev region,
  // which it does not use: P[b] at OFF_UP + 4096 b, Lam[b] at OFF_UP + 8192 + 2048 b
  static constexpr int OFF_P2 = OFF_UP, OFF_L2 = OFF_UP + 8192;
  static_assert(OFF_L2 % 1024 == 0 && OFF_L2 + 4096 <= OFF_FQ, "implicit factor buffers");
  static constexpr int OFF_BAR = OFF_L + 2048;
  static constexpr int N_BARS = 2 * STAGES + 8 + 7 * NBUF + 6;
  static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
  static constexpr int SMEM_BYTES = OFF_TMEM + 16 + 1024;  // + slack for 1024-byte alignment
  static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};

struct Params {
  const bf16* q;      // non-fused: gates / input, rows (b*C + c)*L
  const bf16* k;
  const bf16* v;
  const bf16* proj;   // fused: (B, 3C, L) projections [q; k; v]
  bf16* y;
  const float* taps_hat;   // (n_groups, lh)
  const float* decay;      // (n_groups) rate*log2(base), or null
  const float* feat_taps;  // fused: (3, C, lhf), per channel
  const bf16* fpack;       // fused: packed featurizer matrices, (C, 3, KS, 256) bf16, or null
  const bf16* hist;        // fused: (B, 3C, HIST) projections before t = 0, or null (zeros)
  const float* poles;      // implicit: (n_groups, npoles)
  const float* residues;   // implicit: (n_groups, npoles)
  int npoles;
  int B, C, L, lh, gs, lhf;
  int tiles_per_seq, total_tiles;
  int trace;
  // implicit, non-fused only: rows stored as L / seg_len time segments, element (row, t) at
  // row * seg_len + (t / seg_len) * seg_stride + t % seg_len (the rank-major layout of an
  // all-to-all buffer); seg_len = 0: plain rows of L. seg_len is a multiple of TILE_T.
  int seg_len;
  long long seg_stride;
};

// offset of element (row, t) of a q / k / v / y row
__device__ __forceinline__ size_t elem_off(const Params& p, int row, int t) {
  if (p.seg_len == 0) return static_cast<size_t>(row) * p.L + t;
  const int sg = t / p.seg_len;
  return static_cast<size_t>(row) * p.seg_len + static_cast<size_t>(sg) * p.seg_stride + (t - sg * p.seg_len);
}

// Optional timeline trace (debug/tuning): CTA 0 records clock64 per tile and event.
constexpr int TRACE_TILES = 256, TRACE_EV = 24;
__device__ unsigned long long g_trace[TRACE_TILES * TRACE_EV];
// per-CTA start / end (globaltimer, ns) of a traced launch: load balance across SMs
constexpr int TRACE_CTAS = 256;
__device__ unsigned long long g_cta_times[2 * TRACE_CTAS];
__device__ __forceinline__ void trace_cta(const Params& p, int which) {
  if (p.trace && threadIdx.x == 0 && blockIdx.x < TRACE_CTAS) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_cta_times[2 * blockIdx.x + which] = t;
  }
}
__device__ __forceinline__ void trace(const Params& p, int it, int ev) {
  if (p.trace && blockIdx.x == 0 && it < TRACE_TILES) g_trace[it * TRACE_EV + ev] = clock64();
}

// Tiles are ordered (channel, batch, time-tile) with the time tile fastest; each role
// walks its contiguous range with an incremental iterator (one division at start).
struct Tile {
  int c, b, j, t0;
  __device__ __noinline__ void init(int tile, const Params& p) {
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
  // last tile of its channel: the next tile (if any) belongs to channel c + 1
  __device__ __forceinline__ bool last_of_channel(const Params& p) const {
    return j == p.tiles_per_seq - 1 && b == p.B - 1;
  }
};

// window start in row `which` (0 = q, 1 = k, 2 = v) at time t
template <bool FEAT>
__device__ __forceinline__ const bf16* src_ptr(const Params& p, int which, int b, int c, int t) {
  if (FEAT) return p.proj + (static_cast<size_t>(b) * 3 * p.C + which * p.C + c) * p.L + t;
  const bf16* base = which == 0 ? p.q : which == 1 ? p.k : p.v;
  return base + elem_off(p, b * p.C + c, t);
}

__device__ __forceinline__ int4 pack8(const float* in) {
  int4 raw;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(in[2 * i], in[2 * i + 1]);
  return raw;
}

// Swizzled byte offset of the 16-byte unit (row, unit j in 0..15) of a K-major
// SW128 operand with `rows` rows and K = 128 (two 64-element atoms).
__device__ __forceinline__ uint32_t sw128_off(int row, int j, int rows) {
  return (j >> 3) * (rows * 128) + row * 128 + (((j & 7) ^ (row & 7)) << 4);
}

// No-swizzle K-major descriptor with explicit leading / stride byte offsets.
__device__ __forceinline__ uint64_t desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (static_cast<uint64_t>((saddr >> 4) & 0x3FFF)) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(sbo >> 4) << 32) | (static_cast<uint64_t>(1) << 46);
}

// 32 lanes x 8 consecutive fp32 columns.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// KS: K-steps of 16 in the featurizer GEMM (1 for lhf <= 9, 2 for lhf <= 16).
// IMPL: implicit long filter h_t = sum_n R_n lam_n^t (Hyena-LI): the intra-chunk part is the
// T0 MMA over h[0..127]; every longer lag goes through the exact per-mode recurrence
// s_n[t] = lam_n s_n[t-1] + u[t] carried chunk to chunk (E = per-chunk mode inputs,
// S_prev = state entering each chunk) and applied by one tf32 MMA, P . S_prev.
template <bool FEAT, bool GK, bool GQ, int KS, bool IMPL>
__global__ void __launch_bounds__(Warps<IMPL>::THREADS, 1) two_stage_kernel(const Params p) {
  using LY = Layout<KS>;
  constexpr int W_SCAN = Warps<IMPL>::SCAN, W_FMMA = Warps<IMPL>::FMMA, W_MMA = Warps<IMPL>::MMA,
                W_PROD = Warps<IMPL>::PROD;
  constexpr int STAGES = LY::STAGES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // keep the pointer in the shared window (offset arithmetic, not an integer round trip)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + LY::OFF_BAR);
  uint64_t* full = bars;                 // [STAGES] producer -> MMA
  uint64_t* empty = bars + STAGES;       // [STAGES] MMA commit (featurizer done) -> producer
  uint64_t* ffull = bars + 2 * STAGES;   // [1] MMA commit -> converter (featurized in TMEM)
  uint64_t* fempty = ffull + 2;          // [1] converter warps -> MMA (feat TMEM drained)
  uint64_t* tfree = ffull + 4;           // [2] MMA commit: last reader of T0 / T1 done
  uint64_t* tready = ffull + 6;          // [2] T builder -> MMA: T0 / T1 of the next group
  uint64_t* ufull = ffull + 8;           // [NBUF] converter -> MMA
  uint64_t* uempty = ufull + NBUF;       // [NBUF] MMA commit (U / U_prev read) -> converter
  uint64_t* tfull = uempty + NBUF;       // [NBUF] MMA commit -> epilogue
  uint64_t* tempty = tfull + NBUF;       // [NBUF] epilogue warps -> MMA
  uint64_t* qfull = tempty + NBUF;       // [NBUF] converter -> epilogue: featurized q in SMEM
  uint64_t* qempty = qfull + NBUF;       // [NBUF] epilogue warps -> converter
  uint64_t* efull = qempty + NBUF;       // [2] IMPL: MMA commit -> scan warp (E in TMEM)
  uint64_t* eempty = efull + 2;          // [2] IMPL: scan warp -> MMA (E drained)
  // IMPL factor buffers b = 0 / 1: tfree[b] (MMA warp: last T0 . U / Lam . U of buffer b
  // retired), tfreep[b] (scan warp: last P . S_prev of buffer b retired), tready[b]
  uint64_t* tfreep = eempty + 2;         // [2]
  // explicit modes: T0 is double-buffered (tready[b] / tfree[b] per T0 buffer), T1 is single
  uint64_t* t1ready = tfreep + 2;        // [1] T builder -> MMA: T1 of the current group
  uint64_t* t1free = t1ready + 1;        // [1] MMA commit: last T1 . U_prev of a group retired
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + LY::OFF_TMEM);
  bf16* hpad = reinterpret_cast<bf16*>(smem + LY::OFF_HP);  // hpad[i + 128] = h[i], i in [-128, 384)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  trace_cta(p, 0);
  // IMPL carries the recurrence state from tile to tile, so a CTA owns whole sequences
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
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ffull[i], 1);
      mbar_init(&fempty[i], N_CONV_WARPS);
      mbar_init(&tfree[i], 1);
      mbar_init(&tready[i], 1);
    }
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&ufull[i], 1);
      mbar_init(&uempty[i], 1);
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], 1);  // the epilogue's store issuer, once its bulk store has read the buffer
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], N_EPI_WARPS);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&efull[i], 1);
      mbar_init(&eempty[i], 1);
      mbar_init(&tfreep[i], 1);
    }
    mbar_init(t1ready, 1);
    mbar_init(t1free, 1);
    fence_mbar_init();
  }
  if (warp == W_MMA) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp >= W_PROD) {
    // ------------------------------------------------------------ producers
    const int pw = warp - W_PROD;  // tiles it with it % 2 == pw
    int stage_c[STAGES];
#pragma unroll
    for (int s = 0; s < STAGES; ++s) stage_c[s] = -1;
    Tile t;
    t.init(tb, p);
    if (pw == 1 && ntiles > 0) t.next(p);
    for (int it = pw; it < ntiles; it += N_PROD_WARPS, t.next(p), t.next(p)) {
      const int s = it % STAGES;
      if (lane == 0) trace(p, it, 12);
      mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
      if (lane == 0) trace(p, it, 0);
      unsigned char* st = smem + LY::OFF_ST + s * LY::STAGE_BYTES;
      bf16* kbuf = reinterpret_cast<bf16*>(st);
      bf16* vbuf = reinterpret_cast<bf16*>(st + KV_BYTES);
      bf16* qbuf = reinterpret_cast<bf16*>(st + 2 * KV_BYTES);
      bf16* fmat = reinterpret_cast<bf16*>(st + 2 * KV_BYTES + Q_BYTES);  // [3 tensors][KS][256]
      const int kws = t.t0 - LB - HALO, kwe = t.t0 + TILE_T;
      // segmented rows: windows stop at the segment start (the history there is unused
      // in implicit mode, whose earlier steps arrive through the carried states)
      const int lo = p.seg_len ? (t.t0 / p.seg_len) * p.seg_len : 0;
      const int kvs = max(kws, lo), kve = min(kwe, p.L);
      const int qws = t.t0 - HALO, qwe = t.t0 + TILE_T;
      const int qvs = max(qws, lo), qve = min(qwe, p.L);
      bool wrote = false;  // generic-proxy SMEM writes to order before the async proxy
      // first tile with a predecessor's history: the head of the windows comes from hist
      const bool use_hist = FEAT && p.hist != nullptr && t.t0 == 0;
      if (kvs != kws || kve != kwe || qvs != qws || qve != qwe) {
        // zero the parts of the windows outside [0, L) (whole 8-element units)
        const int4 z = make_int4(0, 0, 0, 0);
        for (int i = lane * 8; !use_hist && i < kvs - kws; i += 256) {
          *reinterpret_cast<int4*>(vbuf + i) = z;
          if (GK) *reinterpret_cast<int4*>(kbuf + i) = z;
        }
        for (int i = (kve - kws) + lane * 8; i < KV_LEN; i += 256) {
          *reinterpret_cast<int4*>(vbuf + i) = z;
          if (GK) *reinterpret_cast<int4*>(kbuf + i) = z;
        }
        if (GQ) {
          for (int i = lane * 8; !use_hist && i < qvs - qws; i += 256) *reinterpret_cast<int4*>(qbuf + i) = z;
          for (int i = (qve - qws) + lane * 8; i < Q_LEN; i += 256) *reinterpret_cast<int4*>(qbuf + i) = z;
        }
        wrote = true;
      }
      // featurizer matrices of this tile's channel: copied in from the packed table
      // (FEAT), or the identity built in place once per stage (two_stage API)
      const int want_c = FEAT ? t.c : 0;
      const bool need_f = stage_c[s] != want_c;
      stage_c[s] = want_c;
      if (!FEAT && need_f) {
        // F[n][k] = [8*KS + n - k == 0] (n < 8), no-swizzle K-major element (n, k) of K-step
        // ks at (n%8)*16 + (n/8)*256 + (k%8)*2 + (k/8)*128 bytes
        for (int e = lane; e < 3 * KS * 256; e += 32) {
          const int ks = (e / 256) % KS, n = (e / 16) % 16, kk = e % 16;
          const int off = (n & 7) * 8 + (n >> 3) * 128 + (kk & 7) + (kk >> 3) * 64;
          fmat[(e / (KS * 256)) * KS * 256 + ks * 256 + off] =
              __float2bfloat16_rn((n < 8 && 8 * KS + n == 16 * ks + kk) ? 1.f : 0.f);
        }
        wrote = true;
      }
      if (wrote) fence_proxy_async();
      __syncwarp();
      if (elect_one()) {
        const uint32_t kvb = static_cast<uint32_t>(kve - kvs) * 2, qb = static_cast<uint32_t>(qve - qvs) * 2;
        const uint32_t fb = (FEAT && need_f) ? static_cast<uint32_t>(LY::F_SET) : 0u;
        const uint32_t hb = use_hist ? static_cast<uint32_t>(2 * HIST + HALO) * 2 : 0u;  // k, v 144 + q 16 steps
        mbar_arrive_expect_tx(&full[s], kvb * (GK ? 2 : 1) + (GQ ? qb : 0) + fb + hb);
        if (use_hist) {
          const bf16* hrow = p.hist + (static_cast<size_t>(t.b) * 3 * p.C + t.c) * HIST;  // q row
          const size_t tstride = static_cast<size_t>(p.C) * HIST;                       // q -> k -> v
          bulk_g2s(kbuf, hrow + tstride, HIST * 2, &full[s]);
          bulk_g2s(vbuf, hrow + 2 * tstride, HIST * 2, &full[s]);
          bulk_g2s(qbuf, hrow + (HIST - HALO), HALO * 2, &full[s]);
        }
        bulk_g2s(vbuf + (kvs - kws), src_ptr<FEAT>(p, 2, t.b, t.c, kvs), kvb, &full[s]);
        if (GK) bulk_g2s(kbuf + (kvs - kws), src_ptr<FEAT>(p, 1, t.b, t.c, kvs), kvb, &full[s]);
        if (GQ) bulk_g2s(qbuf + (qvs - qws), src_ptr<FEAT>(p, 0, t.b, t.c, qvs), qb, &full[s]);
        if (fb) bulk_g2s(fmat, p.fpack + static_cast<size_t>(t.c) * (LY::F_SET / 2), fb, &full[s]);
        trace(p, it, 11);
      }
    }
  } else if (warp == W_FMMA) {
    // ------------------------------------------------------------ featurizer MMA issuer
    // (the whole warp walks the loop so operands stay warp-uniform; one lane issues)
    {
      constexpr uint32_t idesc_feat = idesc_bf16_f32<128, 16>();
      for (int it = 0; it < ntiles; ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        if (lane == 0) trace(p, it, 14);
        mbar_wait(&fempty[0], (it & 1) ^ 1);
        if (lane == 0) trace(p, it, 15);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + LY::OFF_ST + s * LY::STAGE_BYTES);
        const uint32_t fm = st + 2 * KV_BYTES + Q_BYTES;
        const uint32_t dfe = tmem_base + TM_FEAT;
        const uint32_t w0 = 2 * (HALO - 8 * KS);  // byte offset of window 0
        // one elected lane issues the whole tile's featurizer MMAs back to back
        if (elect_one()) {
#pragma unroll
          for (int tensor = 0; tensor < 3; ++tensor) {
            if (tensor == 0 && !GQ) continue;
            if (tensor == 1 && !GK) continue;
            const uint32_t buf = tensor == 0 ? st + 2 * KV_BYTES : st + (tensor == 1 ? 0 : KV_BYTES);
            const int nmb = tensor == 0 ? Q_MB : KV_MB;
            const uint32_t dcol = tensor == 0 ? TM_Q : tensor == 1 ? TM_K : TM_V;
#pragma unroll
            for (int b = 0; b < nmb; ++b) {
#pragma unroll
              for (int ks = 0; ks < KS; ++ks) {
                const uint64_t ad = desc_noswz(buf + w0 + b * 2048 + ks * 32, 16, 128);
                const uint64_t bd = desc_noswz(fm + (tensor * KS + ks) * F_BYTES, 128, 256);
                mma_bf16(dfe + dcol + b * 16, ad, bd, idesc_feat, ks > 0 ? 1u : 0u);
              }
            }
          }
          mma_commit(&empty[s]);
          mma_commit(&ffull[0]);
          trace(p, it, 13);
        }
        __syncwarp();
      }
    }
    __syncwarp();
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ main MMA issuer
    constexpr uint32_t idesc_main = idesc_bf16_f32<LB, NCH>();
    const uint32_t t0a = tmem_base + TM_T0, t1a = tmem_base + TM_T1;
    if (IMPL) {
      // per tile j: T0 . U and E = Lam . U (one commit -> scan warp); the inter-chunk term
      // P . S_prev of tile j is issued by the scan warp itself once the states are in SMEM
      // (its efull wait orders it after this tile's T0 . U), keeping this loop short
      const uint32_t la0 = smem_u32(smem + LY::OFF_L2);
      constexpr uint32_t idesc_e = idesc_bf16_f32<64, NCH>();
      int gi = -1, g_prev = -1;
      Tile t;
      t.init(tb, p);
      for (int j = 0; j < ntiles; ++j, t.next(p)) {
        const int u = j % NBUF;
        const uint32_t ph = (j / NBUF) & 1;
        const int g = t.c / p.gs;
        const bool first = g != g_prev;
        const bool last = j + 1 < ntiles && t.last_of_channel(p) && (t.c + 1) / p.gs != g;
        if (first) ++gi;
        g_prev = g;
        mbar_wait(&ufull[u], ph);  // U written and accumulator u drained (converter)
        if (lane == 0) trace(p, j, 16);
        if (lane == 0) trace(p, j, 17);
        if (lane == 0) trace(p, j, 4);
        const int fb = gi & 1;  // this group's factor buffer
        if (first) mbar_wait(&tready[fb], (gi >> 1) & 1);
        if (lane == 0) trace(p, j, 18);
        tc_fence_after();
        const uint32_t d = tmem_base + TM_ACC + u * NCH;
        const uint32_t de = tmem_base + TM_E + (j & 1) * NCH;
        const uint32_t ua = smem_u32(smem + LY::OFF_U + u * NCH * LB * 2);
        const uint32_t ta = tmem_base + (fb ? TM_T0B : TM_T0);
        const uint32_t la = la0 + fb * 2048;
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < LB / 16; ++ks) {
            const uint32_t bo = (ks >> 2) * (NCH * 128) + (ks & 3) * 32;
            mma_bf16_ts(d, ta + ks * 8, desc_sw128(ua + bo), idesc_main, ks > 0 ? 1u : 0u);
          }
#pragma unroll
          for (int ks = 0; ks < LB / 16; ++ks) {
            const uint32_t bo = (ks >> 2) * (NCH * 128) + (ks & 3) * 32;
            // M = 64: the 8 mode rows are re-read through the zero group stride 8 times instead of
            // 16 (half the shared-memory A traffic of an M = 128 MMA); rows 0..7 of D land in TMEM
            // lanes 0..7 either way, where the scan warp reads them
            mma_bf16(de, desc_sw128_sbo(la + (ks >> 2) * 1024 + (ks & 3) * 32, 0), desc_sw128(ua + bo), idesc_e,
                     ks > 0 ? 1u : 0u);
          }
          mma_commit(&efull[j & 1]);
          mma_commit(&uempty[u]);
          if (last) mma_commit(&tfree[fb]);
          trace(p, j, 7);
        }
        __syncwarp();
      }
    } else {
      int gi = -1, g_prev = -1;
      Tile t;
      t.init(tb, p);
      for (int j = 0; j < ntiles; ++j, t.next(p)) {
        const int u = j % NBUF;
        const uint32_t ph = (j / NBUF) & 1;
        const int g = t.c / p.gs;
        const bool first = g != g_prev;
        const bool last = j + 1 < ntiles && t.last_of_channel(p) && (t.c + 1) / p.gs != g;
        if (first) ++gi;
        g_prev = g;
        mbar_wait(&ufull[u], ph);  // U written and accumulator u drained (converter)
        if (lane == 0) trace(p, j, 4);
        const int fb = gi & 1;  // T0 buffer of this group (built one group ahead)
        if (first) mbar_wait(&tready[fb], (gi >> 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem_base + TM_ACC + u * NCH;
        constexpr int UR = LY::UROWS_X;
        const uint32_t ua = smem_u32(smem + LY::OFF_U + u * UR * LB * 2);  // row 0 = chunk -1
        const uint32_t ta = fb ? tmem_base + TM_T0B : t0a;
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < LB / 16; ++ks) {
            const uint32_t bo = (ks >> 2) * (UR * 128) + (ks & 3) * 32;
            mma_bf16_ts(d, ta + ks * 8, desc_sw128(ua + 128 + bo), idesc_main, ks > 0 ? 1u : 0u);
          }
          if (last) mma_commit(&tfree[fb]);
          if (first) {
            mbar_wait(t1ready, gi & 1);
            tc_fence_after();
          }
#pragma unroll
          for (int ks = 0; ks < LB / 16; ++ks) {
            const uint32_t bo = (ks >> 2) * (UR * 128) + (ks & 3) * 32;
            mma_bf16_ts(d, t1a + ks * 8, desc_sw128(ua + bo), idesc_main, 1u);  // rows 0..NCH-1: U_{n-1}
          }
          if (last) mma_commit(t1free);
          mma_commit(&uempty[u]);
          mma_commit(&tfull[u]);
        }
        __syncwarp();
      }
    }
    __syncwarp();
  } else if (warp >= W_CONV0 && warp < W_EPI0) {
    // ------------------------------------------------------------ converters
    const int ctid = threadIdx.x - W_CONV0 * 32;
    const int quarter = warp & 3;                 // TMEM lane quarter this warp may access
    const int half = (warp - W_CONV0) >> 2;       // two warps per quarter split the M-blocks
    const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
    // M-blocks of this warp: k / v blocks half, half+2, half+4; q blocks half, half+2
    constexpr int KVB_PER = (KV_MB + 1) / 2, QB_PER = Q_MB / 2;
    Tile t;
    t.init(tb, p);
    for (int it = 0; it < ntiles; ++it, t.next(p)) {
      const int u = it % NBUF;
      const uint32_t uph = (it / NBUF) & 1;
      // 1) drain the featurized k / v / q of this tile from TMEM into registers and
      //    release the single featurizer buffer for the next tile's MMAs at once
      mbar_wait(&ffull[0], it & 1);
      if (ctid == 0) trace(p, it, 1);
      tc_fence_after();
      const uint32_t tf = tmem_base + lane_addr + TM_FEAT;
      uint32_t rv[KVB_PER][8], rk[KVB_PER][8], rq[QB_PER][8];
#pragma unroll
      for (int i = 0; i < KVB_PER; ++i) {
        const int b = half + 2 * i;
        if (b < KV_MB && b * 128 + quarter * 32 < KV_WIN) {  // warp-uniform
          tmem_ld8(tf + TM_V + b * 16, rv[i]);
          if (GK) tmem_ld8(tf + TM_K + b * 16, rk[i]);
        }
      }
      if (GQ) {
#pragma unroll
        for (int i = 0; i < QB_PER; ++i) tmem_ld8(tf + TM_Q + (half + 2 * i) * 16, rq[i]);
      }
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&fempty[0]);
      // 2) u = k * v -> U / U_prev: window m holds times t0 - 128 + 8m .. +7, i.e. chunk
      //    m/16 - 1, 16-byte unit m%16
      mbar_wait(&uempty[u], uph ^ 1);
      if (ctid == 0) trace(p, it, 2);
      unsigned char* ub = smem + LY::OFF_U + u * (IMPL ? NCH : LY::UROWS_X) * LB * 2;
#pragma unroll
      for (int i = 0; i < KVB_PER; ++i) {
        const int b = half + 2 * i;
        const int m = b * 128 + quarter * 32 + lane;
        if (!(b < KV_MB && b * 128 + quarter * 32 < KV_WIN)) continue;  // warp-uniform
        const int n = m / 16 - 1, j = m % 16;
        float uv[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          uv[e] = GK ? __uint_as_float(rv[i][e]) * __uint_as_float(rk[i][e]) : __uint_as_float(rv[i][e]);
        if (m < KV_WIN) {
          const int4 packed = pack8(uv);
          if (IMPL) {
            if (n >= 0) *reinterpret_cast<int4*>(ub + sw128_off(n, j, NCH)) = packed;
          } else {  // chunk n at row n + 1 (row 0 = the chunk before the tile)
            *reinterpret_cast<int4*>(ub + sw128_off(n + 1, j, LY::UROWS_X)) = packed;
          }
        }
      }
      fence_proxy_async();
      named_bar_sync(BAR_CONV, CONV_THREADS);
      // ufull also certifies that the accumulator buffer u is free (the epilogue drained
      // tile it - NBUF): the MMA warp, the pipeline's bottleneck, then waits on one barrier
      if (ctid == 0) {
        mbar_wait(&tempty[u], uph ^ 1);
        if (IMPL) mbar_wait(&eempty[it & 1], ((it >> 1) & 1) ^ 1);  // E buffer drained by the scan
        mbar_arrive(&ufull[u]);
      }
      // 3) featurized q -> SMEM for the epilogue (times t0 + 8m .. +7)
      if (GQ) {
        mbar_wait(&qempty[u], uph ^ 1);
        bf16* fq = reinterpret_cast<bf16*>(smem + LY::OFF_FQ + u * NCH * LB * 2);
#pragma unroll
        for (int i = 0; i < QB_PER; ++i) {
          float o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = __uint_as_float(rq[i][e]);
          const int m = (half + 2 * i) * 128 + quarter * 32 + lane;
          *reinterpret_cast<int4*>(fq + 8 * m) = pack8(o);
        }
        named_bar_sync(BAR_CONV, CONV_THREADS);
        if (ctid == 0) mbar_arrive(&qfull[u]);
      }
      if (ctid == 0) trace(p, it, 3);
    }
  } else if (warp >= W_EPI0 && warp < W_TB0) {
    // ------------------------------------------------------------ epilogue
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int tout = quarter * 32 + lane;
    const int etid = threadIdx.x - W_EPI0 * 32;
    // y = q * acc goes into the tile's featurized-q buffer in place (each thread overwrites only
    // the elements it read), then ONE 1-D bulk store writes the tile's contiguous y segment (the
    // tile is 4096 consecutive steps of one row): one instruction instead of 32 2-byte stores per
    // thread. The buffer returns to the converters (qempty) once a later store wait has seen the
    // bulk store read it, one tile deferred so the issuer never stalls on its own store.
    int prev_a = -1;
    Tile t;
    t.init(tb, p);
    for (int it = 0; it < ntiles; ++it, t.next(p)) {
      const int a = it % NBUF;
      const uint32_t aph = (it / NBUF) & 1;
      mbar_wait(&tfull[a], aph);
      if (quarter == 0 && lane == 0) trace(p, it, 5);
      tc_fence_after();
      float acc[NCH];
      tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + TM_ACC + a * NCH, acc);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
      if (GQ) mbar_wait(&qfull[a], aph);
      bf16* stg = reinterpret_cast<bf16*>(smem + LY::OFF_FQ + a * NCH * LB * 2);
      bf16* yrow = p.y + elem_off(p, t.b * p.C + t.c, t.t0);
      const int nt = min(TILE_T, p.L - t.t0);
#pragma unroll
      for (int n = 0; n < NCH; ++n) {
        const int tt = n * LB + tout;
        float val = acc[n];
        if (GQ) val *= __bfloat162float(stg[tt]);
        stg[tt] = __float2bfloat16_rn(val);
      }
      fence_proxy_async();  // the generic writes above, before the async-proxy bulk read
      named_bar_sync(BAR_EPI, N_EPI_WARPS * 32);
      if (etid == 0) {
        bulk_s2g(yrow, stg, static_cast<uint32_t>(nt) * 2);
        bulk_commit();
        bulk_wait_read<1>();  // every earlier tile's store has read its buffer
        if (GQ && prev_a >= 0) mbar_arrive(&qempty[prev_a]);
      }
      prev_a = a;
      if (quarter == 0 && lane == 0) trace(p, it, 6);
    }
    if (etid == 0) {
      bulk_wait_read<0>();
      if (GQ && prev_a >= 0) mbar_arrive(&qempty[prev_a]);
      bulk_wait<0>();
    }
  } else if (warp == W_SCAN) {
    // ------------------------------------------------------------ IMPL state scan
    // (lane n < NPOLE = mode n): E[n][chunk] from TMEM, then the sequential state
    // recurrence over the tile's chunks; the state entering chunk c is written as the tf32
    // B operand S_prev[c][n] (element (c, n) at (c%8)*16 + (c/8)*256 + (n%4)*4 + (n/4)*128
    // bytes) and carried to the next tile of the sequence. Then D += P . S_prev (tf32 MMA,
    // issued here: the efull wait orders it after the tile's T0 . U; the epilogue waits on
    // its commit). A warp of its own, so the factor builds never stall it.
    if (IMPL) {
      constexpr uint32_t idesc_tf32 = idesc_tf32_f32<LB, NCH>();
      const uint32_t pa_s = smem_u32(smem + LY::OFF_P2);
      float lam128 = 0.f, carry = 0.f;
      const int g_end = ntiles > 0 ? ((te - 1) / (p.tiles_per_seq * p.B)) / p.gs : -1;
      auto pole = [&](int g) {
        return (lane < NPOLE && lane < p.npoles) ? p.poles[static_cast<size_t>(g) * p.npoles + lane] : 0.f;
      };
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
        const int fb = gi & 1;
        const int eb = j & 1;
        mbar_wait(&efull[eb], (j >> 1) & 1);
        if (lane == 0) trace(p, j, 9);
        tc_fence_after();
        float ev[NCH];
        tmem_ld_32x32b_x32(tmem_base + TM_E + eb * NCH, ev);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&eempty[eb]);
        float* sp = reinterpret_cast<float*>(smem + LY::OFF_S + (j % NBUF) * NCH * NPOLE * 4);
        float st = t.t0 == 0 ? 0.f : carry;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          if (lane < NPOLE) sp[((c & 7) * 16 + (c >> 3) * 256 + (lane & 3) * 4 + (lane >> 2) * 128) / 4] = st;
          st = fmaf(lam128, st, ev[c]);
        }
        carry = st;
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) trace(p, j, 10);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(smem + LY::OFF_S + (j % NBUF) * NCH * NPOLE * 4);
          mma_tf32(tmem_base + TM_ACC + (j % NBUF) * NCH, desc_noswz(pa_s + fb * 4096, 128, 256),
                   desc_noswz(sa, 128, 256), idesc_tf32, 1u);
          if (lst) mma_commit(&tfreep[fb]);
          mma_commit(&tfull[j % NBUF]);
          trace(p, j, 8);
        }
        __syncwarp();
      }
    }
  } else if (warp >= W_TB0 && warp < W_TB0 + N_TB_WARPS) {
    // ------------------------------------------------------------ Toeplitz factor builder
    const int bt = threadIdx.x - W_TB0 * 32;
    constexpr int PER = 512 / TB_THREADS;  // hpad entries per thread
    float pf_h[PER], pf_dec = 0.f;
    float pf_pole[NPOLE], pf_res[NPOLE];  // IMPL: the group's modes
    // raw loads of a group's taps; the decay is applied at use so the loads stay in flight
    auto prefetch = [&](int g) {
      if (IMPL) {
#pragma unroll
        for (int n = 0; n < NPOLE; ++n) {
          const bool ok = n < p.npoles;
          pf_pole[n] = ok ? p.poles[static_cast<size_t>(g) * p.npoles + n] : 0.f;
          pf_res[n] = ok ? p.residues[static_cast<size_t>(g) * p.npoles + n] : 0.f;
        }
        return;
      }
      pf_dec = p.decay ? p.decay[g] : 0.f;
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int tt = bt + r * TB_THREADS - 128;
        pf_h[r] = (tt >= 0 && tt < p.lh) ? p.taps_hat[static_cast<size_t>(g) * p.lh + tt] : 0.f;
      }
    };
    // one factor into TMEM as the A operand of the main MMA: lane m = output row, column c
    // = packed bf16 pair (T_f[m][2c], T_f[m][2c+1]) = (h[f*128 + m - 2c], h[f*128 + m - 2c - 1])
    const int quarter = warp & 3;
    const int mrow = quarter * 32 + lane;
    const uint32_t trow = tmem_base + (static_cast<uint32_t>(quarter * 32) << 16);
    auto build = [&](int fct, uint32_t tcol, uint64_t* rdy, const bf16* hbuf) {
      // pair c = (hpad[p], hpad[p - 1]) with p = p0 - 2c, from 32-bit words of hpad: for odd
      // p both halves sit in word p >> 1 (swapped); for even p they straddle words p >> 1 and
      // p >> 1 - 1. One byte permute with a per-lane selector covers both, and consecutive
      // columns share a word, so a thread loads 65 words instead of 128 halves.
      const int p0 = 128 + fct * 128 + mrow;
      const uint32_t* hw = reinterpret_cast<const uint32_t*>(hbuf);
      const uint32_t sel = (p0 & 1) ? 0x1032u : 0x7610u;
      uint32_t wa = hw[p0 >> 1];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        uint32_t w[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const int cc = half * 32 + c;
          const uint32_t wb = hw[(p0 >> 1) - cc - 1];
          w[c] = __byte_perm(wa, wb, sel);
          wa = wb;
        }
        tmem_st_32x32b_x32(trow + tcol + half * 32, w);
      }
      tmem_wait_st();
      tc_fence_before();
      named_bar_sync(BAR_TB, TB_THREADS);
      if (bt == 0) mbar_arrive(rdy);
    };
    // IMPL: group gb's factors into buffer gb & 1 (T0 in TMEM, P / Lam in SMEM), built one
    // group ahead from the prefetched modes once group gb - 2's last readers retired:
    // h[t] = sum_n R_n lam_n^t for t < 128 (T0 only; longer lags go through the states),
    // P[m][n] = R_n lam_n^(m+1) as the tf32 A operand (element (m, n) at
    // (m%8)*16 + (m/8)*256 + (n%4)*4 + (n/4)*128 bytes) and Lam[n][t] = lam_n^(127 - t)
    auto build_impl = [&](int gb) {
      const int b = gb & 1;
      if (gb >= 2) {
        mbar_wait(&tfree[b], ((gb - 2) >> 1) & 1);   // T0 / Lam of buffer b: last readers retired
        mbar_wait(&tfreep[b], ((gb - 2) >> 1) & 1);  // P of buffer b
      }
      float hv = 0.f, pm[NPOLE];
      unsigned char* lrow = smem + LY::OFF_L2 + b * 2048 + (bt >> 6) * 1024 + (bt & 7) * 2;
#pragma unroll
      for (int n = 0; n < NPOLE; ++n) {
        // lam^t for integer t = exp2(t log2|lam|) with the sign of lam^t (|lam| <= 1); the
        // relative error (~t ulp of the exponent) is far below the bf16 / tf32 operands'
        const float lam = pf_pole[n], la = log2f(fabsf(lam));
        auto ipow = [&](int e) {
          if (e == 0) return 1.f;
          if (lam == 0.f) return 0.f;
          const float m = exp2f(static_cast<float>(e) * la);
          return (lam < 0.f && (e & 1)) ? -m : m;
        };
        const float lt = ipow(bt);
        hv = fmaf(pf_res[n], lt, hv);
        pm[n] = pf_res[n] * lt * lam;
        const int jj = (bt >> 3) & 7;
        *reinterpret_cast<bf16*>(lrow + n * 128 + ((jj ^ n) << 4)) = __float2bfloat16_rn(ipow(127 - bt));
      }
      hpad[bt] = __float2bfloat16_rn(0.f);
      hpad[128 + bt] = __float2bfloat16_rn(hv);
      hpad[256 + bt] = __float2bfloat16_rn(0.f);
      hpad[384 + bt] = __float2bfloat16_rn(0.f);
      float* pa = reinterpret_cast<float*>(smem + LY::OFF_P2 + b * 4096 + (bt & 7) * 16 + (bt >> 3) * 256);
      *reinterpret_cast<float4*>(pa) = make_float4(pm[0], pm[1], pm[2], pm[3]);
      *reinterpret_cast<float4*>(pa + 32) = make_float4(pm[4], pm[5], pm[6], pm[7]);
      fence_proxy_async();
      named_bar_sync(BAR_TB, TB_THREADS);
      build(0, b ? TM_T0B : TM_T0, &tready[b], hpad);
    };
    int gi = 0, g_prev = -1;
    Tile t;
    t.init(tb, p);
    const int g_end = ntiles > 0 ? ((te - 1) / (p.tiles_per_seq * p.B)) / p.gs : -1;  // last group
    // explicit modes: hpad[b] <- the prefetched group's taps (decay applied), b = group & 1
    auto fill_hpad = [&](bf16* hb) {
#pragma unroll
      for (int r = 0; r < PER; ++r) {
        const int tt = bt + r * TB_THREADS - 128;
        const float h = (tt >= 0 && tt < p.lh) ? pf_h[r] * exp2f(-pf_dec * static_cast<float>(tt)) : 0.f;
        hb[bt + r * TB_THREADS] = __float2bfloat16_rn(h);
      }
      named_bar_sync(BAR_TB, TB_THREADS);
    };
    if (ntiles > 0) {
      const int g0 = t.c / p.gs;
      prefetch(g0);
      if (IMPL) {
        build_impl(0);
        if (g0 < g_end) prefetch(g0 + 1);
      } else {
        // group 0: T0 (buffer 0) and T1; then group 1's T0 into buffer 1 ahead of time
        fill_hpad(hpad);
        build(0, TM_T0, &tready[0], hpad);
        build(1, TM_T1, t1ready, hpad);
        if (g0 < g_end) {
          prefetch(g0 + 1);
          fill_hpad(hpad + 512);
          build(0, TM_T0B, &tready[1], hpad + 512);
          if (g0 + 1 < g_end) prefetch(g0 + 2);
        }
      }
    }
    for (int j = 0; j < ntiles; ++j, t.next(p)) {
      const int g = t.c / p.gs;
      if (g == g_prev) continue;
      g_prev = g;
      if (IMPL) {
        // group gi starts: its factors were built one group ahead; build group gi + 1 into
        // the other buffer
        if (g < g_end) {
          build_impl(gi + 1);
          if (g + 1 < g_end) prefetch(g + 2);
        }
        ++gi;
        continue;
      }
      // group gi starts (gi >= 1; group 0 was built in the prologue): its T0 is already in
      // buffer gi & 1; T1 (single buffer) waits for the previous group's last T1 . U_prev,
      // then group gi + 1's T0 is built into the other buffer (its previous user, group
      // gi - 1, retired long ago) from the taps prefetched during the previous group
      if (gi > 0) {
        mbar_wait(t1free, (gi - 1) & 1);
        build(1, TM_T1, t1ready, hpad + 512 * (gi & 1));
        if (g < g_end) {
          const int nb = (gi + 1) & 1;
          fill_hpad(hpad + 512 * nb);
          mbar_wait(&tfree[nb], ((gi - 1) >> 1) & 1);
          build(0, nb ? TM_T0B : TM_T0, &tready[nb], hpad + 512 * nb);
          if (g + 1 < g_end) prefetch(g + 2);
        }
      }
      ++gi;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == W_MMA) tmem_dealloc<512>(tmem_base);
  trace_cta(p, 1);
}

template <bool FEAT, bool GK, bool GQ, int KS, bool IMPL = false>
static int launch_ks(const Params& p, cudaStream_t st) {
  auto kern = two_stage_kernel<FEAT, GK, GQ, KS, IMPL>;
  constexpr int smem = Layout<KS>::SMEM_BYTES;
  {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int units = IMPL ? p.total_tiles / p.tiles_per_seq : p.total_tiles;  // IMPL: whole sequences
  const int grid = units < sms ? units : sms;
  kern<<<grid, Warps<IMPL>::THREADS, smem, st>>>(p);
  return check_launch("two_stage_kernel");
}

template <bool FEAT, bool GK, bool GQ, bool IMPL = false>
static int launch(Params p, cudaStream_t st) {
  static const int tr = [] { const char* e = getenv("HY_TS_TRACE"); return e ? atoi(e) : 0; }();
  p.trace = tr;
  if (p.lhf <= 9) return launch_ks<FEAT, GK, GQ, 1, IMPL>(p, st);
  return launch_ks<FEAT, GK, GQ, 2, IMPL>(p, st);
}

int check_shapes(int B, int C, int L, int lh, int gs) {
  if (B < 1 || C < 1 || L < 1 || lh < 1 || gs < 1)
    return fail(HY_ERR_INVALID, "sizes must be >= 1 (B=%d C=%d L=%d lh=%d gs=%d)", B, C, L, lh, gs);
  if (C % gs != 0) return fail(HY_ERR_INVALID, "group_size %d does not divide channel count %d", gs, C);
  if (lh > LB + 1)
    return fail(HY_ERR_INELIGIBLE, "filter_len %d needs more than one spill factor at block %d", lh, LB);
  if (L % 8 != 0) return fail(HY_ERR_UNSUPPORTED, "tcgen05 two-stage path needs L %% 8 == 0 (L=%d)", L);
  return HY_OK;
}

}  // namespace ts
}  // namespace hy

using namespace hy;

extern "C" int hy_two_stage_fwd(const void* q, const void* k, const void* v, void* y, const float* taps_hat,
                                const float* decay, int B, int C, int L, int lh, int gs, int dtype,
                                void* stream) {
  if (dtype != HY_BF16) return fail(HY_ERR_UNSUPPORTED, "hy_two_stage_fwd: tcgen05 path is bf16 only");
  if (!v || !y || !taps_hat) return fail(HY_ERR_INVALID, "null pointer argument");
  int s = ts::check_shapes(B, C, L, lh, gs);
  if (s != HY_OK) return s;
  if (!aligned16(v) || !aligned16(y) || (q && !aligned16(q)) || (k && !aligned16(k)))
    return fail(HY_ERR_UNSUPPORTED, "tcgen05 two-stage path needs 16-byte aligned tensors");
  ts::Params p{};
  p.q = static_cast<const ts::bf16*>(q);
  p.k = static_cast<const ts::bf16*>(k);
  p.v = static_cast<const ts::bf16*>(v);
  p.y = static_cast<ts::bf16*>(y);
  p.taps_hat = taps_hat;
  p.decay = decay;
  p.B = B, p.C = C, p.L = L, p.lh = lh, p.gs = gs, p.lhf = 1;
  p.tiles_per_seq = (L + ts::TILE_T - 1) / ts::TILE_T;
  p.total_tiles = p.tiles_per_seq * B * C;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (q && k) return ts::launch<false, true, true>(p, st);
  if (k) return ts::launch<false, true, false>(p, st);
  if (q) return ts::launch<false, false, true>(p, st);
  return ts::launch<false, false, false>(p, st);
}

// Fused MR mixer (bf16): featurizers + gates + two-stage conv in one pass.
int hy::mr_mixer_fwd(const void* proj, void* y, const float* feat_taps, const void* feat_pack,
                     const void* hist, int lhf, const float* taps_hat, const float* decay, int lh, int gs,
                     int B, int C, int L, void* stream) {
  int s = ts::check_shapes(B, C, L, lh, gs);
  if (s != HY_OK) return s;
  if (lhf < 1 || lhf > ts::MAX_LHF) return fail(HY_ERR_UNSUPPORTED, "featurizer length %d > 16", lhf);
  if (!aligned16(proj) || !aligned16(y)) return fail(HY_ERR_UNSUPPORTED, "needs 16-byte aligned tensors");
  if (!feat_pack || !aligned16(feat_pack))
    return fail(HY_ERR_INVALID, "tcgen05 mixer needs the packed featurizer (hy_feat_pack), 16-byte aligned");
  ts::Params p{};
  p.proj = static_cast<const ts::bf16*>(proj);
  p.fpack = static_cast<const ts::bf16*>(feat_pack);
  if (hist && !aligned16(hist)) return fail(HY_ERR_INVALID, "history buffer must be 16-byte aligned");
  p.hist = static_cast<const ts::bf16*>(hist);
  p.y = static_cast<ts::bf16*>(y);
  p.taps_hat = taps_hat;
  p.decay = decay;
  p.feat_taps = feat_taps;
  p.B = B, p.C = C, p.L = L, p.lh = lh, p.gs = gs, p.lhf = lhf;
  p.tiles_per_seq = (L + ts::TILE_T - 1) / ts::TILE_T;
  p.total_tiles = p.tiles_per_seq * B * C;
  return ts::launch<true, true, true>(p, static_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- implicit long filter (Hyena-LI)

// HY_LI_LEGACY=1 keeps the ungated / gated implicit conv on the 32-chunk FEAT-capable kernel
// (the mixer always runs there: its featurizers need the staged raw windows)
static bool legacy_li() {
  static const bool v = [] { const char* e = getenv("HY_LI_LEGACY"); return e && atoi(e) != 0; }();
  return v;
}

static int check_impl(const void* residues, const void* poles, int npoles, int B, int C, int L, int gs) {
  if (!residues || !poles) return fail(HY_ERR_INVALID, "null residues / poles");
  if (npoles < 1 || npoles > ts::NPOLE) return fail(HY_ERR_UNSUPPORTED, "implicit filter needs 1..%d poles", ts::NPOLE);
  return ts::check_shapes(B, C, L, 1, gs);
}

// LI mixer: featurizers + u = k*v + implicit long conv + q gate, bf16 (hyena.py:162-186, LI).
extern "C" HY_API int hy_li_mixer_fwd(const void* proj, void* y, const float* feat_taps, const void* feat_pack,
                                      int lhf, const float* residues, const float* poles, int npoles, int gs,
                                      int B, int C, int L, int dtype, void* stream) {
  if (dtype != HY_BF16) return fail(HY_ERR_UNSUPPORTED, "hy_li_mixer_fwd: tcgen05 path is bf16 only");
  if (!proj || !y || !feat_taps || !feat_pack) return fail(HY_ERR_INVALID, "null pointer argument");
  int s = check_impl(residues, poles, npoles, B, C, L, gs);
  if (s != HY_OK) return s;
  if (lhf < 1 || lhf > ts::MAX_LHF) return fail(HY_ERR_UNSUPPORTED, "featurizer length %d > 16", lhf);
  if (!aligned16(proj) || !aligned16(y) || !aligned16(feat_pack))
    return fail(HY_ERR_UNSUPPORTED, "needs 16-byte aligned tensors");
  // HY_LI_MIXER_KB=1: the staged-row kernel's FEAT mode (CUDA-core featurizers, 64-chunk tiles).
  // Measured slower at C3 (1.51 ms vs 0.81 ms: the converter warps' FIRs set its tile period),
  // so the tensor-core featurizers of this kernel stay the default for the fused mixer.
  static const bool kb_mixer = [] { const char* e = getenv("HY_LI_MIXER_KB"); return e && atoi(e) != 0; }();
  if (kb_mixer && lhf <= 8)
    return mixer_tc_fwd(proj, y, feat_taps, lhf, nullptr, nullptr, 1, residues, poles, npoles, gs, B, C, L, stream);
  ts::Params p{};
  p.proj = static_cast<const ts::bf16*>(proj);
  p.y = static_cast<ts::bf16*>(y);
  p.feat_taps = feat_taps;
  p.fpack = static_cast<const ts::bf16*>(feat_pack);
  p.poles = poles;
  p.residues = residues;
  p.npoles = npoles;
  p.B = B, p.C = C, p.L = L, p.lh = 1, p.gs = gs, p.lhf = lhf;
  p.tiles_per_seq = (L + ts::TILE_T - 1) / ts::TILE_T;
  p.total_tiles = p.tiles_per_seq * B * C;
  return ts::launch<true, true, true, true>(p, static_cast<cudaStream_t>(stream));
}

// Gated implicit long conv y = q * (h conv (k * v)), h_t = sum_n R_n lam_n^t over the whole
// sequence (fft.py:128-145 on an ImplicitFilter, core.py:147-151); q / k may be NULL.
extern "C" HY_API int hy_li_conv_fwd(const void* q, const void* k, const void* v, void* y, const float* residues,
                                     const float* poles, int npoles, int gs, int B, int C, int L, int dtype,
                                     void* stream) {
  if (dtype != HY_BF16) return fail(HY_ERR_UNSUPPORTED, "hy_li_conv_fwd: tcgen05 path is bf16 only");
  if (!v || !y) return fail(HY_ERR_INVALID, "null pointer argument");
  int s = check_impl(residues, poles, npoles, B, C, L, gs);
  if (s != HY_OK) return s;
  if (!aligned16(v) || !aligned16(y) || (q && !aligned16(q)) || (k && !aligned16(k)))
    return fail(HY_ERR_UNSUPPORTED, "needs 16-byte aligned tensors");
  if (!legacy_li())  // 64-chunk tiles, deep staging ring (block_conv_sm100.cu)
    return li_conv_tc_fwd(q, k, v, y, residues, poles, npoles, gs, B, C, L, 0, 0, stream);
  ts::Params p{};
  p.q = static_cast<const ts::bf16*>(q);
  p.k = static_cast<const ts::bf16*>(k);
  p.v = static_cast<const ts::bf16*>(v);
  p.y = static_cast<ts::bf16*>(y);
  p.poles = poles;
  p.residues = residues;
  p.npoles = npoles;
  p.B = B, p.C = C, p.L = L, p.lh = 1, p.gs = gs, p.lhf = 1;
  p.tiles_per_seq = (L + ts::TILE_T - 1) / ts::TILE_T;
  p.total_tiles = p.tiles_per_seq * B * C;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (q && k) return ts::launch<false, true, true, true>(p, st);
  if (k) return ts::launch<false, true, false, true>(p, st);
  if (q) return ts::launch<false, false, true, true>(p, st);
  return ts::launch<false, false, false, true>(p, st);
}

// Ungated implicit long conv of rows stored in time segments (the all-to-all buffer of the
// context-parallel LI layer, cp.py): element (c, t) of v and y at
// c * seg_len + (t / seg_len) * seg_stride + t % seg_len; seg_len a multiple of 4096.
extern "C" HY_API int hy_li_conv_segmented_fwd(const void* v, void* y, const float* residues, const float* poles,
                                               int npoles, int gs, int C, int L, int seg_len,
                                               long long seg_stride, int dtype, void* stream) {
  if (dtype != HY_BF16) return fail(HY_ERR_UNSUPPORTED, "hy_li_conv_segmented_fwd: tcgen05 path is bf16 only");
  if (!v || !y) return fail(HY_ERR_INVALID, "null pointer argument");
  int s = check_impl(residues, poles, npoles, 1, C, L, gs);
  if (s != HY_OK) return s;
  if (seg_len < ts::TILE_T || seg_len % ts::TILE_T != 0 || L % seg_len != 0)
    return fail(HY_ERR_INVALID, "segment length %d must be a multiple of %d dividing L = %d", seg_len, ts::TILE_T,
                L);
  if (seg_stride < static_cast<long long>(C) * seg_len)
    return fail(HY_ERR_INVALID, "segment stride %lld overlaps the %d rows of a segment", seg_stride, C);
  if (!aligned16(v) || !aligned16(y)) return fail(HY_ERR_UNSUPPORTED, "needs 16-byte aligned tensors");
  if (!legacy_li() && seg_len % 8192 == 0)
    return li_conv_tc_fwd(nullptr, nullptr, v, y, residues, poles, npoles, gs, 1, C, L, seg_len, seg_stride, stream);
  ts::Params p{};
  p.v = static_cast<const ts::bf16*>(v);
  p.y = static_cast<ts::bf16*>(y);
  p.poles = poles;
  p.residues = residues;
  p.npoles = npoles;
  p.B = 1, p.C = C, p.L = L, p.lh = 1, p.gs = gs, p.lhf = 1;
  p.seg_len = seg_len;
  p.seg_stride = seg_stride;
  p.tiles_per_seq = L / ts::TILE_T;
  p.total_tiles = p.tiles_per_seq * C;
  return ts::launch<false, false, false, true>(p, static_cast<cudaStream_t>(stream));
}

// Debug: copy the CTA-0 timeline of the last traced two-stage launch (HY_TS_TRACE=1); with
// n >= TRACE_TILES * TRACE_EV + 2 * TRACE_CTAS also every CTA's start / end globaltimer.
extern "C" HY_API int hy_debug_two_stage_trace(unsigned long long* host_out, int n) {
  const int nt = ts::TRACE_TILES * ts::TRACE_EV;
  cudaError_t e = cudaMemcpyFromSymbol(host_out, ts::g_trace, (n < nt ? n : nt) * sizeof(unsigned long long));
  if (e == cudaSuccess && n >= nt + 2 * ts::TRACE_CTAS)
    e = cudaMemcpyFromSymbol(host_out + nt, ts::g_cta_times, 2 * ts::TRACE_CTAS * sizeof(unsigned long long));
  return e == cudaSuccess ? HY_OK : fail(HY_ERR_CUDA, "trace copy: %s", cudaGetErrorString(e));
}

// ---------------------------------------------------------------- featurizer packing
namespace hy {
namespace ts {
// out[c][tensor][ks][256]: F[n][k] = h[8*KS + n - k] for n < 8 in the no-swizzle K-major
// core-matrix order the featurizer MMA reads (element (n,k) at (n%8)*8 + (n/8)*128 +
// (k%8) + (k/8)*64 within a K-step).
__global__ void feat_pack_kernel(const float* __restrict__ taps, int C, int lhf, int KS, bf16* __restrict__ out) {
  const int per = 3 * KS * 256;
  const long long total = static_cast<long long>(C) * per;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i / per), e = static_cast<int>(i % per);
    const int tensor = e / (KS * 256), ks = (e / 256) % KS, r = e % 256;
    // r = (n%8)*8 + (n/8)*128 + (k%8) + (k/8)*64
    const int n = ((r >> 3) & 7) + ((r >> 7) & 1) * 8, kk = (r & 7) + ((r >> 6) & 1) * 8;
    const int tap = 8 * KS + n - (16 * ks + kk);
    float h = 0.f;
    if (n < 8 && tap >= 0 && tap < lhf) h = taps[(static_cast<size_t>(tensor) * C + c) * lhf + tap];
    out[i] = __float2bfloat16_rn(h);
  }
}
}  // namespace ts
}  // namespace hy

extern "C" size_t hy_feat_pack_size(int C, int lhf) {
  const int KS = lhf <= 9 ? 1 : 2;
  return static_cast<size_t>(C) * 3 * KS * 256 * sizeof(ts::bf16);
}

extern "C" int hy_feat_pack(const float* feat_taps, int C, int lhf, void* out, void* stream) {
  if (!feat_taps || !out) return fail(HY_ERR_INVALID, "null pointer argument");
  if (C < 1 || lhf < 1 || lhf > ts::MAX_LHF) return fail(HY_ERR_INVALID, "bad featurizer shape C=%d lhf=%d", C, lhf);
  const int KS = lhf <= 9 ? 1 : 2;
  ts::feat_pack_kernel<<<256, 256, 0, static_cast<cudaStream_t>(stream)>>>(feat_taps, C, lhf, KS,
                                                                           static_cast<ts::bf16*>(out));
  return check_launch("feat_pack_kernel");
}
