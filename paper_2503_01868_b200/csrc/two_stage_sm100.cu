// Two-stage blocked causal convolution on 5th-gen tensor cores (sm_100a).
//
// Restates blockconv.py:160-220 (two_stage_forward / _two_stage_core) and, in
// the fused form, hyena.py:162-186 (featurizers + gates) for bf16:
//
//     u = k * v                       (k, v optionally featurized in-kernel)
//     Y_n = T0 . U_n + T1 . U_{n-1}   (128-step chunks, T0/T1 = Toeplitz factors)
//     y = q * Y                       (q optionally featurized in-kernel)
//
// Mapping (per channel c, tile = NCH consecutive chunks of one sequence (b, c)):
//   MMA M = 128 output steps within a chunk, N = NCH chunks, K = 128 input steps.
//   A = T0 / T1 (built in SMEM from taps_hat with the decay applied, SW128 K-major),
//   B = U / U_prev (built in SMEM by the converter warps from staged k, v),
//   D = fp32 accumulator in TMEM (double buffered).
//
// Warp roles (448 threads, 1 CTA per SM, persistent over a contiguous tile range):
//   warp 0      producer : 1-D bulk copies (cp.async.bulk, UBLKCP) of the raw k / v / q
//                          windows of a tile into a STAGES-deep SMEM ring
//   warp 1      MMA      : TMEM alloc; one lane issues 16 tcgen05.mma per tile
//   warps 2-9   converter: Toeplitz factors on group change; featurizer FIRs;
//                          u = k*v -> bf16 swizzled operand U and U_prev; featurized q
//   warps 10-13 epilogue : tcgen05.ld accumulator -> y = q * acc -> SMEM -> bulk store
#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"

#include <cstdlib>

namespace hy {
namespace ts {

using bf16 = __nv_bfloat16;
using namespace sm100;

constexpr int LB = 128;            // chunk length (= MMA M = MMA K)
constexpr int NCH = 32;            // chunks per tile (= MMA N)
constexpr int TILE_T = NCH * LB;   // time steps per tile
constexpr int HALO = 16;           // featurizer history staged before each window
constexpr int STAGES = 3;
constexpr int KV_LEN = (NCH + 1) * LB + HALO;  // staged k / v: prev chunk + tile + halo
constexpr int Q_LEN = NCH * LB + HALO;
constexpr int MAX_LHF = 16;

constexpr int N_EPI_WARPS = 4;
constexpr int W_PROD = 0, W_MMA = 1, W_CONV0 = 2;
constexpr int EPI_THREADS = N_EPI_WARPS * 32;
template <int CW>
struct Roles {
  static constexpr int W_EPI0 = W_CONV0 + CW;
  static constexpr int THREADS = (W_EPI0 + N_EPI_WARPS) * 32;
  static constexpr int CONV_THREADS = CW * 32;
};
constexpr uint32_t BAR_CONV = 1, BAR_EPI = 2;

constexpr int round_up(int a, int m) { return (a + m - 1) / m * m; }
constexpr int T_BYTES = LB * LB * 2;           // one factor, bf16
constexpr int U_BYTES = NCH * LB * 2;          // one operand buffer
constexpr int FQ_BYTES = NCH * LB * 4;         // featurized q, fp32
constexpr int Y_BYTES = NCH * LB * 2;
constexpr int KV_BYTES = round_up(KV_LEN * 2, 128);
constexpr int Q_BYTES = round_up(Q_LEN * 2, 128);
constexpr int STAGE_BYTES = 2 * KV_BYTES + Q_BYTES;
constexpr int OFF_T0 = 0;
constexpr int OFF_T1 = OFF_T0 + T_BYTES;
constexpr int OFF_U = OFF_T1 + T_BYTES;        // U[2]
constexpr int OFF_UP = OFF_U + 2 * U_BYTES;    // U_prev[2]
constexpr int OFF_FQ = OFF_UP + 2 * U_BYTES;   // featq[2]
constexpr int OFF_Y = OFF_FQ + 2 * FQ_BYTES;   // ybuf[2]
constexpr int OFF_ST = OFF_Y + 2 * Y_BYTES;    // stage ring
constexpr int OFF_HP = OFF_ST + STAGES * STAGE_BYTES;  // padded taps, bf16 [512]
constexpr int OFF_BAR = OFF_HP + 1024;
constexpr int N_BARS = 2 * STAGES + 8;
constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
constexpr int SMEM_BYTES = OFF_TMEM + 16 + 1024;  // + slack for 1024-byte alignment
static_assert(SMEM_BYTES <= 232448, "shared memory budget");
static_assert((U_BYTES % 1024) == 0 && (OFF_U % 1024) == 0 && (OFF_UP % 1024) == 0, "SW128 alignment");

struct Params {
  const bf16* q;      // non-fused: gates / input, rows (b*C + c)*L
  const bf16* k;
  const bf16* v;
  const bf16* proj;   // fused: (B, 3C, L) projections [q; k; v]
  bf16* y;
  const float* taps_hat;   // (n_groups, lh)
  const float* decay;      // (n_groups) rate*log2(base), or null
  const float* feat_taps;  // fused: (3, C, lhf), per channel
  int B, C, L, lh, gs, lhf;
  int tiles_per_seq, total_tiles;
};

struct Tile {
  int c, b, t0;
};
__device__ __forceinline__ Tile decode(int tile, const Params& p) {
  Tile t;
  const int j = tile % p.tiles_per_seq;
  const int r = tile / p.tiles_per_seq;
  t.b = r % p.B;
  t.c = r / p.B;
  t.t0 = j * TILE_T;
  return t;
}

template <bool FEAT>
__device__ __forceinline__ const bf16* row_ptr(const Params& p, int which, int b, int c) {
  // which: 0 = q, 1 = k, 2 = v
  if (FEAT) return p.proj + (static_cast<size_t>(b) * 3 * p.C + which * p.C + c) * p.L;
  const bf16* base = which == 0 ? p.q : which == 1 ? p.k : p.v;
  return base + (static_cast<size_t>(b) * p.C + c) * p.L;
}

__device__ __forceinline__ void unpack8(int4 raw, float* out) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f = __bfloat1622float2(h[i]);
    out[2 * i] = f.x;
    out[2 * i + 1] = f.y;
  }
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

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

// Unpack two bf16 vectors elementwise into float2 pairs: out[i] = (a[i], b[i]).
__device__ __forceinline__ void unpack8_pair(int4 ra, int4 rb, float2* out) {
  const uint32_t* a = reinterpret_cast<const uint32_t*>(&ra);
  const uint32_t* b = reinterpret_cast<const uint32_t*>(&rb);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    out[2 * i] = make_float2(__uint_as_float(a[i] << 16), __uint_as_float(b[i] << 16));
    out[2 * i + 1] = make_float2(__uint_as_float(a[i] & 0xFFFF0000u), __uint_as_float(b[i] & 0xFFFF0000u));
  }
}

// Two FIRs at once on f32x2 lanes: acc[e] = sum_jj h[jj] * r[16 + e - jj] (r: 24-wide pair window).
template <int LHF>
__device__ __forceinline__ void fir8x2(const float2* r, const float2* h, float2* acc) {
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    float2 a = make_float2(0.f, 0.f);
#pragma unroll
    for (int jj = 0; jj < LHF; ++jj) a = ffma2(h[jj], r[16 + e - jj], a);
    acc[e] = a;
  }
}

// Load a pair window of 24 (a, b) values ending at idx+8 from two staging buffers.
template <int LHF>
__device__ __forceinline__ void load_raw_pair(const bf16* ba, const bf16* bb, int ia, int ib, float2* r) {
  if (LHF > 9)
    unpack8_pair(*reinterpret_cast<const int4*>(ba + ia - 16), *reinterpret_cast<const int4*>(bb + ib - 16), r);
  if (LHF > 1)
    unpack8_pair(*reinterpret_cast<const int4*>(ba + ia - 8), *reinterpret_cast<const int4*>(bb + ib - 8), r + 8);
  unpack8_pair(*reinterpret_cast<const int4*>(ba + ia), *reinterpret_cast<const int4*>(bb + ib), r + 16);
}

template <bool FEAT, bool GK, bool GQ, int LHF, int CW>
__global__ void __launch_bounds__(Roles<CW>::THREADS, 1) two_stage_kernel(const Params p) {
  constexpr int W_EPI0 = Roles<CW>::W_EPI0;
  constexpr int CONV_THREADS = Roles<CW>::CONV_THREADS;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // keep the pointer in the shared window (offset arithmetic, not an integer round trip)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* full = bars;                 // [STAGES] producer -> converter
  uint64_t* empty = bars + STAGES;       // [STAGES] converter -> producer
  uint64_t* ufull = bars + 2 * STAGES;   // [2] converter -> MMA
  uint64_t* uempty = ufull + 2;          // [2] MMA commit + epilogue -> converter
  uint64_t* tfull = ufull + 4;           // [2] MMA commit -> epilogue
  uint64_t* tempty = ufull + 6;          // [2] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_TMEM);
  bf16* hpad = reinterpret_cast<bf16*>(smem + OFF_HP);  // hpad[i + 128] = h[i], i in [-128, 384)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tb = static_cast<int>((static_cast<long long>(blockIdx.x) * p.total_tiles) / gridDim.x);
  const int te = static_cast<int>((static_cast<long long>(blockIdx.x + 1) * p.total_tiles) / gridDim.x);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&ufull[i], 1);
      mbar_init(&uempty[i], 1 + N_EPI_WARPS);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], N_EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == W_MMA) tmem_alloc<2 * NCH>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == W_PROD) {
    // ------------------------------------------------------------ producer
    int it = 0;
    for (int tile = tb; tile < te; ++tile, ++it) {
      const int s = it % STAGES;
      mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
      const Tile t = decode(tile, p);
      bf16* kbuf = reinterpret_cast<bf16*>(smem + OFF_ST + s * STAGE_BYTES);
      bf16* vbuf = kbuf + KV_BYTES / 2;
      bf16* qbuf = vbuf + KV_BYTES / 2;
      const int kws = t.t0 - LB - HALO, kwe = t.t0 + TILE_T;
      const int kvs = max(kws, 0), kve = min(kwe, p.L);
      const int qws = t.t0 - HALO, qwe = t.t0 + TILE_T;
      const int qvs = max(qws, 0), qve = min(qwe, p.L);
      // zero the parts of the windows outside [0, L) (whole 8-element units)
      const int4 z = make_int4(0, 0, 0, 0);
      for (int i = lane * 8; i < kvs - kws; i += 256) {
        *reinterpret_cast<int4*>(vbuf + i) = z;
        if (GK) *reinterpret_cast<int4*>(kbuf + i) = z;
      }
      for (int i = (kve - kws) + lane * 8; i < KV_LEN; i += 256) {
        *reinterpret_cast<int4*>(vbuf + i) = z;
        if (GK) *reinterpret_cast<int4*>(kbuf + i) = z;
      }
      if (GQ) {
        for (int i = lane * 8; i < qvs - qws; i += 256) *reinterpret_cast<int4*>(qbuf + i) = z;
        for (int i = (qve - qws) + lane * 8; i < Q_LEN; i += 256) *reinterpret_cast<int4*>(qbuf + i) = z;
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        const uint32_t kvb = static_cast<uint32_t>(kve - kvs) * 2, qb = static_cast<uint32_t>(qve - qvs) * 2;
        mbar_arrive_expect_tx(&full[s], kvb * (GK ? 2 : 1) + (GQ ? qb : 0));
        bulk_g2s(vbuf + (kvs - kws), row_ptr<FEAT>(p, 2, t.b, t.c) + kvs, kvb, &full[s]);
        if (GK) bulk_g2s(kbuf + (kvs - kws), row_ptr<FEAT>(p, 1, t.b, t.c) + kvs, kvb, &full[s]);
        if (GQ) bulk_g2s(qbuf + (qvs - qws), row_ptr<FEAT>(p, 0, t.b, t.c) + qvs, qb, &full[s]);
      } else {
        mbar_arrive(&full[s]);
      }
    }
  } else if (warp == W_MMA) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32<LB, NCH>();
      const uint32_t t0a = smem_u32(smem + OFF_T0), t1a = smem_u32(smem + OFF_T1);
      int it = 0;
      for (int tile = tb; tile < te; ++tile, ++it) {
        const int u = it & 1;
        const uint32_t ph = (it >> 1) & 1;
        mbar_wait(&ufull[u], ph);
        mbar_wait(&tempty[u], ph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + u * NCH;
        const uint32_t ua = smem_u32(smem + OFF_U + u * U_BYTES);
        const uint32_t upa = smem_u32(smem + OFF_UP + u * U_BYTES);
#pragma unroll
        for (int ks = 0; ks < LB / 16; ++ks) {
          const uint32_t ao = (ks >> 2) * (LB * 128) + (ks & 3) * 32;
          const uint32_t bo = (ks >> 2) * (NCH * 128) + (ks & 3) * 32;
          mma_bf16(d, desc_sw128(t0a + ao), desc_sw128(ua + bo), idesc, ks > 0 ? 1u : 0u);
        }
#pragma unroll
        for (int ks = 0; ks < LB / 16; ++ks) {
          const uint32_t ao = (ks >> 2) * (LB * 128) + (ks & 3) * 32;
          const uint32_t bo = (ks >> 2) * (NCH * 128) + (ks & 3) * 32;
          mma_bf16(d, desc_sw128(t1a + ao), desc_sw128(upa + bo), idesc, 1u);
        }
        mma_commit(&uempty[u]);
        mma_commit(&tfull[u]);
      }
    }
    __syncwarp();
  } else if (warp < W_EPI0) {
    // ------------------------------------------------------------ converters
    const int ctid = threadIdx.x - W_CONV0 * 32;
    float2 hkv[LHF], hqq[LHF];  // (k, v) and (q, q) featurizer taps on f32x2 lanes
#pragma unroll
    for (int i = 0; i < LHF; ++i) hkv[i] = hqq[i] = make_float2(i == 0 ? 1.f : 0.f, i == 0 ? 1.f : 0.f);
    int cur_g = -1, cur_c = -1;
    int it = 0;
    for (int tile = tb; tile < te; ++tile, ++it) {
      const int s = it % STAGES;
      const int u = it & 1;
      const Tile t = decode(tile, p);
      const int g = t.c / p.gs;
      mbar_wait(&full[s], (it / STAGES) & 1);
      mbar_wait(&uempty[u], ((it >> 1) & 1) ^ 1);
      if (g != cur_g) {
        // all MMAs reading the old factors must be done before they are overwritten
        if (it > 0) mbar_wait(&tfull[u ^ 1], ((it - 1) >> 1) & 1);
        for (int i = ctid; i < 512; i += CONV_THREADS) {
          const int tt = i - 128;
          float h = 0.f;
          if (tt >= 0 && tt < p.lh) {
            h = p.taps_hat[static_cast<size_t>(g) * p.lh + tt];
            if (p.decay) h *= exp2f(-p.decay[g] * static_cast<float>(tt));
          }
          hpad[i] = __float2bfloat16_rn(h);
        }
        named_bar_sync(BAR_CONV, CONV_THREADS);
        // T_f[m][k] = h[f*128 + m - k]: unit (f, m, j) holds k = 8j .. 8j+7
        for (int i = ctid; i < 2 * LB * 16; i += CONV_THREADS) {
          const int f = i / (LB * 16), m = (i / 16) % LB, j = i % 16;
          const bf16* src = hpad + 128 + f * 128 + m - 8 * j;
          int4 raw;
          bf16* e = reinterpret_cast<bf16*>(&raw);
#pragma unroll
          for (int q = 0; q < 8; ++q) e[q] = src[-q];
          *reinterpret_cast<int4*>(smem + (f ? OFF_T1 : OFF_T0) + sw128_off(m, j, LB)) = raw;
        }
        cur_g = g;
      }
      if (FEAT && t.c != cur_c) {
#pragma unroll
        for (int i = 0; i < LHF; ++i) {
          const bool ok = i < p.lhf;
          const float hq = ok ? p.feat_taps[(static_cast<size_t>(0) * p.C + t.c) * p.lhf + i] : 0.f;
          const float hk = ok ? p.feat_taps[(static_cast<size_t>(1) * p.C + t.c) * p.lhf + i] : 0.f;
          const float hv = ok ? p.feat_taps[(static_cast<size_t>(2) * p.C + t.c) * p.lhf + i] : 0.f;
          hkv[i] = make_float2(hk, hv);
          hqq[i] = make_float2(hq, hq);
        }
        cur_c = t.c;
      }
      const bf16* kbuf = reinterpret_cast<const bf16*>(smem + OFF_ST + s * STAGE_BYTES);
      const bf16* vbuf = kbuf + KV_BYTES / 2;
      const bf16* qbuf = vbuf + KV_BYTES / 2;
      unsigned char* ub = smem + OFF_U + u * U_BYTES;
      unsigned char* upb = smem + OFF_UP + u * U_BYTES;
      // u = k * v for chunks n = -1 .. NCH-1 (chunk -1 only feeds U_prev row 0)
      for (int i = ctid; i < (NCH + 1) * 16; i += CONV_THREADS) {
        const int n = i / 16 - 1, j = i % 16;
        const int idx = (n + 1) * LB + HALO + 8 * j;
        float uv[8];
        if (FEAT) {
          float2 r[24], acc[8];
          load_raw_pair<LHF>(kbuf, vbuf, idx, idx, r);
          fir8x2<LHF>(r, hkv, acc);
#pragma unroll
          for (int e = 0; e < 8; ++e) uv[e] = acc[e].x * acc[e].y;
        } else {
          unpack8(*reinterpret_cast<const int4*>(vbuf + idx), uv);
          if (GK) {
            float kv[8];
            unpack8(*reinterpret_cast<const int4*>(kbuf + idx), kv);
#pragma unroll
            for (int e = 0; e < 8; ++e) uv[e] *= kv[e];
          }
        }
        const int4 packed = pack8(uv);
        if (n >= 0) *reinterpret_cast<int4*>(ub + sw128_off(n, j, NCH)) = packed;
        if (n + 1 < NCH) *reinterpret_cast<int4*>(upb + sw128_off(n + 1, j, NCH)) = packed;
      }
      if (GQ) {
        float* fq = reinterpret_cast<float*>(smem + OFF_FQ + u * FQ_BYTES);
        constexpr int NQ = NCH * 16, HQ = NQ / 2;  // q units, processed in pairs (i, i + HQ)
        for (int i = ctid; i < HQ; i += CONV_THREADS) {
          // unit i -> time 8i (= chunk n*128 + 8j with i = n*16 + j)
          const int ia = HALO + 8 * i, ib = HALO + 8 * (i + HQ);
          float2 o[8];
          if (FEAT) {
            float2 r[24];
            load_raw_pair<LHF>(qbuf, qbuf, ia, ib, r);
            fir8x2<LHF>(r, hqq, o);
          } else {
            float2 r[8];
            unpack8_pair(*reinterpret_cast<const int4*>(qbuf + ia), *reinterpret_cast<const int4*>(qbuf + ib), r);
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = r[e];
          }
          *reinterpret_cast<float4*>(fq + 8 * i) = make_float4(o[0].x, o[1].x, o[2].x, o[3].x);
          *reinterpret_cast<float4*>(fq + 8 * i + 4) = make_float4(o[4].x, o[5].x, o[6].x, o[7].x);
          *reinterpret_cast<float4*>(fq + 8 * (i + HQ)) = make_float4(o[0].y, o[1].y, o[2].y, o[3].y);
          *reinterpret_cast<float4*>(fq + 8 * (i + HQ) + 4) = make_float4(o[4].y, o[5].y, o[6].y, o[7].y);
        }
      }
      fence_proxy_async();
      named_bar_sync(BAR_CONV, CONV_THREADS);
      if (ctid == 0) {
        mbar_arrive(&ufull[u]);
        mbar_arrive(&empty[s]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int etid = threadIdx.x - W_EPI0 * 32;
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int tout = quarter * 32 + lane;
    int it = 0;
    for (int tile = tb; tile < te; ++tile, ++it) {
      const int a = it & 1;
      const Tile t = decode(tile, p);
      mbar_wait(&tfull[a], (it >> 1) & 1);
      tc_fence_after();
      float acc[NCH];
      tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + a * NCH, acc);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[a]);
      if (etid == 0 && it >= 2) bulk_wait_read<1>();
      named_bar_sync(BAR_EPI, EPI_THREADS);
      bf16* yb = reinterpret_cast<bf16*>(smem + OFF_Y + a * Y_BYTES);
      const float* fq = reinterpret_cast<const float*>(smem + OFF_FQ + a * FQ_BYTES);
#pragma unroll
      for (int n = 0; n < NCH; ++n) {
        float val = acc[n];
        if (GQ) val *= fq[n * LB + tout];
        yb[n * LB + tout] = __float2bfloat16_rn(val);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&uempty[a]);
      fence_proxy_async();
      named_bar_sync(BAR_EPI, EPI_THREADS);
      if (etid == 0) {
        const int nt = min(TILE_T, p.L - t.t0);
        bf16* dst = p.y + (static_cast<size_t>(t.b) * p.C + t.c) * p.L + t.t0;
        bulk_s2g(dst, yb, static_cast<uint32_t>(nt) * 2);
        bulk_commit();
      }
    }
    if (etid == 0) bulk_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == W_MMA) tmem_dealloc<2 * NCH>(tmem_base);
}

template <bool FEAT, bool GK, bool GQ, int LHF, int CW>
static int launch_cw(const Params& p, cudaStream_t st) {
  auto kern = two_stage_kernel<FEAT, GK, GQ, LHF, CW>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    attr_set = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = p.total_tiles < sms ? p.total_tiles : sms;
  kern<<<grid, Roles<CW>::THREADS, SMEM_BYTES, st>>>(p);
  return check_launch("two_stage_kernel");
}

// Converter warp count: 8 (default) or 12 (HY_TS_CONV_WARPS=12), for tuning.
static int conv_warps() {
  static int cw = [] {
    const char* e = getenv("HY_TS_CONV_WARPS");
    return (e && atoi(e) == 12) ? 12 : 8;
  }();
  return cw;
}

template <bool FEAT, bool GK, bool GQ, int LHF>
static int launch(const Params& p, cudaStream_t st) {
  if (conv_warps() == 12) return launch_cw<FEAT, GK, GQ, LHF, 12>(p, st);
  return launch_cw<FEAT, GK, GQ, LHF, 8>(p, st);
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
  if (q && k) return ts::launch<false, true, true, 1>(p, st);
  if (k) return ts::launch<false, true, false, 1>(p, st);
  if (q) return ts::launch<false, false, true, 1>(p, st);
  return ts::launch<false, false, false, 1>(p, st);
}

// Fused MR mixer (bf16): featurizers + gates + two-stage conv in one pass.
int hy::mr_mixer_fwd(const void* proj, void* y, const float* feat_taps, int lhf, const float* taps_hat,
                    const float* decay, int lh, int gs, int B, int C, int L, void* stream) {
  int s = ts::check_shapes(B, C, L, lh, gs);
  if (s != HY_OK) return s;
  if (lhf < 1 || lhf > ts::MAX_LHF) return fail(HY_ERR_UNSUPPORTED, "featurizer length %d > 16", lhf);
  if (!aligned16(proj) || !aligned16(y)) return fail(HY_ERR_UNSUPPORTED, "needs 16-byte aligned tensors");
  ts::Params p{};
  p.proj = static_cast<const ts::bf16*>(proj);
  p.y = static_cast<ts::bf16*>(y);
  p.taps_hat = taps_hat;
  p.decay = decay;
  p.feat_taps = feat_taps;
  p.B = B, p.C = C, p.L = L, p.lh = lh, p.gs = gs, p.lhf = lhf;
  p.tiles_per_seq = (L + ts::TILE_T - 1) / ts::TILE_T;
  p.total_tiles = p.tiles_per_seq * B * C;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (lhf <= 8) return ts::launch<true, true, true, 8>(p, st);
  return ts::launch<true, true, true, 16>(p, st);
}
