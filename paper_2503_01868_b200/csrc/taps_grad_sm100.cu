// Two-stage filter gradient on 5th-gen tensor cores (sm_100a): the reference's two-pass
// algorithm (blockconv.py:246-262) with both passes in one kernel and nothing spilled to HBM.
//
//   pass 1: P0 = sum_n dC_n U_n^T,  P1 = sum_n dC_n U_{n-1}^T      (lb = 128, chunk index n = K)
//   pass 2: dtaps[j] = sum_{i-i'=j} P0[i][i'] + sum_{128+i-i'=j} P1[i][i']
//
// per channel c, summed over the batch and all chunks of the sequence. dC_n / U_n are the
// 128-step chunks of dc (gradient at the conv output) and u (conv input), bf16.
//
// Per CTA (persistent over channels, one CTA per SM):
//   warp 12     producer : 1-D bulk copies of a 64-chunk segment of dc and of u (plus u's
//                          previous chunk) into a 3-deep linear staging ring
//   warps 0-7   transpose: a thread gathers rows r, r+1 of the segment (8 chunks at a time,
//                          one 4-byte load per chunk, conflict-free across the warp) into the SW128
//                          K-major operands A[i][n] = dC_n[i], B0[i'][n] = U_n[i'],
//                          B1[i'][n] = U_{n-1}[i'] (K = 64 chunks, one 128-byte atom per row)
//   warp 13     MMA      : TMEM alloc (512 columns = two (P0, P1) accumulator pairs, so one
//                          channel's epilogue overlaps the next channel's MMAs); one lane
//                          issues 4 K-steps x (A B0^T, A B1^T), M = N = 128, K = 16
//   warps 8-11  epilogue : TMEM rows -> 32 x 32 slabs staged in shared memory -> the slab's
//                          diagonal sums (lane = diagonal, conflict-free) -> per-warp lag
//                          arrays -> summed across the 4 warps -> part[c][j]
// A fixed-order group reduction over channels gives dtaps (G, lh).
#include "common.cuh"
#include "sm100.cuh"

namespace hy {
namespace tg {

using bf16 = __nv_bfloat16;
using namespace sm100;

constexpr int LB = 128;          // chunk (block) length
constexpr int SEG = 64;          // chunks per stage = MMA K per stage
constexpr int THREADS = 448;     // 14 warps
constexpr int N_TR = 8;          // transpose warps 0-7
constexpr int W_EPI = 8, W_PROD = 12, W_MMA = 13;
constexpr int NSTAGE = 3;        // linear staging ring depth

// shared memory layout (bytes)
constexpr int STAGE_DC = SEG * LB * 2;             // 16 KB linear dc segment
constexpr int STAGE_U = (SEG + 1) * LB * 2;        // previous chunk + 64 chunks of u
constexpr int OP = LB * 128;                       // one SW128 operand: 128 rows x 128 B
constexpr int OFF_OPS = 0;                         // [2][A, B0, B1], 1024-aligned
constexpr int OFF_STAGE = OFF_OPS + 2 * 3 * OP;    // [2][dc | u]
constexpr int OFF_SW = OFF_STAGE + NSTAGE * (STAGE_DC + STAGE_U);  // epilogue [4][256] fp32
constexpr int OFF_T = OFF_SW + 4 * 256 * 4;                  // epilogue [4][32][33] fp32 slab tiles
constexpr int OFF_BAR = OFF_T + 4 * 32 * 33 * 4;
constexpr int SMEM = OFF_BAR + 16 * 8 + 16 + 1024;  // + barriers, tmem slot, alignment slack

struct Params {
  const bf16* dc;
  const bf16* u;
  float* part;  // (C, lh)
  int B, C, L, lh;
};

__global__ void __launch_bounds__(THREADS, 1) taps_grad_kernel(Params p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* opready = bars;       // [2] transpose -> MMA (256 arrivals)
  uint64_t* opfree = bars + 2;    // [2] MMA -> transpose (commit)
  uint64_t* accfull = bars + 4;   // [2] MMA -> epilogue (commit)
  uint64_t* accempty = bars + 6;  // [2] epilogue -> MMA (128 arrivals)
  uint64_t* full = bars + 8;      // [NSTAGE] producer -> transpose (tx bytes)
  uint64_t* empty = bars + 8 + NSTAGE;  // [NSTAGE] transpose -> producer (256 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_BAR + 16 * 8);
  float* sw = reinterpret_cast<float*>(smem + OFF_SW);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&opready[i], N_TR * 32);
      mbar_init(&opfree[i], 1);
      mbar_init(&accfull[i], 1);
      mbar_init(&accempty[i], 128);
    }
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], N_TR * 32);
    }
    fence_mbar_init();
  }
  if (warp == W_MMA) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int L = p.L, B = p.B, C = p.C;
  const int nch = (L + LB - 1) / LB;
  const int nseg = (nch + SEG - 1) / SEG;

  if (warp == W_PROD) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      int g = 0;
      for (int c = blockIdx.x; c < C; c += gridDim.x)
        for (int b = 0; b < B; ++b)
          for (int s = 0; s < nseg; ++s, ++g) {
            const int slot = g % NSTAGE;
            mbar_wait(&empty[slot], ((g / NSTAGE) & 1) ^ 1);
            const size_t row = (static_cast<size_t>(b) * C + c) * L;
            const int t0 = s * SEG * LB;
            const int tend = min(L, t0 + SEG * LB);
            unsigned char* st = smem + OFF_STAGE + slot * (STAGE_DC + STAGE_U);
            const uint32_t nb = static_cast<uint32_t>((tend - t0) * 2);
            const int us = t0 > 0 ? t0 - LB : 0;  // u from the previous chunk on
            const uint32_t ub = static_cast<uint32_t>((tend - us) * 2);
            fence_proxy_async();
            mbar_arrive_expect_tx(&full[slot], nb + ub);
            bulk_g2s(st, p.dc + row + t0, nb, &full[slot]);
            bulk_g2s(st + STAGE_DC + (t0 > 0 ? 0 : LB * 2), p.u + row + us, ub, &full[slot]);
          }
    }
  } else if (warp < N_TR) {
    // ---------------------------------------------------------------- transpose
    // thread: rows 2p, 2p+1 (one 4-byte load covers both), unit pair jq (units 2jq, 2jq+1)
    const int pr = threadIdx.x & 63, jq = threadIdx.x >> 6;
    const int r = 2 * pr;
    int g = 0;
    for (int c = blockIdx.x; c < C; c += gridDim.x)
      for (int b = 0; b < B; ++b)
        for (int s = 0; s < nseg; ++s, ++g) {
          const int st_slot = g % NSTAGE, op_slot = g & 1;
          mbar_wait(&full[st_slot], (g / NSTAGE) & 1);
          mbar_wait(&opfree[op_slot], ((g >> 1) & 1) ^ 1);
          const unsigned char* st = smem + OFF_STAGE + st_slot * (STAGE_DC + STAGE_U);
          const uint32_t* dcl = reinterpret_cast<const uint32_t*>(st);                  // bf16 pairs
          const uint32_t* ul = reinterpret_cast<const uint32_t*>(st + STAGE_DC) + LB / 2;  // chunk n at ul[64 n]
          const int n0 = s * SEG;
          const int cnt = min(SEG, nch - n0);
          unsigned char* ops = smem + OFF_OPS + op_slot * 3 * OP;
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int j = 2 * jq + jj;
            uint32_t uv[9], av[8];  // (row r, row r+1) pairs per chunk
#pragma unroll
            for (int e = -1; e < 8; ++e) {
              const int n = 8 * j + e;
              const bool ok = n < cnt && n0 + n >= 0 && (n0 + n) * LB + r < L;
              uv[e + 1] = ok ? ul[n * (LB / 2) + pr] : 0u;
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int n = 8 * j + e;
              const bool ok = n < cnt && (n0 + n) * LB + r < L;
              av[e] = ok ? dcl[n * (LB / 2) + pr] : 0u;
            }
            // row r takes the low halves, row r+1 the high halves
            uint32_t a0[4], a1[4], b00[4], b01[4], b10[4], b11[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              a0[h] = __byte_perm(av[2 * h], av[2 * h + 1], 0x5410);
              a1[h] = __byte_perm(av[2 * h], av[2 * h + 1], 0x7632);
              b00[h] = __byte_perm(uv[2 * h + 1], uv[2 * h + 2], 0x5410);
              b01[h] = __byte_perm(uv[2 * h + 1], uv[2 * h + 2], 0x7632);
              b10[h] = __byte_perm(uv[2 * h], uv[2 * h + 1], 0x5410);
              b11[h] = __byte_perm(uv[2 * h], uv[2 * h + 1], 0x7632);
            }
            const uint32_t o0 = static_cast<uint32_t>(r * 128 + ((j ^ (r & 7)) << 4));
            const uint32_t o1 = static_cast<uint32_t>((r + 1) * 128 + ((j ^ ((r + 1) & 7)) << 4));
            *reinterpret_cast<uint4*>(ops + o0) = make_uint4(a0[0], a0[1], a0[2], a0[3]);
            *reinterpret_cast<uint4*>(ops + o1) = make_uint4(a1[0], a1[1], a1[2], a1[3]);
            *reinterpret_cast<uint4*>(ops + OP + o0) = make_uint4(b00[0], b00[1], b00[2], b00[3]);
            *reinterpret_cast<uint4*>(ops + OP + o1) = make_uint4(b01[0], b01[1], b01[2], b01[3]);
            *reinterpret_cast<uint4*>(ops + 2 * OP + o0) = make_uint4(b10[0], b10[1], b10[2], b10[3]);
            *reinterpret_cast<uint4*>(ops + 2 * OP + o1) = make_uint4(b11[0], b11[1], b11[2], b11[3]);
          }
          mbar_arrive(&empty[st_slot]);
          fence_proxy_async();  // operand writes -> visible to the tensor core
          mbar_arrive(&opready[op_slot]);
        }
  } else if (warp == W_MMA) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32<128, 128>();
    int g = 0, cc = 0;
    for (int c = blockIdx.x; c < C; c += gridDim.x, ++cc) {
      const int ab = cc & 1;
      mbar_wait(&accempty[ab], ((cc >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d0 = tmem_base + ab * 256, d1 = d0 + 128;
      bool first = true;
      for (int b = 0; b < B; ++b)
        for (int s = 0; s < nseg; ++s, ++g) {
          const int slot = g & 1;
          mbar_wait(&opready[slot], (g >> 1) & 1);
          tc_fence_after();
          const uint32_t oa = smem_u32(smem + OFF_OPS + slot * 3 * OP);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < SEG / 16; ++ks) {
              const uint32_t acc = (first && ks == 0) ? 0u : 1u;
              mma_bf16(d0, desc_sw128(oa + ks * 32), desc_sw128(oa + OP + ks * 32), idesc, acc);
              mma_bf16(d1, desc_sw128(oa + ks * 32), desc_sw128(oa + 2 * OP + ks * 32), idesc, acc);
            }
            mma_commit(&opfree[slot]);
            if (b == B - 1 && s == nseg - 1) mma_commit(&accfull[ab]);
          }
          __syncwarp();
          first = false;
        }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 4-7)
    // Each 32 x 32 slab (rows i = 32q + l, columns col0 + e) is staged row-major in a padded
    // shared tile; lane lam then walks the slab's diagonals d = lam and d = lam - 32
    // (l - e = d), one conflict-free load per row, and adds the two sums to the warp's
    // lag array at lag = base + 32q - col0 + d (distinct lags across the lanes).
    const int q = warp - W_EPI;  // TMEM lane quarter
    float* s = sw + q * 256;
    float* T = reinterpret_cast<float*>(smem + OFF_T) + q * 32 * 33;
    int cc = 0;
    for (int c = blockIdx.x; c < C; c += gridDim.x, ++cc) {
      const int ab = cc & 1;
      for (int k = lane; k < 256; k += 32) s[k] = 0.f;
      mbar_wait(&accfull[ab], (cc >> 1) & 1);
      tc_fence_after();
      const uint32_t trow = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + ab * 256;
#pragma unroll 1
      for (int sl = 0; sl < 8; ++sl) {  // 4 slabs of P0, then 4 of P1
        // only lags 0..128 are kept: P0 slabs above the diagonal (lags < 0) and P1 slabs
        // below it (lags > 128) contribute nothing
        if ((sl < 4 && sl > q) || (sl >= 4 && (sl & 3) < q)) continue;
        float v[32];
        tmem_ld_32x32b_x32(trow + sl * 32, v);
        __syncwarp();
#pragma unroll
        for (int e = 0; e < 32; ++e) T[lane * 33 + e] = v[e];
        __syncwarp();
        float a1 = 0.f, a2 = 0.f;  // diagonals d = lane, d = lane - 32
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          const float x = T[r * 33 + ((r - lane) & 31)];
          if (r >= lane) a1 += x;
          else a2 += x;
        }
        const int off = (sl < 4 ? 0 : LB) + 32 * q - (sl & 3) * 32;
        const int l1 = off + lane, l2 = off + lane - 32;
        if (l1 >= 0 && l1 < 256) s[l1] += a1;
        __syncwarp();
        if (l2 >= 0 && l2 < 256) s[l2] += a2;
        __syncwarp();
      }
      tc_fence_before();
      mbar_arrive(&accempty[ab]);
      named_bar_sync(1, 128);
      const float* s0 = sw;
      for (int j = threadIdx.x - W_EPI * 32; j < p.lh; j += 128)
        p.part[static_cast<size_t>(c) * p.lh + j] = s0[j] + s0[256 + j] + s0[512 + j] + s0[768 + j];
      named_bar_sync(1, 128);
    }
  }
  __syncthreads();
  if (warp == W_MMA) tmem_dealloc<512>(tmem_base);
}

// dtaps[g][j] = sum_{c in g} part[c][j] (fixed order)
__global__ void group_reduce_kernel(const float* __restrict__ part, float* __restrict__ dtaps, int lh, int gs) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x, g = blockIdx.y;
  if (j >= lh) return;
  double acc = 0.0;
  for (int c = g * gs; c < (g + 1) * gs; ++c) acc += part[static_cast<size_t>(c) * lh + j];
  dtaps[static_cast<size_t>(g) * lh + j] = static_cast<float>(acc);
}

}  // namespace tg
}  // namespace hy

using namespace hy;

extern "C" size_t hy_two_stage_taps_grad_workspace_size(int C, int lh) {
  return C < 1 || lh < 1 ? 0 : static_cast<size_t>(C) * lh * sizeof(float);
}

extern "C" int hy_two_stage_taps_grad(const void* dc, const void* u, float* dtaps, int B, int C, int L, int lh,
                                      int gs, int dtype, void* ws, size_t ws_bytes, void* stream) {
  if (!dc || !u || !dtaps || !ws) return fail(HY_ERR_INVALID, "null pointer argument");
  if (B < 1 || C < 1 || L < 1 || lh < 1 || gs < 1 || C % gs)
    return fail(HY_ERR_INVALID, "bad sizes (B=%d C=%d L=%d lh=%d gs=%d)", B, C, L, lh, gs);
  if (dtype != HY_BF16) return fail(HY_ERR_UNSUPPORTED, "tcgen05 taps gradient: bf16 only");
  if (lh > tg::LB + 1) return fail(HY_ERR_INELIGIBLE, "filter_len %d needs more than one spill factor", lh);
  if (L % 8 != 0 || !aligned16(dc) || !aligned16(u))
    return fail(HY_ERR_UNSUPPORTED, "tcgen05 taps gradient needs L %% 8 == 0 and 16-byte aligned rows");
  if (ws_bytes < hy_two_stage_taps_grad_workspace_size(C, lh)) return fail(HY_ERR_INVALID, "workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  {
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(tg::taps_grad_kernel), tg::SMEM);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  tg::Params p{static_cast<const tg::bf16*>(dc), static_cast<const tg::bf16*>(u), static_cast<float*>(ws), B, C, L,
               lh};
  tg::taps_grad_kernel<<<C < sms ? C : sms, tg::THREADS, tg::SMEM, st>>>(p);
  int s = check_launch("taps_grad_kernel");
  if (s != HY_OK) return s;
  dim3 grid((lh + 127) / 128, C / gs);
  tg::group_reduce_kernel<<<grid, 128, 0, st>>>(static_cast<const float*>(ws), dtaps, lh, gs);
  return check_launch("group_reduce_kernel");
}
