// The q/k/v projection GEMM with the featurizers in its epilogue (SURVEY §8(f) rank 2,
// hyena.py:122-126 then hyena.py:184's gate product):
//
//     p = W_qkv^T x_b                      (3D, L) per sequence, fp32 accumulators in TMEM
//     fq = h_q * p_q,  u = (h_k * p_k) (h_v * p_v)      causal FIRs along time, lhf <= 8
//     fq, u (B, D, L) bf16
//
// so the inner conv reads two rows per channel instead of three and the featurizers never see
// rounded projections.
//
// GEMM: A = the permuted weight (3D, D) K-major, B = x (B*D, L) time-major ("MN-major"), both
// TMA-loaded (128-byte swizzle) into a 4-stage ring; one elected thread issues
// tcgen05.mma M = 128, N = 256, K = 16 into one of two 256-column TMEM accumulators while the
// four epilogue warps drain the other. Weight rows are permuted so that an M tile holds either
// the q rows of 128 channels or the k rows of 64 channels over the v rows of the same 64
// (lanes 0..63 / 64..127): each epilogue thread owns one row, runs its FIR along the columns in
// registers, and the v threads hand fv to the k threads through shared memory for u = fk fv.
//
// Time order carries the FIR history: a CTA walks its tiles of one M tile in increasing time,
// keeping each row's last 7 raw values in registers. Work units are (M tile, run of time tiles)
// and a unit that starts mid-sequence first computes the 64 columns before it (an N = 64
// "halo" accumulation) for that history. Units are ordered M-group -> time segment -> M tile,
// so the CTAs running at the same time share a few x tiles and one group's weights in L2.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace hy {
namespace qg {

using namespace sm100;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4, HN = 64;
constexpr int A_BYTES = BM * BK * 2;      // 16 KB
constexpr int BOX_BYTES = BK * 64 * 2;    // one 64 (time) x 64 (k) box, 8 KB
constexpr int B_BYTES = BK * BN * 2;      // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int XS = 36;                    // fv exchange row stride (floats): conflict-free float4
constexpr int XCH_BYTES = 2 * 64 * XS * 4;
constexpr int SMEM = STAGES * STAGE_BYTES + XCH_BYTES + 256 + 1024;
constexpr int THREADS = 192;  // warps 0-3 epilogue (TMEM lane quarters), 4 TMA, 5 MMA
constexpr int NTAP = 8;

struct Params {
  const float* taps;   // (3, D, lhf)
  __nv_bfloat16* fq;   // (B, D, L)
  __nv_bfloat16* u;    // (B, D, L)
  int B, D, L, lhf;
  int n_m, n_q, n_bt, tpb;
  int S, MG, n_units;
};

// unit -> (M tile, time-tile range [bt0, bt1)); units ordered M-group -> segment -> M tile
__device__ __forceinline__ void unit_decode(const Params& p, int u, int& m, int& bt0, int& bt1) {
  const int gsz = p.MG * p.S;
  const int g = u / gsz;
  const int rem = u - g * gsz;
  const int gm = min(p.MG, p.n_m - g * p.MG);
  const int seg = rem / gm;
  m = g * p.MG + (rem - seg * gm);
  bt0 = static_cast<int>(static_cast<long long>(seg) * p.n_bt / p.S);
  bt1 = static_cast<int>(static_cast<long long>(seg + 1) * p.n_bt / p.S);
}

// Every role walks the same sequence of accumulations ("uses"): per unit an optional halo
// (the 64 columns before a mid-sequence start), then one main tile per time tile.
template <typename F>
__device__ __forceinline__ void for_each_use(const Params& p, F&& f) {
  for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {
    int m, bt0, bt1;
    unit_decode(p, u, m, bt0, bt1);
    for (int bt = bt0; bt < bt1; ++bt) {
      const int b = bt / p.tpb, t0 = (bt - b * p.tpb) * BN;
      if (bt == bt0 && t0 > 0) f(true, m, b, t0);
      f(false, m, b, t0);
    }
  }
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// SW128 MN-major descriptor: 64-element atoms along MN every lbo bytes, 8-row K groups every
// sbo bytes ((T,8,m),(8,k)) : ((1,T,LBO),(8T,SBO)).
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (static_cast<uint64_t>((saddr >> 4) & 0x3FFF)) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}

constexpr uint32_t IDESC_MAIN = idesc_bf16_f32<BM, BN>() | (1u << 16);  // B MN-major
constexpr uint32_t IDESC_HALO = idesc_bf16_f32<BM, HN>() | (1u << 16);

__device__ __forceinline__ void store32_bf16(__nv_bfloat16* dst, const float (&f)[32]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const __nv_bfloat162 h2 = __floats2bfloat162_rn(f[8 * q + 2 * e], f[8 * q + 2 * e + 1]);
      w[e] = *reinterpret_cast<const uint32_t*>(&h2);
    }
    *reinterpret_cast<int4*>(dst + 8 * q) = make_int4(w[0], w[1], w[2], w[3]);
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    qkv_feat_gemm_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx, Params p) {
  extern __shared__ __align__(1024) unsigned char raw_smem[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw_smem) + 1023) & ~uintptr_t(1023));
  float* xch = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + XCH_BYTES);
  uint64_t* full = bars;                 // [STAGES] TMA -> MMA
  uint64_t* empty = bars + STAGES;       // [STAGES] MMA -> TMA
  uint64_t* tfull = bars + 2 * STAGES;   // [2] MMA -> epilogue
  uint64_t* tfree = bars + 2 * STAGES + 2;  // [2] epilogue -> MMA
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tfree[i], 128);
    }
    fence_mbar_init();
  }
  if (warp == 4 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tw)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tx)) : "memory");
  }
  if (warp == 5) tmem_alloc<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int KB = p.D / BK;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0;
      for_each_use(p, [&](bool halo, int m, int b, int t0) {
        const uint32_t bytes = A_BYTES + (halo ? BOX_BYTES : B_BYTES);
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], bytes);
          unsigned char* sa = smem + stage * STAGE_BYTES;
          unsigned char* sb = sa + A_BYTES;
          tma_2d(sa, &tw, kb * BK, m * BM, &full[stage]);
          const int xrow = b * p.D + kb * BK;
          if (halo) {
            tma_2d(sb, &tx, t0 - HN, xrow, &full[stage]);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tma_2d(sb + j * BOX_BYTES, &tx, t0 + 64 * j, xrow, &full[stage]);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      });
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      uint32_t stage = 0, phase = 0, n = 0;
      for_each_use(p, [&](bool halo, int, int, int) {
        const uint32_t buf = n & 1, aph = (n >> 1) & 1;
        ++n;
        mbar_wait(&tfree[buf], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * BN;
        const uint32_t idesc = halo ? IDESC_HALO : IDESC_MAIN;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma_bf16(d, desc_sw128(sa + kk * 32), desc_mn_sw128(sb + kk * 2048, BOX_BYTES, 1024), idesc,
                     (kb | kk) != 0);
          mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(&tfull[buf]);
      });
    }
  } else {
    // ------------------------------------------------------------ epilogue: FIRs, gate product
    const int row = threadIdx.x;  // TMEM lane = accumulator row
    const size_t L = p.L;
    float carry[NTAP - 1];
    float tap[NTAP];
    uint32_t n = 0;
    for_each_use(p, [&](bool halo, int m, int b, int t0) {
      const uint32_t buf = n & 1, aph = (n >> 1) & 1;
      ++n;
      const bool qt = m < p.n_q;
      const int j = m - p.n_q;
      // channel and which featurizer this row applies
      const int c = qt ? m * BM + row : j * 64 + (row & 63);
      const int which = qt ? 0 : (row < 64 ? 1 : 2);
      if (!halo) {
        const float* tp = p.taps + (static_cast<size_t>(which) * p.D + c) * p.lhf;
#pragma unroll
        for (int i = 0; i < NTAP; ++i) tap[i] = i < p.lhf ? __ldg(tp + i) : 0.f;
        if (t0 == 0) {
#pragma unroll
          for (int i = 0; i < NTAP - 1; ++i) carry[i] = 0.f;
        }
      }
      mbar_wait(&tfull[buf], aph);
      tc_fence_after();
      const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16) + buf * BN;
      if (halo) {
        float v[32];
        tmem_ld_32x32b_x32(trow + 32, v);  // columns t0-32 .. t0-1
#pragma unroll
        for (int i = 0; i < NTAP - 1; ++i) carry[i] = v[32 - (NTAP - 1) + i];
      } else {
        __nv_bfloat16* dst = (qt ? p.fq : p.u) + (static_cast<size_t>(b) * p.D + c) * L + t0;
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          float w[NTAP - 1 + 32];
          {
            float v[32];
            tmem_ld_32x32b_x32(trow + ch * 32, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) w[NTAP - 1 + i] = v[i];
          }
#pragma unroll
          for (int i = 0; i < NTAP - 1; ++i) w[i] = carry[i];
#pragma unroll
          for (int i = 0; i < NTAP - 1; ++i) carry[i] = w[32 + i];
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < NTAP; ++k) acc = fmaf(tap[k], w[NTAP - 1 + i - k], acc);
            f[i] = acc;
          }
          if (qt) {
            store32_bf16(dst + ch * 32, f);
          } else {
            float* xb = xch + (ch & 1) * 64 * XS + (row & 63) * XS;
            if (row >= 64) {
#pragma unroll
              for (int i = 0; i < 8; ++i)
                *reinterpret_cast<float4*>(xb + 4 * i) = make_float4(f[4 * i], f[4 * i + 1], f[4 * i + 2], f[4 * i + 3]);
            }
            named_bar_sync(1, 128);
            if (row < 64) {
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float4 g = *reinterpret_cast<const float4*>(xb + 4 * i);
                f[4 * i] *= g.x;
                f[4 * i + 1] *= g.y;
                f[4 * i + 2] *= g.z;
                f[4 * i + 3] *= g.w;
              }
              store32_bf16(dst + ch * 32, f);
            }
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tfree[buf]);
    });
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc<512>(tmem);
}

// --------------------------------------------------------------------------- host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 2-D bf16 row-major tensor (outer rows of `inner` elements), 128-byte swizzled boxes
bool make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
              uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace qg
}  // namespace hy

using namespace hy;

extern "C" HY_API int hy_qkv_feat_gemm(const void* w_perm, const void* x, const float* feat_taps, int lhf, void* fq,
                                       void* u, int B, int D, int L, int segments, int dtype, void* stream) {
  if (!w_perm || !x || !feat_taps || !fq || !u) return fail(HY_ERR_INVALID, "null pointer argument");
  if (dtype != HY_BF16) return fail(HY_ERR_UNSUPPORTED, "hy_qkv_feat_gemm: bf16 only");
  if (B < 1 || D < qg::BM || D % qg::BM || L < qg::BN || L % qg::BN)
    return fail(HY_ERR_INVALID, "hy_qkv_feat_gemm needs D %% 128 == 0 and L %% 256 == 0 (D=%d, L=%d)", D, L);
  if (lhf < 1 || lhf > qg::NTAP) return fail(HY_ERR_UNSUPPORTED, "featurizer length %d > %d", lhf, qg::NTAP);
  if (segments < 0) return fail(HY_ERR_INVALID, "segments must be >= 0");
  qg::Params p{};
  p.taps = feat_taps;
  p.fq = static_cast<__nv_bfloat16*>(fq);
  p.u = static_cast<__nv_bfloat16*>(u);
  p.B = B;
  p.D = D;
  p.L = L;
  p.lhf = lhf;
  p.n_q = D / qg::BM;
  p.n_m = 3 * D / qg::BM;
  p.tpb = L / qg::BN;
  p.n_bt = B * p.tpb;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // time segments: the fewest whose units fill the persistent grid evenly (>= 95%), keeping
  // >= 4 tiles per unit so the halo accumulation stays a small fraction
  int S = segments;
  if (S == 0) {
    double best = -1.0;
    for (int s = 1; s <= 64 && (s == 1 || p.n_bt / s >= 4); ++s) {
      const long long units = static_cast<long long>(p.n_m) * s;
      const long long waves = (units + sms - 1) / sms;
      const double eff = static_cast<double>(units) / static_cast<double>(waves * sms);
      if (eff > best + 1e-9) {
        best = eff;
        S = s;
      }
      if (eff >= 0.95) break;
    }
  }
  if (S > p.n_bt) S = p.n_bt;
  p.S = S;
  p.n_units = p.n_m * S;
  const int grid = p.n_units < sms ? p.n_units : sms;
  p.MG = grid / S > 0 ? (grid / S < p.n_m ? grid / S : p.n_m) : 1;
  CUtensorMap tw, tx;
  if (!qg::make_map(&tw, w_perm, static_cast<uint64_t>(D), static_cast<uint64_t>(3) * D, qg::BK, qg::BM) ||
      !qg::make_map(&tx, x, static_cast<uint64_t>(L), static_cast<uint64_t>(B) * D, 64, qg::BK))
    return fail(HY_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(qg::qkv_feat_gemm_kernel), qg::SMEM);
  if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  qg::qkv_feat_gemm_kernel<<<grid, qg::THREADS, qg::SMEM, static_cast<cudaStream_t>(stream)>>>(tw, tx, p);
  return check_launch("qkv_feat_gemm_kernel");
}
