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
// TMA-loaded (128-byte swizzle) into a shared-memory ring; one elected thread issues the MMAs
// into one of two 256-column TMEM accumulators while the four epilogue warps drain the other.
// With an even number of 128-row tiles the kernel runs on CTA pairs (cluster of 2,
// tcgen05.mma.cta_group::2, M = 256, N = 256, K = 16, 6-stage ring of 32 KB per CTA); otherwise
// one CTA per 128 x 256 tile (4 stages of 48 KB). Weight rows are permuted so that a 128-row tile
// holds either the q rows of 128 channels or the k rows of 64 channels over the v rows of the
// same 64 (lanes 0..63 / 64..127): each epilogue thread owns one row, runs its FIR along the
// columns in registers, and the v threads hand fv to the k threads through shared memory for
// u = fk fv.
//
// Time order carries the FIR history: a CTA walks its tiles of one M tile in increasing time,
// keeping each row's last 7 raw values in registers. Work units are (M tile, run of time tiles)
// and a unit that starts mid-sequence first accumulates the 64 (128 on CTA pairs) columns before
// it (a "halo" pass) for that history. Units are ordered M-group -> time segment -> M tile, so
// the CTAs running at the same time share a few x tiles and one group's weights in L2.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace hy {
namespace qg {

using namespace sm100;

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int A_BYTES = BM * BK * 2;    // 16 KB: one CTA's 128 weight rows x 64 k
constexpr int BOX_BYTES = BK * 64 * 2;  // one 64 (time) x 64 (k) box of x, 8 KB
constexpr int XS = 36;                  // fv exchange row stride (floats): conflict-free float4
constexpr int XCH_BYTES = 2 * 64 * XS * 4;
constexpr int THREADS = 192;  // warps 0-3 epilogue (TMEM lane quarters), 4 TMA, 5 MMA
constexpr int NTAP = 8;

// NCTA = 1: one CTA per 128 x 256 tile. NCTA = 2: a CTA pair (cluster of 2) per 256 x 256 tile,
// tcgen05.mma.cta_group::2 issued by the even CTA: each CTA stages its own 128 weight rows and
// half of the x columns, and holds its 128 accumulator rows x 256 columns in its own TMEM.
template <int NCTA>
struct Cfg {
  static constexpr int BNL = BN / NCTA;                  // x columns staged per CTA
  static constexpr int B_BYTES = BK * BNL * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = NCTA == 2 ? 6 : 4;
  static constexpr int HN = 64 * NCTA;                   // halo columns (one box per CTA)
  static constexpr int SMEM = STAGES * STAGE_BYTES + XCH_BYTES + 256 + 1024;
  static constexpr uint32_t IDESC_MAIN = idesc_bf16_f32<BM * NCTA, BN>() | (1u << 16);  // B MN-major
  static constexpr uint32_t IDESC_HALO = idesc_bf16_f32<BM * NCTA, HN>() | (1u << 16);
};

struct Params {
  const float* taps;   // (3, D, lhf)
  __nv_bfloat16* fq;   // (B, D, L)
  __nv_bfloat16* u;    // (B, D, L)
  int B, D, L, lhf;
  int n_mt, n_q, n_bt, tpb;  // n_mt: M tiles of BM * NCTA rows
  int S, MG, n_units;
};

// unit -> (M tile, time-tile range [bt0, bt1)); units ordered M-group -> segment -> M tile
__device__ __forceinline__ void unit_decode(const Params& p, int u, int& mt, int& bt0, int& bt1) {
  const int gsz = p.MG * p.S;
  const int g = u / gsz;
  const int rem = u - g * gsz;
  const int gm = min(p.MG, p.n_mt - g * p.MG);
  const int seg = rem / gm;
  mt = g * p.MG + (rem - seg * gm);
  bt0 = static_cast<int>(static_cast<long long>(seg) * p.n_bt / p.S);
  bt1 = static_cast<int>(static_cast<long long>(seg + 1) * p.n_bt / p.S);
}

// Every role walks the same sequence of accumulations ("uses"): per unit an optional halo
// (the HN columns before a mid-sequence start), then one main tile per time tile.
template <int NCTA, typename F>
__device__ __forceinline__ void for_each_use(const Params& p, F&& f) {
  for (int u = blockIdx.x / NCTA; u < p.n_units; u += gridDim.x / NCTA) {
    int mt, bt0, bt1;
    unit_decode(p, u, mt, bt0, bt1);
    for (int bt = bt0; bt < bt1; ++bt) {
      const int b = bt / p.tpb, t0 = (bt - b * p.tpb) * BN;
      if (bt == bt0 && t0 > 0) f(true, mt, b, t0);
      f(false, mt, b, t0);
    }
  }
}

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same variable in cluster CTA `rank`
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int NCTA>
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  if constexpr (NCTA == 1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
  } else {  // completion counted on the even CTA's barrier
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
  }
}

// SW128 MN-major descriptor: 64-element atoms along MN every lbo bytes, 8-row K groups every
// sbo bytes ((T,8,m),(8,k)) : ((1,T,LBO),(8T,SBO)).
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (static_cast<uint64_t>((saddr >> 4) & 0x3FFF)) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}

template <int NCTA>
__device__ __forceinline__ void mma_issue(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  if constexpr (NCTA == 1) {
    mma_bf16(d, adesc, bdesc, idesc, acc);
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  }
}
// arrive on `bar` (same offset) in every CTA of the group once the issued MMAs complete
template <int NCTA>
__device__ __forceinline__ void mma_commit_all(uint64_t* bar) {
  if constexpr (NCTA == 1) {
    mma_commit(bar);
  } else {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
  }
}

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

template <int NCTA>
__global__ void __launch_bounds__(THREADS, 1)
    qkv_feat_gemm_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx, Params p) {
  using C = Cfg<NCTA>;
  extern __shared__ __align__(1024) unsigned char raw_smem[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw_smem) + 1023) & ~uintptr_t(1023));
  float* xch = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + XCH_BYTES);
  uint64_t* full = bars;                       // [STAGES] TMA -> MMA (the even CTA's count)
  uint64_t* empty = bars + C::STAGES;          // [STAGES] MMA -> TMA (every CTA)
  uint64_t* tfull = bars + 2 * C::STAGES;      // [2] MMA -> epilogue (every CTA)
  uint64_t* tfree = bars + 2 * C::STAGES + 2;  // [2] epilogue warps of the group -> MMA
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = NCTA == 1 ? 0 : cta_rank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tfree[i], 4 * NCTA);
    }
    fence_mbar_init();
  }
  if (warp == 4 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tw)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tx)) : "memory");
  }
  if (warp == 5) {
    if constexpr (NCTA == 1) {
      tmem_alloc<512>(tslot);
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (NCTA == 1) __syncthreads();
  else cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int KB = p.D / BK;

  if (warp == 4) {
    // ------------------------------------------------------------ TMA producer (every CTA)
    {
      uint32_t stage = 0, phase = 0;
      for_each_use<NCTA>(p, [&](bool halo, int mt, int b, int t0) {
        const uint32_t bytes = A_BYTES + (halo ? BOX_BYTES : C::B_BYTES);
        const int m = mt * NCTA + rank;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one()) {
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], bytes * NCTA);
            const uint32_t fb = NCTA == 1 ? smem_u32(&full[stage]) : mapa(smem_u32(&full[stage]), 0);
            unsigned char* sa = smem + stage * C::STAGE_BYTES;
            unsigned char* sb = sa + A_BYTES;
            tma_2d<NCTA>(sa, &tw, kb * BK, m * BM, fb);
            const int xrow = b * p.D + kb * BK;
            if (halo) {
              tma_2d<NCTA>(sb, &tx, t0 - C::HN + 64 * rank, xrow, fb);
            } else {
#pragma unroll
              for (int j = 0; j < C::BNL / 64; ++j)
                tma_2d<NCTA>(sb + j * BOX_BYTES, &tx, t0 + C::BNL * rank + 64 * j, xrow, fb);
            }
          }
          __syncwarp();
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      });
    }
  } else if (warp == 5) {
    // ------------------------------------------------------------ MMA issuer (even CTA)
    // The whole warp walks the pipeline (warp-uniform descriptors, no per-lane waterfall); one
    // elected lane issues. Descriptors are stage-0 values plus the stage / k offsets (the 14-bit
    // start-address field cannot carry inside shared memory).
    if (rank == 0) {
      const uint32_t s0 = smem_u32(smem);
      const uint64_t a0 = desc_sw128(s0);
      const uint64_t b0 = desc_mn_sw128(s0 + A_BYTES, BOX_BYTES, 1024);
      uint32_t stage = 0, phase = 0, n = 0;
      for_each_use<NCTA>(p, [&](bool halo, int, int, int) {
        const uint32_t buf = n & 1, aph = (n >> 1) & 1;
        ++n;
        mbar_wait(&tfree[buf], aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * BN;
        const uint32_t idesc = halo ? C::IDESC_HALO : C::IDESC_MAIN;
        for (int kb = 0; kb < KB; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t so = (stage * C::STAGE_BYTES) >> 4;
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk)
              mma_issue<NCTA>(d, a0 + so + 2 * kk, b0 + so + 128 * kk, idesc, (kb | kk) != 0);
            mma_commit_all<NCTA>(&empty[stage]);
          }
          __syncwarp();
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) mma_commit_all<NCTA>(&tfull[buf]);
        __syncwarp();
      });
    }
  } else {
    // ------------------------------------------------------------ epilogue: FIRs, gate product
    const int row = threadIdx.x;  // TMEM lane = accumulator row of this CTA
    const size_t L = p.L;
    const uint32_t tfree0 = NCTA == 1 ? smem_u32(&tfree[0]) : mapa(smem_u32(&tfree[0]), 0);
    float carry[NTAP - 1];
    float tap[NTAP];
    uint32_t n = 0;
    for_each_use<NCTA>(p, [&](bool halo, int mt, int b, int t0) {
      const uint32_t buf = n & 1, aph = (n >> 1) & 1;
      ++n;
      const int m = mt * NCTA + rank;
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
        tmem_ld_32x32b_x32(trow + C::HN - 32, v);  // columns t0-32 .. t0-1
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
          if (ch == BN / 32 - 1) {  // accumulator drained: hand the buffer back to the MMA issuer
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              const uint32_t fb = tfree0 + buf * 8;
              asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(fb) : "memory");
            }
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
      if (halo) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          const uint32_t fb = tfree0 + buf * 8;
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(fb) : "memory");
        }
      }
    });
  }
  __syncwarp();
  tc_fence_before();
  if constexpr (NCTA == 1) {
    __syncthreads();
  } else {
    cluster_sync();
  }
  tc_fence_after();
  if (warp == 5) {
    if constexpr (NCTA == 1) tmem_dealloc<512>(tmem);
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
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
  if ((reinterpret_cast<uintptr_t>(w_perm) | reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(fq) |
       reinterpret_cast<uintptr_t>(u)) & 15)
    return fail(HY_ERR_INVALID, "hy_qkv_feat_gemm needs 16-byte aligned w_perm, x, fq and u");
  qg::Params p{};
  p.taps = feat_taps;
  p.fq = static_cast<__nv_bfloat16*>(fq);
  p.u = static_cast<__nv_bfloat16*>(u);
  p.B = B;
  p.D = D;
  p.L = L;
  p.lhf = lhf;
  p.n_q = D / qg::BM;
  p.tpb = L / qg::BN;
  p.n_bt = B * p.tpb;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // CTA pairs (M = 256 per tile) when the 128-row tiles pair up; HY_QKV_NCTA=1 forces single CTAs
  const char* env = getenv("HY_QKV_NCTA");
  const int ncta = (env && env[0] == '1') || (3 * D / qg::BM) % 2 ? 1 : 2;
  p.n_mt = 3 * D / qg::BM / ncta;
  const int slots = sms / ncta;
  // time segments: the fewest whose units fill the persistent grid evenly (>= 95%), keeping
  // >= 4 tiles per unit so the halo accumulation stays a small fraction
  int S = segments;
  if (S == 0) {
    double best = -1.0;
    for (int s = 1; s <= 64 && (s == 1 || p.n_bt / s >= 4); ++s) {
      const long long units = static_cast<long long>(p.n_mt) * s;
      const long long waves = (units + slots - 1) / slots;
      const double eff = static_cast<double>(units) / static_cast<double>(waves * slots);
      if (eff > best + 1e-9) {
        best = eff;
        S = s;
      }
      if (eff >= 0.95) break;
    }
  }
  if (S > p.n_bt) S = p.n_bt;
  p.S = S;
  p.n_units = p.n_mt * S;
  const int groups = p.n_units < slots ? p.n_units : slots;
  p.MG = groups / S > 0 ? (groups / S < p.n_mt ? groups / S : p.n_mt) : 1;
  CUtensorMap tw, tx;
  if (!qg::make_map(&tw, w_perm, static_cast<uint64_t>(D), static_cast<uint64_t>(3) * D, qg::BK, qg::BM) ||
      !qg::make_map(&tx, x, static_cast<uint64_t>(L), static_cast<uint64_t>(B) * D, 64, qg::BK))
    return fail(HY_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (ncta == 1) {
    auto kern = qg::qkv_feat_gemm_kernel<1>;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), qg::Cfg<1>::SMEM);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    kern<<<groups, qg::THREADS, qg::Cfg<1>::SMEM, st>>>(tw, tx, p);
  } else {
    auto kern = qg::qkv_feat_gemm_kernel<2>;
    cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), qg::Cfg<2>::SMEM);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * groups);
    cfg.blockDim = dim3(qg::THREADS);
    cfg.dynamicSmemBytes = qg::Cfg<2>::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, tw, tx, p);
    if (e != cudaSuccess) return fail(HY_ERR_CUDA, "cudaLaunchKernelEx: %s", cudaGetErrorString(e));
  }
  return check_launch("qkv_feat_gemm_kernel");
}
