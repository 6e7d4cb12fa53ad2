// Memory-system microbenchmark for B200 (tuning aid, not product code):
// streaming read bandwidth of 1-D bulk async copies (cp.async.bulk -> mbarrier ring)
// versus plain 128-bit LDG, for several stage sizes / depths / pieces per stage.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/membench.cu -o build/membench
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(d)),
               "l"(s), "r"(n), "r"(su32(b))
               : "memory");
}

// One CTA per SM. Warp 0 lane 0 produces; warp 1 consumes (touches one word, releases).
__global__ void bulk_ring(const char* src, size_t total, int stage_bytes, int stages, int pieces,
                          unsigned long long* sink) {
  extern __shared__ __align__(1024) char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 64;
  char* buf = sm + 1024;
  const size_t nchunks = total / stage_bytes;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    int it = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
      int s = it % stages;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      mbar_expect(&full[s], stage_bytes);
      int pb = stage_bytes / pieces;
      for (int p = 0; p < pieces; ++p)
        bulk_g2s(buf + (size_t)s * stage_bytes + p * pb, src + c * stage_bytes + p * pb, pb, &full[s]);
    }
  } else if (warp == 1) {
    int it = 0;
    unsigned long long acc = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
      int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      acc += buf[(size_t)s * stage_bytes + lane * 4];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345) *sink = acc;
  }
}

__global__ void ldg_stream(const int4* src, size_t n, unsigned long long* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x * 4) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      size_t j = i + (size_t)u * gridDim.x * blockDim.x;
      v[u] = j < n ? __ldcs(src + j) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc.x ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc.x == 0x12345) *sink = acc.x;
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const size_t total = (size_t)3 << 30;
  char* src;
  unsigned long long* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 1, total);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(bulk_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  int cfgs[][3] = {{8192, 3, 1},  {8192, 8, 1},   {8192, 16, 1},  {16384, 4, 1},  {16384, 8, 1},
                   {24576, 3, 3}, {24576, 6, 3},  {32768, 4, 1},  {32768, 6, 1},  {32768, 6, 8},
                   {49152, 4, 1}, {65536, 3, 1},  {65536, 3, 16}, {4096, 32, 1},  {2048, 64, 1}};
  for (auto& c : cfgs) {
    int sb = c[0], st = c[1], pc = c[2];
    size_t smem = 1024 + (size_t)sb * st;
    if (smem > 220 * 1024) continue;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      bulk_ring<<<sms, 64, smem>>>(src, total, sb, st, pc, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    fflush(stdout);
    printf("bulk stage=%6d B x %2d stages, %2d pieces: %7.1f GB/s (in flight/SM <= %d KB)\n", sb, st, pc,
           total / (ms * 1e-3) / 1e9, sb * st / 1024);
  }
  for (int blocks_per_sm : {2, 4, 8}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      ldg_stream<<<sms * blocks_per_sm, 256>>>((const int4*)src, total / 16, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("ldg.128 x4 unroll, %d CTAs/SM x 256 thr: %7.1f GB/s\n", blocks_per_sm, total / (ms * 1e-3) / 1e9);
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
