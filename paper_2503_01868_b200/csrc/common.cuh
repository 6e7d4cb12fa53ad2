// Shared helpers for the sm_100a kernels: element traits, vector memory ops,
// error plumbing for the C-ABI.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <map>
#include <set>
#include <mutex>
#include <tuple>
#include <string>

#include "../../include/hyena_b200.h"

namespace hy {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
int fail(int status, const char* fmt, ...);
int check_launch(const char* what);

// ---------------------------------------------------------------- element traits
// T = storage type in HBM, A = arithmetic (accumulation) type.
template <typename T> struct Elem;
template <> struct Elem<float> {
  using A = float;
  static constexpr int VEC = 4;  // elements per 16-byte vector
  __device__ __forceinline__ static float to_a(float x) { return x; }
  __device__ __forceinline__ static float from_a(float x) { return x; }
};
template <> struct Elem<double> {
  using A = double;
  static constexpr int VEC = 2;
  __device__ __forceinline__ static double to_a(double x) { return x; }
  __device__ __forceinline__ static double from_a(double x) { return x; }
};
template <> struct Elem<__nv_bfloat16> {
  using A = float;
  static constexpr int VEC = 8;
  __device__ __forceinline__ static float to_a(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ __forceinline__ static __nv_bfloat16 from_a(float x) { return __float2bfloat16_rn(x); }
};

// 16-byte global load bypassing L1 allocation (streamed once).
__device__ __forceinline__ int4 ld_stream16(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream16(void* p, int4 v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w));
}

// Unpack one 16-byte vector of T into VEC arithmetic values.
template <typename T>
__device__ __forceinline__ void unpack16(int4 raw, typename Elem<T>::A* out) {
  const T* e = reinterpret_cast<const T*>(&raw);
#pragma unroll
  for (int i = 0; i < Elem<T>::VEC; ++i) out[i] = Elem<T>::to_a(e[i]);
}
template <typename T>
__device__ __forceinline__ int4 pack16(const typename Elem<T>::A* in) {
  int4 raw;
  T* e = reinterpret_cast<T*>(&raw);
#pragma unroll
  for (int i = 0; i < Elem<T>::VEC; ++i) e[i] = Elem<T>::from_a(in[i]);
  return raw;
}

// Resident-CTA grid cap (SMs x CTAs per SM) of `kern` at (threads, smem) on the current device,
// queried once per key: the attribute + occupancy queries cost host microseconds per launch.
inline long long resident_cap(const void* kern, int threads, int smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int, int>, long long> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(kern, dev, threads, smem);
  {
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int sms = 148, per_sm = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  const long long cap = static_cast<long long>(sms) * (per_sm > 0 ? per_sm : 1);
  std::lock_guard<std::mutex> g(mu);
  cache[key] = cap;
  return cap;
}

// Opt a kernel into `smem` bytes of dynamic shared memory on the CURRENT device. The
// attribute belongs to each device's context, so the once-only cache is keyed by device.
inline cudaError_t ensure_smem_attr(const void* kern, int smem) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(kern, dev, smem);
  {
    std::lock_guard<std::mutex> g(mu);
    if (done.count(key)) return cudaSuccess;
  }
  const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> g(mu);
    done.insert(key);
  }
  return e;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline size_t elem_size(int dtype) {
  return dtype == HY_F64 ? 8 : dtype == HY_F32 ? 4 : 2;
}

}  // namespace hy
