// Shared helpers for the msGeMM sm_100a kernels: error plumbing, element
// types, codebook parameter block.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "msgemm_b200.h"

namespace msg {

// ----------------------------------------------------------------------------
// errors (thread-local message, negative status codes)
// ----------------------------------------------------------------------------
void set_error(const std::string& s);
int fail(int code, const char* fmt, ...);

#define MSG_CUDA_CHECK(expr)                                                   \
  do {                                                                         \
    cudaError_t err__ = (expr);                                                \
    if (err__ != cudaSuccess)                                                  \
      return ::msg::fail(MSG_ERR_CUDA, "%s failed: %s", #expr,                 \
                         cudaGetErrorString(err__));                           \
  } while (0)

#define MSG_LAUNCH_CHECK() MSG_CUDA_CHECK(cudaGetLastError())

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();  // cached multiProcessorCount of the current device
int max_smem_optin();

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Fan-out of Y (msg_gemm_fanout): every Y store of the finishing kernels is
// repeated at the same element offset into up to kMaxFan more buffers -- the
// other ranks' copies of Y, mapped peer memory over NVLink -- so a row-sharded
// call leaves its slice in every rank's Y without a separate all-gather.
constexpr int kMaxFan = 7;
struct YFan {
  void* p[kMaxFan];
  int n;
};
YFan& current_fan();  // thread-local; empty outside msg_gemm_fanout

inline int row_bytes(int64_t k, int width) {
  // packing.py:39-47 bytes_per_row
  if (width == 4) return (int)((k + 1) / 2);
  if (width == 2) return (int)((k + 3) / 4);
  return (int)k;
}

// ----------------------------------------------------------------------------
// codebook parameter block: up to 256 values (width <= 8), passed by value
// ----------------------------------------------------------------------------
struct CodebookParam {
  double v[256];
  int width;
  int n;
};

inline CodebookParam make_codebook(const double* values, int width) {
  CodebookParam cb{};
  cb.width = width;
  cb.n = 1 << width;
  for (int i = 0; i < cb.n; ++i) cb.v[i] = values[i];
  return cb;
}

// ----------------------------------------------------------------------------
// element type traits
// ----------------------------------------------------------------------------
inline int dtype_size(int dt) {
  switch (dt) {
    case MSG_F32: case MSG_I32: return 4;
    case MSG_F16: case MSG_I16: case MSG_BF16: return 2;
    case MSG_F64: case MSG_I64: return 8;
    case MSG_U8: case MSG_I8: return 1;
  }
  return 0;
}
inline bool dtype_is_int(int dt) {
  return dt == MSG_I32 || dt == MSG_I64 || dt == MSG_U8 || dt == MSG_I8 || dt == MSG_I16;
}

// load element i of a typed array as T
template <typename T>
__device__ __forceinline__ T load_as(const void* p, int dt, int64_t i);

template <>
__device__ __forceinline__ double load_as<double>(const void* p, int dt, int64_t i) {
  switch (dt) {
    case MSG_F32: return (double)((const float*)p)[i];
    case MSG_F16: return (double)__half2float(((const __half*)p)[i]);
    case MSG_F64: return ((const double*)p)[i];
    case MSG_I32: return (double)((const int32_t*)p)[i];
    case MSG_I64: return (double)((const int64_t*)p)[i];
    case MSG_U8: return (double)((const uint8_t*)p)[i];
    case MSG_I8: return (double)((const int8_t*)p)[i];
    case MSG_I16: return (double)((const int16_t*)p)[i];
  }
  return 0.0;
}

template <>
__device__ __forceinline__ int64_t load_as<int64_t>(const void* p, int dt, int64_t i) {
  switch (dt) {
    case MSG_I32: return (int64_t)((const int32_t*)p)[i];
    case MSG_I64: return ((const int64_t*)p)[i];
    case MSG_U8: return (int64_t)((const uint8_t*)p)[i];
    case MSG_I8: return (int64_t)((const int8_t*)p)[i];
    case MSG_I16: return (int64_t)((const int16_t*)p)[i];
    case MSG_F32: return (int64_t)((const float*)p)[i];
    case MSG_F64: return (int64_t)((const double*)p)[i];
    case MSG_F16: return (int64_t)__half2float(((const __half*)p)[i]);
  }
  return 0;
}

template <>
__device__ __forceinline__ float load_as<float>(const void* p, int dt, int64_t i) {
  switch (dt) {
    case MSG_F32: return ((const float*)p)[i];
    case MSG_F16: return __half2float(((const __half*)p)[i]);
    default: return (float)load_as<double>(p, dt, i);
  }
}

// store a value held in accumulator type A into a typed array
template <typename A>
__device__ __forceinline__ void store_as(void* p, int dt, int64_t i, A v) {
  switch (dt) {
    case MSG_F32: ((float*)p)[i] = (float)v; break;
    case MSG_F16: ((__half*)p)[i] = __float2half_rn((float)v); break;
    case MSG_F64: ((double*)p)[i] = (double)v; break;
    case MSG_I32: ((int32_t*)p)[i] = (int32_t)(int64_t)v; break;
    case MSG_I64: ((int64_t*)p)[i] = (int64_t)v; break;
    case MSG_I16: ((int16_t*)p)[i] = (int16_t)(int64_t)v; break;
    case MSG_I8: ((int8_t*)p)[i] = (int8_t)(int64_t)v; break;
    case MSG_U8: ((uint8_t*)p)[i] = (uint8_t)(int64_t)v; break;
  }
}

}  // namespace msg

namespace msg {

// ----------------------------------------------------------------------------
// mbarrier + cp.async.bulk (TMA bulk copy) helpers
// ----------------------------------------------------------------------------
// Programmatic dependent launch (PDL): wait for the preceding grid's results
// / let the next grid start its prologue.  No-ops without the launch attribute.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// ----------------------------------------------------------------------------
// debug build (-DMSG_DEBUG_CHECKS, libmsgemm_b200_debug.so; compute-sanitizer
// is not available on the GPU pool): device-side bounds assertions, and
// "race provocation" -- a pseudo-random per-warp delay of up to ~2 us in front
// of every barrier / mbarrier wait / phase switch, so a missing barrier or a
// read-before-write between warps shows up as a wrong or non-repeatable
// result in the debug tests.  Both compile to nothing in the release build.
// ----------------------------------------------------------------------------
#if defined(MSG_DEBUG_CHECKS)
#define MSG_DASSERT(cond)                                                              \
  do {                                                                                 \
    if (!(cond)) {                                                                     \
      printf("MSG_DASSERT failed %s:%d block (%d,%d,%d) thread %d: %s\n", __FILE__,   \
             __LINE__, blockIdx.x, blockIdx.y, blockIdx.z, threadIdx.x, #cond);         \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
__device__ __forceinline__ void debug_jitter() {
  uint32_t h = (uint32_t)clock64() * 2654435761u ^ (threadIdx.x >> 5) * 40503u ^ blockIdx.x * 97u;
  h ^= h >> 13;
  h *= 0x5bd1e995u;
  h ^= h >> 15;
  if ((h & 3) == 0) __nanosleep(h >> 21);   // a quarter of the warps, up to ~2 us
}
#define MSG_JITTER() ::msg::debug_jitter()
#else
#define MSG_DASSERT(cond) do { } while (0)
#define MSG_JITTER() do { } while (0)
#endif

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  MSG_JITTER();
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace msg
