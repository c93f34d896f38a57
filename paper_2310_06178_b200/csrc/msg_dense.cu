// Dense comparison baseline for small batches: int4 dequantise + FMA on the
// CUDA cores, streaming the reference's own packed layout (no repack).
//
// Spec: naive_gemm(dense(pwm), X) (gemm.py:206-216, packing.py:191-198) for
// int4 / uint4 codebooks and fp16 X, 1 <= b <= 8 -- the GEMV-like shapes
// where the tensor-core kernel (msg_mma.cu) cannot fill its M128 x N tiles
// and the honest dense baseline is a weight-streaming kernel bound by HBM.
//
// One warp per row (rows strided over all warps of the grid).
// Per 1024-wide k chunk each lane loads 16 bytes of each row (32 nibbles,
// k = 32 lane .. 32 lane + 31, one coalesced 512-byte request per warp and
// row), reads the matching x, converts pairs of
// nibbles to fp16 with one LOP3 (magic number 1024 + (u ^ 8)) and one HSUB2,
// and accumulates w * x exactly in fp32 with FHFMA (fp32 += fp16 * fp16: the
// product of an int4 and an fp16 value is exact in fp32).  X is staged once
// per CTA in shared memory in a lane-major order ([chunk][q][column][lane][8
// halves]) so every LDS.128 is conflict-free; positions past k hold zeros, so
// the padding of the last chunk contributes nothing.  The row sums meet in a
// fixed-order warp reduction (deterministic).
#include <algorithm>

#include "msg_common.cuh"

namespace msg {

constexpr int kDvThreads = 256;
constexpr int kDvRows = 1;  // rows per warp task (more rows per warp: fewer warps in flight, measured slower)
constexpr int kDvBatch = 8;  // k chunks per batch (kDvRows x kDvBatch 16-byte loads in flight per lane)

template <int NB>
__device__ __forceinline__ void dv_word(uint32_t wd, const uint4 (&xq)[NB], uint32_t magic,
                                        uint32_t magic_hi, uint32_t sub2, uint32_t sub_hi,
                                        float (&acc)[NB][2]) {
  // nibbles k0..k7 at bits 0..31: pairs (k0,k4) (k2,k6) from the low nibble
  // of each byte (mask 0x000F000F, before / after one shift by 8) and
  // (k1,k5) (k3,k7) from the high nibble (mask 0x00F000F0: fp16 1024 + 16 u,
  // scaled by 1/16 in the HFMA2 that removes the offset)
  uint32_t h[4];
  {
    const uint32_t w8 = wd >> 8;
    uint32_t t0, t1, t2, t3;
    asm("lop3.b32 %0, %1, 0x000F000F, %2, 0x6A;" : "=r"(t0) : "r"(wd), "r"(magic));   // (a & b) ^ c
    asm("lop3.b32 %0, %1, 0x00F000F0, %2, 0x6A;" : "=r"(t1) : "r"(wd), "r"(magic_hi));
    asm("lop3.b32 %0, %1, 0x000F000F, %2, 0x6A;" : "=r"(t2) : "r"(w8), "r"(magic));
    asm("lop3.b32 %0, %1, 0x00F000F0, %2, 0x6A;" : "=r"(t3) : "r"(w8), "r"(magic_hi));
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(h[0]) : "r"(t0), "r"(sub2));
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(h[1]) : "r"(t1), "r"(0x2C002C00u), "r"(sub_hi));  // x / 16 - off
    asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(h[2]) : "r"(t2), "r"(sub2));
    asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(h[3]) : "r"(t3), "r"(0x2C002C00u), "r"(sub_hi));
  }
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const uint32_t xw[4] = {xq[c].x, xq[c].y, xq[c].z, xq[c].w};  // (x0,x1) (x2,x3) (x4,x5) (x6,x7)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      // w(k_s) * x(k_s) and w(k_{s+4}) * x(k_{s+4})
      const uint32_t xl = xw[s >> 1], xh = xw[2 + (s >> 1)];
      if (s & 1)
        asm("{\n\t.reg .b16 wl, wh, al, ah, bl, bh;\n\tmov.b32 {wl, wh}, %2;\n\t"
            "mov.b32 {al, ah}, %3;\n\tmov.b32 {bl, bh}, %4;\n\t"
            "fma.rn.f32.f16 %0, wl, ah, %0;\n\tfma.rn.f32.f16 %1, wh, bh, %1;\n\t}"
            : "+f"(acc[c][0]), "+f"(acc[c][1]) : "r"(h[s]), "r"(xl), "r"(xh));
      else
        asm("{\n\t.reg .b16 wl, wh, al, ah, bl, bh;\n\tmov.b32 {wl, wh}, %2;\n\t"
            "mov.b32 {al, ah}, %3;\n\tmov.b32 {bl, bh}, %4;\n\t"
            "fma.rn.f32.f16 %0, wl, al, %0;\n\tfma.rn.f32.f16 %1, wh, bl, %1;\n\t}"
            : "+f"(acc[c][0]), "+f"(acc[c][1]) : "r"(h[s]), "r"(xl), "r"(xh));
    }
  }
}

template <int NB>
__global__ void __launch_bounds__(kDvThreads) dq_gemv_kernel(const uint8_t* __restrict__ packed,
                                                             int64_t m, int64_t k, int64_t rb,
                                                             const __half* __restrict__ x,
                                                             uint32_t magic, uint32_t magic_hi,
                                                             uint32_t sub2, uint32_t sub_hi,
                                                             void* __restrict__ y,
                                                             int y_dtype) {
  extern __shared__ __align__(16) uint4 xs[];  // [nchunk][4][NB][32]
  const int tid = threadIdx.x, lane = tid & 31;
  const int nchunk = (int)((k + 1023) / 1024);
  // ---- stage X (k, NB) row-major -> lane-major 16-byte records (after the
  // previous kernel's writes are visible: X may be its output).  Thread
  // (chunk, q, lane) reads the 8 k-rows x NB columns it needs as NB
  // 16-byte loads (16 NB contiguous bytes) and deinterleaves the columns.
  griddep_wait();
  griddep_launch_dependents();
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  for (int r = tid; r < nchunk * 4 * 32; r += kDvThreads) {
    const int l = r & 31, q = (r >> 5) & 3, it = r >> 7;
    const int64_t k0 = (int64_t)it * 1024 + 32 * l + 8 * q;
    unsigned short hv[8 * NB];
    if (vec && k0 + 8 <= k) {
#pragma unroll
      for (int v = 0; v < NB; ++v) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(x + k0 * NB) + v);
        const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          hv[8 * v + 2 * e] = (unsigned short)(w4[e] & 0xFFFF);
          hv[8 * v + 2 * e + 1] = (unsigned short)(w4[e] >> 16);
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8 * NB; ++e)
        hv[e] = k0 + e / NB < k ? __half_as_ushort(x[k0 * NB + e]) : (unsigned short)0;
    }
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      uint32_t w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e)
        w[e] = (uint32_t)hv[(2 * e) * NB + c] | ((uint32_t)hv[(2 * e + 1) * NB + c] << 16);
      xs[((it * 4 + q) * NB + c) * 32 + l] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  __syncthreads();
  // ---- rows in groups of kDvRows per warp: each x record read from shared
  // memory feeds kDvRows rows (X traffic per weight byte / kDvRows)
  const int64_t nwarps = (int64_t)gridDim.x * (kDvThreads / 32);
  const int64_t ngroups = (m + kDvRows - 1) / kDvRows;
  for (int64_t grp = (int64_t)blockIdx.x * (kDvThreads / 32) + (tid >> 5); grp < ngroups; grp += nwarps) {
    const int64_t row0 = grp * kDvRows;
    const uint8_t* rp[kDvRows];
    bool rv[kDvRows];
#pragma unroll
    for (int r = 0; r < kDvRows; ++r) {
      rv[r] = row0 + r < m;
      rp[r] = packed + (rv[r] ? row0 + r : row0) * rb + 16 * lane;
    }
    float acc[kDvRows][NB][2];
#pragma unroll
    for (int r = 0; r < kDvRows; ++r)
#pragma unroll
      for (int c = 0; c < NB; ++c) acc[r][c][0] = acc[r][c][1] = 0.f;
    // batches of kDvBatch chunks x kDvRows rows in flight per lane
    for (int it0 = 0; it0 < nchunk; it0 += kDvBatch) {
      uint4 wv[kDvBatch][kDvRows];
#pragma unroll
      for (int j = 0; j < kDvBatch; ++j)
#pragma unroll
        for (int r = 0; r < kDvRows; ++r) {
          const int64_t o = (int64_t)(it0 + j) * 512 + 16 * lane;
          wv[j][r] = (rv[r] && it0 + j < nchunk && o < rb)
                         ? __ldcs(reinterpret_cast<const uint4*>(rp[r] + (it0 + j) * 512))
                         : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
      for (int j = 0; j < kDvBatch; ++j) {
        if (it0 + j >= nchunk) break;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 xq[NB];
#pragma unroll
          for (int c = 0; c < NB; ++c) xq[c] = xs[(((it0 + j) * 4 + q) * NB + c) * 32 + lane];
#pragma unroll
          for (int r = 0; r < kDvRows; ++r) {
            const uint32_t wd = q == 0 ? wv[j][r].x : q == 1 ? wv[j][r].y : q == 2 ? wv[j][r].z : wv[j][r].w;
            dv_word<NB>(wd, xq, magic, magic_hi, sub2, sub_hi, acc[r]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kDvRows; ++r)
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        float v = acc[r][c][0] + acc[r][c][1];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && rv[r]) {
          if (y_dtype == MSG_F16) reinterpret_cast<__half*>(y)[(row0 + r) * NB + c] = __float2half_rn(v);
          else reinterpret_cast<float*>(y)[(row0 + r) * NB + c] = v;
        }
      }
  }
}

template <int NB>
static int launch_dv(const uint8_t* packed, int64_t m, int64_t k, const __half* x, uint32_t magic,
                     uint32_t magic_hi, uint32_t sub2, uint32_t sub_hi, void* y, int y_dtype,
                     cudaStream_t s) {
  const int nchunk = (int)((k + 1023) / 1024);
  const int smem = nchunk * 4 * NB * 32 * 16;
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    MSG_CUDA_CHECK(cudaFuncSetAttribute(dq_gemv_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        max_smem_optin()));
    configured_dev = dev;
  }
  int per_sm = 0;
  MSG_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dq_gemv_kernel<NB>, kDvThreads, smem));
  if (per_sm < 1) return fail(MSG_ERR_UNSUPPORTED, "dense GEMV: k = %lld too large to stage X", (long long)k);
  const int64_t want = ceil_div(ceil_div(m, kDvRows), kDvThreads / 32);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * per_sm));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kDvThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MSG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, dq_gemv_kernel<NB>, packed, m, k, (int64_t)row_bytes(k, 4),
                                    x, magic, magic_hi, sub2, sub_hi, y, y_dtype));
  return MSG_OK;
}

}  // namespace msg

using namespace msg;

extern "C" int msg_dequant_gemv(const uint8_t* packed, int64_t m, int64_t k, const double* values,
                                const void* x, int x_dtype, int64_t b, void* y, int y_dtype,
                                void* stream) {
  if (x_dtype != MSG_F16)
    return fail(MSG_ERR_UNSUPPORTED, "the dense GEMV baseline takes fp16 activations");
  if (b < 1 || b > 8)
    return fail(MSG_ERR_UNSUPPORTED, "the dense GEMV baseline supports 1 <= b <= 8 (got %lld)", (long long)b);
  if (y_dtype != MSG_F32 && y_dtype != MSG_F16)
    return fail(MSG_ERR_UNSUPPORTED, "the dense GEMV baseline writes fp32 or fp16 Y");
  bool int4 = true, uint4 = true;
  for (int c = 0; c < 16; ++c) {
    int4 = int4 && values[c] == (double)(c < 8 ? c : c - 16);
    uint4 = uint4 && values[c] == (double)c;
  }
  if (!int4 && !uint4) return fail(MSG_ERR_UNSUPPORTED, "the dense GEMV baseline supports int4/uint4");
  if (row_bytes(k, 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(packed) & 15) != 0)
    return fail(MSG_ERR_UNSUPPORTED, "the dense GEMV baseline needs 16-byte aligned rows (k %% 32 == 0)");
  if (m == 0 || k == 0) return MSG_OK;
  // fp16 magic numbers: ((u & 0xF) ^ c) is the fp16 1024 + (u ^ 8) (int4, c = 0x6408) or
  // 1024 + u (uint4, c = 0x6400); subtracting 1032 / 1024 leaves the exact code value
  // (the high nibble of a byte: fp16 1024 + 16 (u ^ 8) / 1024 + 16 u, scaled by 1/16 minus 72 / 64)
  const uint32_t magic = int4 ? 0x64086408u : 0x64006400u;
  const uint32_t magic_hi = int4 ? 0x64806480u : 0x64006400u;
  const __half hs = __float2half_rn(int4 ? 1032.0f : 1024.0f);
  const __half hh = __float2half_rn(int4 ? -72.0f : -64.0f);
  const uint32_t sub2 = (uint32_t)__half_as_ushort(hs) * 0x10001u;
  const uint32_t sub_hi = (uint32_t)__half_as_ushort(hh) * 0x10001u;
  const __half* xh = reinterpret_cast<const __half*>(x);
  cudaStream_t s = as_stream(stream);
  switch (b) {
    case 1: return launch_dv<1>(packed, m, k, xh, magic, magic_hi, sub2, sub_hi, y, y_dtype, s);
    case 2: return launch_dv<2>(packed, m, k, xh, magic, magic_hi, sub2, sub_hi, y, y_dtype, s);
    case 3: return launch_dv<3>(packed, m, k, xh, magic, magic_hi, sub2, sub_hi, y, y_dtype, s);
    case 4: return launch_dv<4>(packed, m, k, xh, magic, magic_hi, sub2, sub_hi, y, y_dtype, s);
    case 5: return launch_dv<5>(packed, m, k, xh, magic, magic_hi, sub2, sub_hi, y, y_dtype, s);
    case 6: return launch_dv<6>(packed, m, k, xh, magic, magic_hi, sub2, sub_hi, y, y_dtype, s);
    case 7: return launch_dv<7>(packed, m, k, xh, magic, magic_hi, sub2, sub_hi, y, y_dtype, s);
    default: return launch_dv<8>(packed, m, k, xh, magic, magic_hi, sub2, sub_hi, y, y_dtype, s);
  }
}
