// Weight-format kernels: nibble pack/unpack, value encoding, group indices.
//
// Device restatements of the reference's packing module
// (/root/reference/pkg/src/msgemm/packing.py).  Layout contract
// (packing.py:99-128): width 4 -> column j in byte j/2, even j in the low
// nibble; width 2 -> column j in byte j/4 at bit 2*(j%4); other widths -> one
// code per byte.  Group index (packing.py:201-228): first code least
// significant, idx = sum_r code(j*d + r) << (width*r).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <mutex>

#include "msg_common.cuh"

namespace msg {

static thread_local std::string g_last_error;

void set_error(const std::string& s) { g_last_error = s; }

YFan& current_fan() {
  static thread_local YFan fan{};
  return fan;
}

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

int max_smem_optin() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cached[dev] = n > 0 ? n : 227 * 1024;
  }
  return cached[dev];
}

// code of column j in a packed row
__device__ __forceinline__ uint32_t code_at(const uint8_t* row, int64_t j, int width) {
  if (width == 4) return (row[j >> 1] >> ((j & 1) * 4)) & 0xF;
  if (width == 2) return (row[j >> 2] >> ((j & 3) * 2)) & 0x3;
  return row[j];
}

// ---------------------------------------------------------------- pack codes
__global__ void pack_codes_kernel(const uint8_t* __restrict__ codes, int64_t m, int64_t k,
                                  int width, int rb, uint8_t* __restrict__ out) {
  int64_t n = m * (int64_t)rb;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / rb, byte = t - i * rb;
    const uint8_t* row = codes + i * k;
    uint32_t v = 0;
    if (width == 4 || width == 2) {
      int per = 8 / width;
      for (int s = 0; s < per; ++s) {
        int64_t j = byte * per + s;
        if (j < k) v |= (uint32_t)(row[j] & ((1u << width) - 1)) << (width * s);
      }
    } else {
      v = row[byte];
    }
    out[t] = (uint8_t)v;
  }
}

// -------------------------------------------------------------- unpack codes
__global__ void unpack_codes_kernel(const uint8_t* __restrict__ packed, int64_t m, int64_t k,
                                    int width, int rb, uint8_t* __restrict__ codes) {
  int64_t n = m * k;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / k, j = t - i * k;
    codes[t] = (uint8_t)code_at(packed + i * rb, j, width);
  }
}

// ------------------------------------------------------------ group indices
__global__ void group_indices_kernel(const uint8_t* __restrict__ packed, int64_t m, int64_t k,
                                     int width, int d, int rb, int64_t* __restrict__ out) {
  int64_t nb = k / d;
  int64_t n = m * nb;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / nb, j = t - i * nb;
    const uint8_t* row = packed + i * rb;
    int64_t idx = 0;
    for (int r = 0; r < d; ++r) idx |= (int64_t)code_at(row, j * d + r, width) << (width * r);
    out[t] = idx;
  }
}

// ------------------------------------------------------------ value encoding
// nearest codebook value, |w - v| <= 1e-6 |v| or both zero (packing.py:146-169)
__global__ void encode_values_kernel(const double* __restrict__ w, const double* __restrict__ grid,
                                     int64_t m, int64_t k, int width, CodebookParam cb, int rb,
                                     uint8_t* __restrict__ out,
                                     unsigned long long* __restrict__ bad) {
  int64_t n = m * (int64_t)rb;
  int per = (width == 4 || width == 2) ? 8 / width : 1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / rb, byte = t - i * rb;
    uint32_t packedv = 0;
    for (int s = 0; s < per; ++s) {
      int64_t j = byte * per + s;
      if (j >= k) break;
      int64_t e = i * k + j;
      double x = w[e];
      if (grid) x = x / grid[e];
      int best = 0;
      double bd = fabs(x - cb.v[0]);
      for (int c = 1; c < cb.n; ++c) {
        double dd = fabs(x - cb.v[c]);
        if (dd < bd) { bd = dd; best = c; }
      }
      double got = cb.v[best];
      bool ok = (fabs(x - got) <= 1e-6 * fabs(got)) || (x == 0.0 && got == 0.0);
      if (!ok) {
        atomicAdd(&bad[0], 1ull);
        atomicMin(&bad[1], (unsigned long long)e);
      }
      packedv |= (uint32_t)best << (per > 1 ? width * s : 0);
    }
    out[t] = (uint8_t)packedv;
  }
}


// ------------------------------------------------------- row conditioning
// Sign-symmetric tables store H = sum_r (v[c_r] - beta) x_r, so a table
// rounding error scales with sum_r |v - beta| |x_r| instead of the reference's
// bound sum_r |v| |x_r| (suites.py:106-124).  ratio[i] is the expected
// (random-walk) accumulated table error of row i relative to that bound, for
// unit activations: sqrt(sum_j (sum_{r<d} |v[c_jr] - beta|)^2) / sum_c |v[c]|
// (+inf for a row without a nonzero weight, which must come out exactly 0,
// and for a row with fewer than min(8, ceil(k/2)) nonzero weights: its bound
// rests on a handful of |x_c|, any of which may be tiny).
// One warp per row, lanes stride over the d-groups.
__global__ void row_conditioning_kernel(const uint8_t* __restrict__ packed, int64_t m, int64_t k,
                                        int d, int rb, CodebookParam cb, double beta,
                                        float* __restrict__ ratio) {
  const int lane = threadIdx.x & 31;
  const int64_t nb = k / d;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < m;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint8_t* row = packed + i * rb;
    double s2 = 0.0, wabs = 0.0;
    int nnz = 0;
    for (int64_t j = lane; j < nb; j += 32) {
      double sj = 0.0;
      for (int r = 0; r < d; ++r) {
        const double v = cb.v[code_at(row, j * d + r, 4)];
        sj += fabs(v - beta);
        wabs += fabs(v);
        nnz += v != 0.0;
      }
      s2 += sj * sj;
    }
    for (int64_t j = nb * d + lane; j < k; j += 32) {
      const double v = cb.v[code_at(row, j, 4)];
      wabs += fabs(v);
      nnz += v != 0.0;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      wabs += __shfl_xor_sync(0xffffffffu, wabs, o);
      nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
    }
    const int64_t few = (k + 1) / 2 < 8 ? (k + 1) / 2 : 8;
    if (lane == 0) ratio[i] = (wabs > 0.0 && nnz >= few) ? (float)(sqrt(s2) / wabs) : INFINITY;
  }
}

// ------------------------------------------------------------- row copies
// dst[idx[i]] = src[i] (scatter) or dst[i] = src[idx[i]] (gather), rows of
// row_bytes bytes; 4-byte words when rows and pointers allow it.
template <typename W>
__global__ void copy_rows_kernel(const W* __restrict__ src, const int64_t* __restrict__ idx,
                                 int64_t n, int64_t row_words, W* __restrict__ dst, int scatter) {
  const int64_t total = n * row_words;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / row_words, w = t - i * row_words;
    const int64_t r = idx[i];
    if (scatter) dst[r * row_words + w] = src[i * row_words + w];
    else dst[i * row_words + w] = src[r * row_words + w];
  }
}

static int grid_for(int64_t n) {
  int64_t g = ceil_div(n, 256);
  int64_t cap = (int64_t)sm_count() * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

static int check_width(int width) {
  if (width < 2 || width > 8) return fail(MSG_ERR_VALUE, "width must be in 2..8, got %d", width);
  return MSG_OK;
}

}  // namespace msg

using namespace msg;

extern "C" {

const char* msg_last_error(void) { return g_last_error.c_str(); }

int msg_version(void) { return 100; }

int msg_device_sm_count(void) { return sm_count(); }

int msg_graph_run(void* graph_exec, void* stream, int sync) {
  MSG_CUDA_CHECK(cudaGraphLaunch(reinterpret_cast<cudaGraphExec_t>(graph_exec), as_stream(stream)));
  if (sync) MSG_CUDA_CHECK(cudaStreamSynchronize(as_stream(stream)));
  return MSG_OK;
}

int msg_stream_sync(void* stream) {
  MSG_CUDA_CHECK(cudaStreamSynchronize(as_stream(stream)));
  return MSG_OK;
}

int msg_pack_codes(const uint8_t* codes, int64_t m, int64_t k, int width, uint8_t* packed,
                   void* stream) {
  if (int e = check_width(width)) return e;
  if (m < 0 || k < 0) return fail(MSG_ERR_VALUE, "matrix dimensions must be non-negative");
  int rb = row_bytes(k, width);
  int64_t n = m * rb;
  if (n == 0) return MSG_OK;
  pack_codes_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(codes, m, k, width, rb, packed);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

int msg_unpack_codes(const uint8_t* packed, int64_t m, int64_t k, int width, uint8_t* codes,
                     void* stream) {
  if (int e = check_width(width)) return e;
  int rb = row_bytes(k, width);
  int64_t n = m * k;
  if (n == 0) return MSG_OK;
  unpack_codes_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(packed, m, k, width, rb, codes);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

int msg_group_indices(const uint8_t* packed, int64_t m, int64_t k, int width, int d,
                      int64_t* out, void* stream) {
  if (d < 1) return fail(MSG_ERR_VALUE, "depth d must be >= 1");
  if (d * width > 32)
    return fail(MSG_ERR_VALUE, "d*width = %d exceeds 32-bit index limit", d * width);
  int rb = row_bytes(k, width);
  int64_t n = m * (k / d);
  if (n == 0) return MSG_OK;
  group_indices_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(packed, m, k, width, d, rb,
                                                                    out);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

int msg_encode_values(const double* weights, const double* grid, int64_t m, int64_t k, int width,
                      const double* values, uint8_t* packed, int64_t* bad, void* stream) {
  if (int e = check_width(width)) return e;
  int rb = row_bytes(k, width);
  int64_t n = m * rb;
  cudaStream_t s = as_stream(stream);
  // bad[0] = count, bad[1] = first flat index (UINT64_MAX when none)
  unsigned long long init[2] = {0ull, ~0ull};
  MSG_CUDA_CHECK(cudaMemcpyAsync(bad, init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (n == 0) return MSG_OK;
  CodebookParam cb = make_codebook(values, width);
  encode_values_kernel<<<grid_for(n), 256, 0, s>>>(weights, grid, m, k, width, cb, rb, packed,
                                                   reinterpret_cast<unsigned long long*>(bad));
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

int msg_row_conditioning(const uint8_t* packed, int64_t m, int64_t k, int d, const double* values,
                         double beta, float* ratio, void* stream) {
  if (d < 1) return fail(MSG_ERR_VALUE, "depth d must be >= 1");
  if (m < 0 || k < 0) return fail(MSG_ERR_VALUE, "matrix dimensions must be non-negative");
  if (m == 0) return MSG_OK;
  CodebookParam cb = make_codebook(values, 4);
  const int grid = (int)std::min<int64_t>(ceil_div(m * 32, 256), (int64_t)sm_count() * 16);
  row_conditioning_kernel<<<grid, 256, 0, as_stream(stream)>>>(packed, m, k, d, row_bytes(k, 4),
                                                               cb, beta, ratio);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

// src -> dst, 16 bytes per thread (tail bytes by thread 0); lets the next
// kernel of the stream start its prologue at once (PDL)
__global__ void __launch_bounds__(256) stage_copy_kernel(const uint8_t* __restrict__ src,
                                                         uint8_t* __restrict__ dst, int64_t bytes) {
  griddep_launch_dependents();
  const int64_t n16 = bytes / 16;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < n16; i += (int64_t)gridDim.x * 256)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int64_t i = n16 * 16; i < bytes; ++i) dst[i] = src[i];
}

int msg_stage_copy(const void* src, void* dst, int64_t bytes, void* stream) {
  if (bytes < 0) return fail(MSG_ERR_VALUE, "negative size");
  if (bytes == 0) return MSG_OK;
  if ((((uintptr_t)src | (uintptr_t)dst) & 15) != 0)
    return fail(MSG_ERR_VALUE, "msg_stage_copy needs 16-byte aligned buffers");
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(bytes / 16, 256), 2 * sm_count()));
  stage_copy_kernel<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const uint8_t*>(src),
                                                        static_cast<uint8_t*>(dst), bytes);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

int msg_copy_rows(const void* src, const int64_t* idx, int64_t n, int64_t row_bytes_, void* dst,
                  int scatter, void* stream) {
  if (n < 0 || row_bytes_ < 0) return fail(MSG_ERR_VALUE, "negative row count or size");
  if (n == 0 || row_bytes_ == 0) return MSG_OK;
  cudaStream_t s = as_stream(stream);
  const bool words = row_bytes_ % 4 == 0 && ((uintptr_t)src & 3) == 0 && ((uintptr_t)dst & 3) == 0;
  if (words) {
    const int64_t rw = row_bytes_ / 4;
    copy_rows_kernel<uint32_t><<<grid_for(n * rw), 256, 0, s>>>(
        static_cast<const uint32_t*>(src), idx, n, rw, static_cast<uint32_t*>(dst), scatter);
  } else {
    copy_rows_kernel<uint8_t><<<grid_for(n * row_bytes_), 256, 0, s>>>(
        static_cast<const uint8_t*>(src), idx, n, row_bytes_, static_cast<uint8_t*>(dst), scatter);
  }
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

}  // extern "C"
