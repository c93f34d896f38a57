// Phase 1 (table build) with the reference's exact rounding, and the generic
// global-memory-table msGeMM path.
//
// Table entries follow lut.py:59-72 bit for bit: for index
// e = i0 + i1*n + ... (n = 2^width), entry = x[d-1]*v[i_{d-1}] + (... +
// (x[1]*v[i1] + x[0]*v[i0])), every product and sum rounded to the activation
// dtype (numpy semantics: fp16 ops are computed in fp32 and rounded once;
// integer ops wrap).
//
// The generic msGeMM (gemm.py:89-153) materialises those tables in HBM for a
// (column chunk x block chunk), then gathers with one thread per (row,
// column) in fixed block order and finishes with the k%d tail and the scales
// (gemm.py:70-86).  It serves every d (<= 7), width and dtype the fused
// shared-memory kernels do not, and is never the headline path.
#include <algorithm>
#include <type_traits>

#include "msg_common.cuh"

namespace msg {

// ------------------------------------------------------------------ arith
template <typename T> struct Arith;

template <> struct Arith<__half> {
  static __device__ __forceinline__ __half cast(double v) { return __double2half(v); }
  static __device__ __forceinline__ __half mul(__half a, __half b) {
    return __float2half_rn(__fmul_rn(__half2float(a), __half2float(b)));
  }
  static __device__ __forceinline__ __half add(__half a, __half b) {
    return __float2half_rn(__fadd_rn(__half2float(a), __half2float(b)));
  }
};
template <> struct Arith<float> {
  static __device__ __forceinline__ float cast(double v) { return (float)v; }
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};
template <> struct Arith<double> {
  static __device__ __forceinline__ double cast(double v) { return v; }
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};
// integers: numpy wraps; do the arithmetic in the unsigned type of equal width
template <typename T, typename U> struct IntArith {
  static __device__ __forceinline__ T cast(double v) { return (T)(int64_t)v; }  // trunc
  static __device__ __forceinline__ T mul(T a, T b) { return (T)(U)((U)a * (U)b); }
  static __device__ __forceinline__ T add(T a, T b) { return (T)(U)((U)a + (U)b); }
};
template <> struct Arith<int64_t> : IntArith<int64_t, unsigned long long> {};
template <> struct Arith<int32_t> : IntArith<int32_t, uint32_t> {};
template <> struct Arith<int16_t> : IntArith<int16_t, uint16_t> {};
template <> struct Arith<int8_t> : IntArith<int8_t, uint8_t> {};
template <> struct Arith<uint8_t> : IntArith<uint8_t, uint8_t> {};

// ------------------------------------------------------------ table build
// out[cc][jj][e] for columns [col0, col0+ncols) and blocks [blk0, blk0+nblk)
template <typename T>
__global__ void lut_build_kernel(const T* __restrict__ x, int64_t ldx, int64_t col0, int ncols,
                                 int64_t blk0, int64_t nblk, int d, CodebookParam cb,
                                 T* __restrict__ out) {
  const int64_t E = (int64_t)1 << (cb.width * d);
  const int64_t total = (int64_t)ncols * nblk * E;
  const uint32_t mask = (1u << cb.width) - 1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t e = t % E;
    int64_t rest = t / E;
    int64_t jj = rest % nblk;
    int64_t cc = rest / nblk;
    int64_t j = blk0 + jj;
    const T* xp = x + col0 + cc;  // column (col0+cc), element r of block j at row j*d+r
    T acc = Arith<T>::mul(xp[(j * d) * ldx], Arith<T>::cast(cb.v[e & mask]));
    for (int r = 1; r < d; ++r) {
      uint32_t code = (uint32_t)(e >> (cb.width * r)) & mask;
      T p = Arith<T>::mul(xp[(j * d + r) * ldx], Arith<T>::cast(cb.v[code]));
      acc = Arith<T>::add(p, acc);
    }
    out[t] = acc;
  }
}

// ------------------------------------------------------------ gather
template <typename T> struct AccOf { using type = double; };
template <> struct AccOf<__half> { using type = float; };     // numpy fp16 sums in fp32
template <> struct AccOf<int64_t> { using type = int64_t; };
template <> struct AccOf<int32_t> { using type = int64_t; };
template <> struct AccOf<int16_t> { using type = int64_t; };
template <> struct AccOf<int8_t> { using type = int64_t; };
template <> struct AccOf<uint8_t> { using type = int64_t; };

template <typename A, typename T> __device__ __forceinline__ A to_acc(T v) { return (A)v; }
template <> __device__ __forceinline__ float to_acc<float, __half>(__half v) {
  return __half2float(v);
}
template <> __device__ __forceinline__ double to_acc<double, __half>(__half v) {
  return (double)__half2float(v);
}

__device__ __forceinline__ uint32_t code_of(const uint8_t* row, int64_t j, int width) {
  if (width == 4) return (row[j >> 1] >> ((j & 1) * 4)) & 0xF;
  if (width == 2) return (row[j >> 2] >> ((j & 3) * 2)) & 0x3;
  return row[j];
}

// acc[i][col0+cc] (+)= sum_{jj} [q(i, grp)] * lut[cc][jj][idx(i, blk0+jj)]
template <typename T>
__global__ void gather_kernel(const uint8_t* __restrict__ packed, int64_t m, int rb, int width,
                              int d, const T* __restrict__ lut, int64_t col0, int ncols,
                              int64_t b, int64_t blk0, int64_t nblk, int first,
                              int scale_mode, int64_t group_size, const void* q, int q_dtype,
                              int64_t qcols, void* accbuf) {
  using A = typename AccOf<T>::type;
  A* acc = reinterpret_cast<A*>(accbuf);
  const int64_t E = (int64_t)1 << (width * d);
  const int64_t total = m * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t cc = t / m;
    int64_t i = t - cc * m;
    const uint8_t* row = packed + i * rb;
    const T* tab = lut + cc * nblk * E;
    A s = first ? (A)0 : acc[i * b + col0 + cc];
    for (int64_t jj = 0; jj < nblk; ++jj) {
      int64_t j = blk0 + jj;
      uint32_t idx = 0;
      for (int r = 0; r < d; ++r) idx |= code_of(row, j * d + r, width) << (width * r);
      A v = to_acc<A>(tab[jj * E + idx]);
      if (scale_mode == MSG_SCALE_PER_GROUP) {
        int64_t g = (j * d) / group_size;
        v = v * load_as<A>(q, q_dtype, i * qcols + g);
      }
      s += v;
    }
    acc[i * b + col0 + cc] = s;
  }
}

// y[i][c] = (acc + tail) * q_row   -> y dtype
template <typename A>
__global__ void finish_kernel(const uint8_t* __restrict__ packed, int64_t m, int64_t k, int rb,
                              int width, int d, CodebookParam cb, const void* x, int x_dtype,
                              int64_t b, const void* accbuf, int scale_mode, const void* q,
                              int q_dtype, void* y, int y_dtype) {
  const A* acc = reinterpret_cast<const A*>(accbuf);
  const int64_t nb = k / d;
  const int64_t total = m * b;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / b, c = t - i * b;
    A s = acc ? acc[t] : (A)0;
    if (scale_mode != MSG_SCALE_PER_GROUP) {
      const uint8_t* row = packed + i * rb;
      for (int64_t j = nb * d; j < k; ++j) {
        uint32_t code = code_of(row, j, width);
        A w;
        if constexpr (std::is_integral<A>::value) w = (A)(int64_t)cb.v[code];
        else w = (A)cb.v[code];
        s += w * load_as<A>(x, x_dtype, j * b + c);
      }
      if (scale_mode == MSG_SCALE_PER_ROW) s = s * load_as<A>(q, q_dtype, i);
    }
    store_as<A>(y, y_dtype, t, s);
  }
}

static int grid_for(int64_t n) {
  int64_t g = ceil_div(n, 256);
  int64_t cap = (int64_t)sm_count() * 32;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

// ------------------------------------------------------------ host drivers
template <typename T>
static int launch_lut(const void* x, int64_t ldx, int64_t col0, int ncols, int64_t blk0,
                      int64_t nblk, int d, const CodebookParam& cb, void* out, cudaStream_t s) {
  int64_t E = (int64_t)1 << (cb.width * d);
  int64_t n = (int64_t)ncols * nblk * E;
  if (n == 0) return MSG_OK;
  lut_build_kernel<T><<<grid_for(n), 256, 0, s>>>((const T*)x, ldx, col0, ncols, blk0, nblk, d,
                                                  cb, (T*)out);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

int lut_dispatch(int dtype, const void* x, int64_t ldx, int64_t col0, int ncols, int64_t blk0,
                 int64_t nblk, int d, const CodebookParam& cb, void* out, cudaStream_t s) {
  switch (dtype) {
    case MSG_F16: return launch_lut<__half>(x, ldx, col0, ncols, blk0, nblk, d, cb, out, s);
    case MSG_F32: return launch_lut<float>(x, ldx, col0, ncols, blk0, nblk, d, cb, out, s);
    case MSG_F64: return launch_lut<double>(x, ldx, col0, ncols, blk0, nblk, d, cb, out, s);
    case MSG_I64: return launch_lut<int64_t>(x, ldx, col0, ncols, blk0, nblk, d, cb, out, s);
    case MSG_I32: return launch_lut<int32_t>(x, ldx, col0, ncols, blk0, nblk, d, cb, out, s);
    case MSG_I16: return launch_lut<int16_t>(x, ldx, col0, ncols, blk0, nblk, d, cb, out, s);
    case MSG_I8: return launch_lut<int8_t>(x, ldx, col0, ncols, blk0, nblk, d, cb, out, s);
    case MSG_U8: return launch_lut<uint8_t>(x, ldx, col0, ncols, blk0, nblk, d, cb, out, s);
  }
  return fail(MSG_ERR_UNSUPPORTED, "activation dtype %d is not supported on the GPU path", dtype);
}

// Generic-path workspace: [acc m*b*8][lut chunk]
static const int64_t kGenericLutCap = (int64_t)1 << 30;

struct GenericPlan {
  int64_t cols_per_chunk, blocks_per_chunk, lut_bytes, acc_bytes;
};

GenericPlan generic_plan(int64_t m, int64_t k, int width, int x_dtype, int64_t b, int d) {
  GenericPlan p{};
  int64_t nb = k / d;
  int64_t E = (int64_t)1 << (width * d);
  int64_t eb = E * dtype_size(x_dtype);
  p.acc_bytes = ((m * b * 8 + 255) / 256) * 256;
  if (nb == 0 || b == 0) {
    p.cols_per_chunk = b > 0 ? b : 1;
    p.blocks_per_chunk = nb > 0 ? nb : 1;
    p.lut_bytes = 0;
    return p;
  }
  int64_t per_col = eb * nb;
  if (per_col <= kGenericLutCap) {
    p.blocks_per_chunk = nb;
    p.cols_per_chunk = std::max<int64_t>(1, std::min<int64_t>(b, kGenericLutCap / per_col));
  } else {
    p.cols_per_chunk = 1;
    p.blocks_per_chunk = std::max<int64_t>(1, kGenericLutCap / eb);
  }
  p.lut_bytes = p.cols_per_chunk * p.blocks_per_chunk * eb;
  return p;
}

int64_t generic_workspace_bytes(int64_t m, int64_t k, int width, int x_dtype, int64_t b, int d) {
  GenericPlan p = generic_plan(m, k, width, x_dtype, b, d);
  return p.acc_bytes + p.lut_bytes;
}

template <typename T>
static int run_generic_t(const uint8_t* packed, int64_t m, int64_t k, int width,
                         const CodebookParam& cb, const void* x, int x_dtype, int64_t b, int d,
                         int scale_mode, int64_t group_size, const void* q, int q_dtype,
                         void* y, int y_dtype, void* ws, cudaStream_t s) {
  using A = typename AccOf<T>::type;
  GenericPlan p = generic_plan(m, k, width, x_dtype, b, d);
  int64_t nb = k / d;
  int rb = row_bytes(k, width);
  void* acc = ws;
  void* lut = (char*)ws + p.acc_bytes;
  int64_t qcols = scale_mode == MSG_SCALE_PER_GROUP ? k / group_size : 1;
  if (nb > 0) {
    for (int64_t c0 = 0; c0 < b; c0 += p.cols_per_chunk) {
      int nc = (int)std::min<int64_t>(p.cols_per_chunk, b - c0);
      for (int64_t j0 = 0; j0 < nb; j0 += p.blocks_per_chunk) {
        int64_t nbk = std::min<int64_t>(p.blocks_per_chunk, nb - j0);
        if (int e = launch_lut<T>(x, b, c0, nc, j0, nbk, d, cb, lut, s)) return e;
        gather_kernel<T><<<grid_for(m * nc), 256, 0, s>>>(
            packed, m, rb, width, d, (const T*)lut, c0, nc, b, j0, nbk, j0 == 0 ? 1 : 0,
            scale_mode, group_size, q, q_dtype, qcols, acc);
        MSG_LAUNCH_CHECK();
      }
    }
  }
  finish_kernel<A><<<grid_for(m * b), 256, 0, s>>>(packed, m, k, rb, width, d, cb, x, x_dtype, b,
                                                  nb > 0 ? acc : nullptr, scale_mode, q, q_dtype,
                                                  y, y_dtype);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

int run_generic(const uint8_t* packed, int64_t m, int64_t k, int width, const CodebookParam& cb,
                const void* x, int x_dtype, int64_t b, int d, int scale_mode, int64_t group_size,
                const void* q, int q_dtype, void* y, int y_dtype, void* ws, int64_t ws_bytes,
                cudaStream_t s) {
  if (ws_bytes < generic_workspace_bytes(m, k, width, x_dtype, b, d))
    return fail(MSG_ERR_WORKSPACE, "workspace too small for the generic path");
  if (m == 0 || b == 0) return MSG_OK;
#define MSG_GEN(T)                                                                          \
  return run_generic_t<T>(packed, m, k, width, cb, x, x_dtype, b, d, scale_mode, group_size, \
                          q, q_dtype, y, y_dtype, ws, s)
  switch (x_dtype) {
    case MSG_F16: MSG_GEN(__half);
    case MSG_F32: MSG_GEN(float);
    case MSG_F64: MSG_GEN(double);
    case MSG_I64: MSG_GEN(int64_t);
    case MSG_I32: MSG_GEN(int32_t);
    case MSG_I16: MSG_GEN(int16_t);
    case MSG_I8: MSG_GEN(int8_t);
    case MSG_U8: MSG_GEN(uint8_t);
  }
#undef MSG_GEN
  return fail(MSG_ERR_UNSUPPORTED, "activation dtype %d is not supported on the GPU path",
              x_dtype);
}

}  // namespace msg

using namespace msg;

extern "C" int msg_lut_build(const void* x, int dtype, int64_t k, int64_t ldx, int d,
                             const double* values, int width, int64_t block_lo,
                             int64_t block_hi, void* entries, void* stream) {
  if (d < 1) return fail(MSG_ERR_VALUE, "depth d must be >= 1");
  if (width < 2 || width > 8) return fail(MSG_ERR_VALUE, "width must be in 2..8");
  if (width * d > 28)
    return fail(MSG_ERR_UNSUPPORTED, "tables of 2^%d entries per block are not supported",
                width * d);
  int64_t nb = k / d;
  if (block_lo < 0 || block_hi > nb || block_lo > block_hi)
    return fail(MSG_ERR_INDEX, "block range [%lld, %lld) out of range; k=%lld, d=%d gives %lld blocks",
                (long long)block_lo, (long long)block_hi, (long long)k, d, (long long)nb);
  CodebookParam cb = make_codebook(values, width);
  return lut_dispatch(dtype, x, ldx, 0, 1, block_lo, block_hi - block_lo, d, cb, entries,
                      as_stream(stream));
}

// ------------------------------------------------------------------ naive_gemm
// Dense reference product Y = W @ X (gemm.py:206-216) with numpy's
// semantics: both operands integer -> int64 products and sums (two's
// complement wrap, order-free); otherwise both operands are converted to the
// result dtype numpy picks (np.result_type) and multiplied:
//   f16: numpy's non-BLAS half loop -- fp32 sum over k in order of exact fp32
//        products, rounded to fp16 once (bit-exact against numpy);
//   f32 / f64: BLAS in numpy (order unspecified); here a correctly rounded
//        fp64 sum in k order, rounded to the result dtype.
// Tiles of 64 rows x 16 columns x 32 k staged through shared memory (coalesced
// row-major loads of W and X); each thread owns 4 rows of one column and walks
// k in order, so the summation order is fixed whatever the tiling.
namespace msg {

enum NaiveMode { NAIVE_INT = 0, NAIVE_F16 = 1, NAIVE_F32 = 2, NAIVE_F64 = 3 };

template <int MODE> struct NaiveT;
template <> struct NaiveT<NAIVE_INT> {
  using V = int64_t; using A = uint64_t;
  static __device__ __forceinline__ V load(const void* p, int dt, int64_t i) { return load_as<int64_t>(p, dt, i); }
  static __device__ __forceinline__ A step(A acc, V a, V b) { return acc + (uint64_t)a * (uint64_t)b; }
  static __device__ __forceinline__ void store(void* p, int dt, int64_t i, A acc) { ((int64_t*)p)[i] = (int64_t)acc; }
};
template <> struct NaiveT<NAIVE_F16> {
  using V = float; using A = float;   // operands hold fp16-rounded values
  static __device__ __forceinline__ V load(const void* p, int dt, int64_t i) {
    return dt == MSG_F16 ? __half2float(((const __half*)p)[i])
                         : __half2float(__double2half(load_as<double>(p, dt, i)));
  }
  static __device__ __forceinline__ A step(A acc, V a, V b) { return __fadd_rn(acc, __fmul_rn(a, b)); }
  static __device__ __forceinline__ void store(void* p, int, int64_t i, A acc) { ((__half*)p)[i] = __float2half_rn(acc); }
};
template <> struct NaiveT<NAIVE_F32> {
  using V = float; using A = double;
  static __device__ __forceinline__ V load(const void* p, int dt, int64_t i) {
    return dt == MSG_F32 ? ((const float*)p)[i] : (float)load_as<double>(p, dt, i);
  }
  static __device__ __forceinline__ A step(A acc, V a, V b) { return fma((double)a, (double)b, acc); }
  static __device__ __forceinline__ void store(void* p, int, int64_t i, A acc) { ((float*)p)[i] = (float)acc; }
};
template <> struct NaiveT<NAIVE_F64> {
  using V = double; using A = double;
  static __device__ __forceinline__ V load(const void* p, int dt, int64_t i) { return load_as<double>(p, dt, i); }
  static __device__ __forceinline__ A step(A acc, V a, V b) { return fma(a, b, acc); }
  static __device__ __forceinline__ void store(void* p, int, int64_t i, A acc) { ((double*)p)[i] = acc; }
};

constexpr int NV_BM = 64, NV_BN = 16, NV_BK = 32, NV_THREADS = 256;

template <int MODE>
__global__ void __launch_bounds__(NV_THREADS)
naive_gemm_kernel(const void* __restrict__ W, int w_dt, const void* __restrict__ X, int x_dt,
                  int64_t m, int64_t k, int64_t b, void* __restrict__ Y) {
  using T = NaiveT<MODE>;
  using V = typename T::V;
  using A = typename T::A;
  __shared__ V ws[NV_BM][NV_BK + 1];
  __shared__ V xs[NV_BK][NV_BN];
  const int tid = threadIdx.x;
  const int col = tid % NV_BN, rq = tid / NV_BN;          // 16 row quads x 16 columns
  const int64_t row0 = (int64_t)blockIdx.x * NV_BM, col0 = (int64_t)blockIdx.y * NV_BN;
  A acc[4] = {A(0), A(0), A(0), A(0)};
  for (int64_t k0 = 0; k0 < k; k0 += NV_BK) {
    for (int e = tid; e < NV_BM * NV_BK; e += NV_THREADS) {
      int r = e / NV_BK, c = e % NV_BK;
      int64_t gr = row0 + r, gc = k0 + c;
      ws[r][c] = (gr < m && gc < k) ? T::load(W, w_dt, gr * k + gc) : V(0);
    }
    for (int e = tid; e < NV_BK * NV_BN; e += NV_THREADS) {
      int r = e / NV_BN, c = e % NV_BN;
      int64_t gr = k0 + r, gc = col0 + c;
      xs[r][c] = (gr < k && gc < b) ? T::load(X, x_dt, gr * b + gc) : V(0);
    }
    __syncthreads();
    const int kk = (k - k0 < NV_BK) ? (int)(k - k0) : NV_BK;
    for (int c = 0; c < kk; ++c) {
      V xv = xs[c][col];
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = T::step(acc[i], ws[rq * 4 + i][c], xv);
    }
    __syncthreads();
  }
  const int64_t gc = col0 + col;
  if (gc >= b) return;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t gr = row0 + rq * 4 + i;
    if (gr < m) T::store(Y, 0, gr * b + gc, acc[i]);
  }
}

}  // namespace msg

extern "C" int msg_naive_gemm(const void* w, int w_dtype, const void* x, int x_dtype, int64_t m,
                              int64_t k, int64_t b, int mode, void* y, void* stream) {
  if (m < 0 || k < 0 || b < 0) return fail(MSG_ERR_VALUE, "negative dimension");
  if (dtype_size(w_dtype) <= 0 || dtype_size(x_dtype) <= 0 || w_dtype == MSG_BF16 || x_dtype == MSG_BF16)
    return fail(MSG_ERR_UNSUPPORTED, "naive_gemm: unsupported operand dtype (%d, %d)", w_dtype, x_dtype);
  if (m == 0 || b == 0) return MSG_OK;
  if (mode == NAIVE_INT && !(dtype_is_int(w_dtype) && dtype_is_int(x_dtype)))
    return fail(MSG_ERR_VALUE, "naive_gemm: integer mode needs integer operands");
  dim3 grid((unsigned)ceil_div(m, NV_BM), (unsigned)ceil_div(b, NV_BN));
  if (grid.y > 65535) return fail(MSG_ERR_UNSUPPORTED, "naive_gemm: b too large");
  cudaStream_t s = as_stream(stream);
  switch (mode) {
    case NAIVE_INT: naive_gemm_kernel<NAIVE_INT><<<grid, NV_THREADS, 0, s>>>(w, w_dtype, x, x_dtype, m, k, b, y); break;
    case NAIVE_F16: naive_gemm_kernel<NAIVE_F16><<<grid, NV_THREADS, 0, s>>>(w, w_dtype, x, x_dtype, m, k, b, y); break;
    case NAIVE_F32: naive_gemm_kernel<NAIVE_F32><<<grid, NV_THREADS, 0, s>>>(w, w_dtype, x, x_dtype, m, k, b, y); break;
    case NAIVE_F64: naive_gemm_kernel<NAIVE_F64><<<grid, NV_THREADS, 0, s>>>(w, w_dtype, x, x_dtype, m, k, b, y); break;
    default: return fail(MSG_ERR_VALUE, "naive_gemm: bad mode %d", mode);
  }
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}
