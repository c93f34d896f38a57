// K3 (weight repack) and K1+K2 fused shared-memory LUT kernel for msGeMM.
//
// Reference semantics: gemm.py:89-153 (msgemm), gemm.py:70-86 (the column
// reduction, k%d tail, per-row scale), lut.py:59-72 (table entries),
// packing.py:201-228 (group index: first code least significant).
//
// Design (sm_100a, one CTA per SM):
//   * K3 repacks the reference's row-major nibbles (packing.py:99-114) into
//     "quad planes": for every 4 consecutive d-groups and every row, a 32-bit
//     word of low index bytes (d=2,3; 16 bits for d=1) and, for d=3, a 16-bit
//     word of high index nibbles.  Density stays 4*d bits per group, and a
//     warp reading one plane word for 32 consecutive rows issues one
//     coalesced 128-byte request.  For antisymmetric codebooks
//     (v[c] + v[~c] = 2*beta, e.g. two's-complement int4 with beta = -1/2)
//     K3 folds the sign symmetry into the stored index: an index with the top
//     bit set is stored complemented with a sign bit, so tables hold only
//     2^(4d-1) entries: L(idx) = +-H[f] + beta*(x_0 + .. + x_{d-1}).
//   * The fused kernel gives each CTA a block of R = 256*RPT rows, a k-slice
//     of quads and a tile of BC batch columns.  Per round it builds the
//     tables of QL quads (4*QL groups x ES entries x BC columns, batch
//     innermost so one vector LDS fetches all BC columns of an entry) into
//     shared memory, then every thread gathers for its RPT rows and
//     accumulates fp32 in registers.  Tables are built once per (row block,
//     k-slice); the build is amortised over R rows.
//   * k-slice partials go to a workspace [S][m][b] (fp32) and a second,
//     deterministic pass sums them in slice order, adds the k%d tail, the
//     symmetry correction and the per-row scale, and casts to Y's dtype.
#include <algorithm>
#include <cstring>

#include "msg_common.cuh"

namespace msg {

int run_generic(const uint8_t* packed, int64_t m, int64_t k, int width, const CodebookParam& cb,
                const void* x, int x_dtype, int64_t b, int d, int scale_mode, int64_t group_size,
                const void* q, int q_dtype, void* y, int y_dtype, void* ws, int64_t ws_bytes,
                cudaStream_t s);
int64_t generic_workspace_bytes(int64_t m, int64_t k, int width, int x_dtype, int64_t b, int d);

static inline int64_t align256(int64_t v) { return (v + 255) / 256 * 256; }

// ============================================================================
// K3: quad-plane repack
// ============================================================================
struct QuadLayout {
  int64_t nb, nq, tail;
  int64_t lo_off, hi_off, tail_off, total;
  int lo_bytes;  // 4 for d=2,3 ; 2 for d=1
  bool has_hi;
};

static QuadLayout quad_layout(int64_t m, int64_t k, int d) {
  QuadLayout L{};
  L.nb = k / d;
  L.nq = (L.nb + 3) / 4;
  L.tail = k - L.nb * d;
  L.lo_bytes = d == 1 ? 2 : 4;
  L.has_hi = d == 3;
  L.lo_off = 0;
  L.hi_off = align256(L.nq * m * L.lo_bytes);
  L.tail_off = L.hi_off + (L.has_hi ? align256(L.nq * m * 2) : 0);
  L.total = L.tail_off + (L.tail ? align256(m * 2) : 0);
  if (L.total == 0) L.total = 256;
  return L;
}

__device__ __forceinline__ uint32_t nib(const uint8_t* row, int64_t j) {
  return (row[j >> 1] >> ((j & 1) * 4)) & 0xF;
}

// one thread per (quad, row): rows fastest so plane stores coalesce
__global__ void repack_quad_kernel(const uint8_t* __restrict__ packed, int64_t m, int64_t k,
                                   int d, int rb, int symmetric, QuadLayout L,
                                   uint8_t* __restrict__ out) {
  const int64_t total = L.nq * m;
  const int bits = 4 * d;
  const uint32_t emask = (1u << bits) - 1;
  const uint32_t top = 1u << (bits - 1);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t q = t / m, i = t - q * m;
    const uint8_t* row = packed + i * rb;
    uint32_t lo = 0, hi = 0;
    for (int g = 0; g < 4; ++g) {
      int64_t j = q * 4 + g;
      uint32_t st = 0;
      if (j < L.nb) {
        uint32_t idx = 0;
        for (int r = 0; r < d; ++r) idx |= nib(row, j * d + r) << (4 * r);
        if (symmetric && (idx & top)) idx = (idx ^ emask) | top;  // complement, keep sign bit
        st = idx;
      }
      if (d == 1) lo |= st << (4 * g);
      else if (d == 2) lo |= st << (8 * g);
      else { lo |= (st & 0xFF) << (8 * g); hi |= (st >> 8) << (4 * g); }
    }
    if (d == 1) reinterpret_cast<uint16_t*>(out + L.lo_off)[t] = (uint16_t)lo;
    else reinterpret_cast<uint32_t*>(out + L.lo_off)[t] = lo;
    if (L.has_hi) reinterpret_cast<uint16_t*>(out + L.hi_off)[t] = (uint16_t)hi;
    if (L.tail && q == 0) {
      uint32_t tc = 0;
      for (int64_t j = L.nb * d; j < k; ++j) tc |= nib(row, j) << (4 * (j - L.nb * d));
      reinterpret_cast<uint16_t*>(out + L.tail_off)[i] = (uint16_t)tc;
    }
  }
}

// ============================================================================
// fused LUT kernel
// ============================================================================
constexpr int kThreads = 256;

struct FusedParams {
  const uint8_t* wrep;
  int64_t lo_off, hi_off;
  int64_t m, nb, nq;
  const void* x;  // (k, b) row-major, F16 or F32
  int64_t b;
  int d;
  float s[16];  // per-code value used in tables: v[c] - beta (symmetric) or v[c]
  float beta;
  int quads_per_slice;  // k-slice length in quads
  int ql;               // quads per table round
  float* partial;       // [S][m][b]
  float* corr;          // [S][b]   beta * sum of x over the slice (symmetric only)
};

template <typename XT> __device__ __forceinline__ float ldx(const void* p, int64_t i);
template <> __device__ __forceinline__ float ldx<float>(const void* p, int64_t i) {
  return reinterpret_cast<const float*>(p)[i];
}
template <> __device__ __forceinline__ float ldx<__half>(const void* p, int64_t i) {
  return __half2float(reinterpret_cast<const __half*>(p)[i]);
}

// BC entries of type ET as raw 32-bit words
template <typename ET, int BC> struct EntryVec {
  static constexpr int kBytes = BC * (int)sizeof(ET);
  static constexpr int kWords = kBytes >= 4 ? kBytes / 4 : 1;
};

template <typename ET, int BC>
__device__ __forceinline__ void load_entry(const uint8_t* p, uint32_t (&w)[EntryVec<ET, BC>::kWords]) {
  constexpr int B = EntryVec<ET, BC>::kBytes;
  if constexpr (B == 2) {
    w[0] = *reinterpret_cast<const uint16_t*>(p);
  } else if constexpr (B == 4) {
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  } else if constexpr (B == 8) {
    uint2 v = *reinterpret_cast<const uint2*>(p);
    w[0] = v.x; w[1] = v.y;
  } else {
#pragma unroll
    for (int i = 0; i < B / 16; ++i) {
      uint4 v = reinterpret_cast<const uint4*>(p)[i];
      w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
    }
  }
}

template <typename ET, int BC>
__device__ __forceinline__ float entry_col(const uint32_t (&w)[EntryVec<ET, BC>::kWords], int c) {
  if constexpr (sizeof(ET) == 4) {
    return __uint_as_float(w[c]);
  } else {
    uint32_t word = w[c >> 1];
    __half h = __ushort_as_half((unsigned short)((c & 1) ? (word >> 16) : (word & 0xFFFF)));
    return __half2float(h);
  }
}

template <typename ET> __device__ __forceinline__ void store_entries(uint8_t* p, const float* v, int n);

template <int D, typename XT, typename ET, int BC, bool SYM, int RPT>
__global__ void __launch_bounds__(kThreads, 1) fused_lut_kernel(FusedParams P) {
  constexpr int ES = SYM ? (1 << (4 * D - 1)) : (1 << (4 * D));  // stored entries per group
  constexpr int EB = BC * (int)sizeof(ET);                        // bytes per entry
  constexpr int LOWN = D == 1 ? 1 : (D == 2 ? 16 : 256);          // combos of the low D-1 codes
  constexpr int HIN = SYM ? 8 : 16;                               // values of the top code
  extern __shared__ __align__(16) uint8_t smem[];

  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * kThreads * RPT;
  const int slice = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.z * BC;
  const int64_t q_begin = (int64_t)slice * P.quads_per_slice;
  const int64_t q_end = (P.nq < q_begin + P.quads_per_slice ? P.nq : q_begin + P.quads_per_slice);

  const int groups_cap = P.ql * 4;
  uint8_t* tab = smem;                                              // [groups][ES][BC] ET
  float* xs = reinterpret_cast<float*>(smem + (size_t)groups_cap * ES * EB);  // [groups*D][BC]

  float acc[RPT][BC];
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int c = 0; c < BC; ++c) acc[r][c] = 0.f;
  float corr = 0.f;  // thread tid < BC accumulates column tid's correction

  const uint32_t* lo_plane = reinterpret_cast<const uint32_t*>(P.wrep + P.lo_off);
  const uint16_t* lo16_plane = reinterpret_cast<const uint16_t*>(P.wrep + P.lo_off);
  const uint16_t* hi_plane = reinterpret_cast<const uint16_t*>(P.wrep + P.hi_off);

  for (int64_t qa = q_begin; qa < q_end; qa += P.ql) {
    const int nql = (int)((int64_t)P.ql < q_end - qa ? (int64_t)P.ql : q_end - qa);
    const int64_t g_first = qa * 4;
    const int ngroups = (int)((int64_t)nql * 4 < P.nb - g_first ? (int64_t)nql * 4 : P.nb - g_first);

    __syncthreads();  // previous round's gathers are done with tab/xs
    // ---- stage x for this round's groups: xs[gl*D + r][c] = x[(g*D + r), c0 + c]
    for (int t = tid; t < ngroups * D * BC; t += kThreads) {
      int c = t % BC, gr = t / BC;
      int64_t col = c0 + c;
      float v = 0.f;
      if (col < P.b) v = ldx<XT>(P.x, (g_first * D + gr) * P.b + col);
      xs[t] = v;
    }
    __syncthreads();
    if (SYM && tid < BC) {
      float s = 0.f;
      for (int gr = 0; gr < ngroups * D; ++gr) s += xs[gr * BC + tid];
      corr += s;
    }
    // ---- build: entry(f) = sum_r s[nibble_r(f)] * x_r, top nibble < HIN
    for (int t = tid; t < ngroups * LOWN; t += kThreads) {
      const int gl = t / LOWN, low = t - gl * LOWN;
      const float* xg = xs + gl * D * BC;
      float base[BC];
#pragma unroll
      for (int c = 0; c < BC; ++c) {
        float v = 0.f;
        if constexpr (D >= 2) v = P.s[low & 15] * xg[c];
        if constexpr (D >= 3) v = fmaf(P.s[(low >> 4) & 15], xg[BC + c], v);
        base[c] = v;
      }
      const float* xt = xg + (D - 1) * BC;
      uint8_t* dst = tab + ((size_t)gl * ES + low) * EB;
#pragma unroll 4
      for (int h = 0; h < HIN; ++h) {
        float e[BC];
        const float sh = P.s[h];
#pragma unroll
        for (int c = 0; c < BC; ++c) e[c] = fmaf(sh, xt[c], base[c]);
        store_entries<ET>(dst + (size_t)h * LOWN * EB, e, BC);
      }
    }
    __syncthreads();
    // ---- gather
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const int64_t i = row0 + (int64_t)r * kThreads + tid;
      if (i < P.m) {
        for (int qq = 0; qq < nql; ++qq) {
          const int64_t q = qa + qq;
          uint32_t lo, hi = 0;
          if constexpr (D == 1) lo = lo16_plane[q * P.m + i];
          else lo = __ldg(lo_plane + q * P.m + i);
          if constexpr (D == 3) hi = hi_plane[q * P.m + i];
          const int gbase = qq * 4;
          const int gmax = min(4, ngroups - gbase);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            if (g < gmax) {
              uint32_t st;
              if constexpr (D == 1) st = (lo >> (4 * g)) & 0xF;
              else if constexpr (D == 2) st = (lo >> (8 * g)) & 0xFF;
              else st = ((lo >> (8 * g)) & 0xFF) | (((hi >> (4 * g)) & 0xF) << 8);
              float sg = 1.f;
              uint32_t f = st;
              if constexpr (SYM) {
                f = st & (ES - 1);
                sg = (st & ES) ? -1.f : 1.f;
              }
              uint32_t w[EntryVec<ET, BC>::kWords];
              load_entry<ET, BC>(tab + ((size_t)(gbase + g) * ES + f) * EB, w);
#pragma unroll
              for (int c = 0; c < BC; ++c) acc[r][c] = fmaf(sg, entry_col<ET, BC>(w, c), acc[r][c]);
            }
          }
        }
      }
    }
  }
  // ---- write partials [slice][i][c]
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int64_t i = row0 + (int64_t)r * kThreads + tid;
    if (i < P.m) {
      float* dst = P.partial + ((int64_t)slice * P.m + i) * P.b + c0;
#pragma unroll
      for (int c = 0; c < BC; ++c)
        if (c0 + c < P.b) dst[c] = acc[r][c];
    }
  }
  if (SYM && blockIdx.x == 0 && tid < BC && c0 + tid < P.b)
    P.corr[(int64_t)slice * P.b + c0 + tid] = P.beta * corr;
}

template <> __device__ __forceinline__ void store_entries<float>(uint8_t* p, const float* v, int n) {
  if (n == 1) { *reinterpret_cast<float*>(p) = v[0]; return; }
  if (n == 2) { *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]); return; }
  for (int i = 0; i < n; i += 4)
    reinterpret_cast<float4*>(p)[i / 4] = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
}
template <> __device__ __forceinline__ void store_entries<__half>(uint8_t* p, const float* v, int n) {
  if (n == 1) { *reinterpret_cast<__half*>(p) = __float2half_rn(v[0]); return; }
  uint32_t w[4];
  for (int i = 0; i < n / 2; ++i) {
    __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
    w[i] = *reinterpret_cast<uint32_t*>(&h);
  }
  if (n == 2) { *reinterpret_cast<uint32_t*>(p) = w[0]; return; }
  if (n == 4) { *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]); return; }
  *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
}

// ============================================================================
// epilogue: deterministic slice reduction + tail + correction + per-row scale
// ============================================================================
struct TailVals {
  float v[16];
};

__global__ void fused_finish_kernel(const float* __restrict__ partial,
                                    const float* __restrict__ corr, int S, int64_t m, int64_t b,
                                    int64_t k, int d, const uint16_t* __restrict__ tailp,
                                    TailVals vals, const void* x, int x_dtype,
                                    int scale_mode, const void* q, int q_dtype, void* y,
                                    int y_dtype) {
  const int64_t nb = k / d;
  const int tail = (int)(k - nb * d);
  const int64_t total = m * b;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t / b, c = t - i * b;
    float s = 0.f;
    for (int sl = 0; sl < S; ++sl) s += partial[(int64_t)sl * total + t];
    if (corr)
      for (int sl = 0; sl < S; ++sl) s += corr[(int64_t)sl * b + c];
    if (tail) {
      uint32_t tc = tailp[i];
      for (int u = 0; u < tail; ++u)
        s = fmaf(vals.v[(tc >> (4 * u)) & 0xF], load_as<float>(x, x_dtype, (nb * d + u) * b + c), s);
    }
    if (scale_mode == MSG_SCALE_PER_ROW) s *= load_as<float>(q, q_dtype, i);
    store_as<float>(y, y_dtype, t, s);
  }
}

// ============================================================================
// host planning / dispatch
// ============================================================================
struct FusedPlan {
  bool ok;
  int bc, rpt, ql, S, nrow_blocks, ncol_tiles, quads_per_slice;
  bool sym, f32_entries;
  int64_t smem, partial_bytes, corr_bytes;
  QuadLayout L;
};

static bool codebook_antisymmetric(const double* v, int n, double* beta) {
  double twob = v[0] + v[n - 1];
  for (int c = 0; c < n; ++c)
    if (v[c] + v[c ^ (n - 1)] != twob) return false;
  *beta = twob / 2;
  return true;
}

static bool fused_eligible(int width, int x_dtype, int d, int scale_mode) {
  return width == 4 && (x_dtype == MSG_F16 || x_dtype == MSG_F32) && d >= 1 && d <= 3 &&
         scale_mode != MSG_SCALE_PER_GROUP;
}

static FusedPlan fused_plan(int64_t m, int64_t k, int width, const double* values, int x_dtype,
                            int64_t b, int d, int scale_mode, int flags) {
  FusedPlan p{};
  p.ok = false;
  if (flags & MSG_FLAG_FORCE_GENERIC) return p;
  if (!fused_eligible(width, x_dtype, d, scale_mode)) return p;
  if (m <= 0 || b <= 0 || k / d == 0) return p;
  double beta = 0;
  p.sym = !(flags & MSG_FLAG_NO_SYMMETRY) && codebook_antisymmetric(values, 16, &beta);
  p.f32_entries = (x_dtype == MSG_F32) || (flags & MSG_FLAG_F32_ENTRIES);
  const int esize = p.f32_entries ? 4 : 2;
  const int64_t ES = p.sym ? (1 << (4 * d - 1)) : (1 << (4 * d));
  const int64_t budget = std::min<int64_t>(max_smem_optin(), 227 * 1024) - 8 * 1024;
  int bc = b >= 8 ? 8 : (b >= 4 ? 4 : (b >= 2 ? 2 : 1));
  if (b == 3) bc = 4;
  if (b > 4 && b < 8) bc = 8;
  // shrink the column tile until one quad of tables fits
  while (bc > 1 && 4 * ES * bc * esize > budget) bc /= 2;
  if (4 * ES * bc * esize > budget) return p;
  p.bc = bc;
  p.rpt = bc == 8 ? 16 : 32;
  p.L = quad_layout(m, k, d);
  const int64_t quad_bytes = 4 * ES * bc * esize + 4 * d * bc * 4;  // tables + staged x
  p.nrow_blocks = (int)ceil_div(m, (int64_t)kThreads * p.rpt);
  p.ncol_tiles = (int)ceil_div(b, bc);
  const int64_t base = (int64_t)p.nrow_blocks * p.ncol_tiles;
  int64_t S = std::max<int64_t>(1, sm_count() / std::max<int64_t>(1, base));
  S = std::min<int64_t>(S, p.L.nq);
  p.quads_per_slice = (int)ceil_div(p.L.nq, S);
  p.S = (int)ceil_div(p.L.nq, p.quads_per_slice);
  p.ql = (int)std::max<int64_t>(1, std::min<int64_t>(budget / quad_bytes, p.quads_per_slice));
  p.smem = p.ql * quad_bytes;
  p.partial_bytes = align256((int64_t)p.S * m * b * 4);
  p.corr_bytes = align256((int64_t)p.S * b * 4);
  p.ok = true;
  return p;
}

template <int D, typename XT, typename ET, int BC, bool SYM, int RPT>
static int launch_fused_t(const FusedPlan& pl, FusedParams& P, cudaStream_t s) {
  auto kern = fused_lut_kernel<D, XT, ET, BC, SYM, RPT>;
  static int configured_dev = -1;  // one attribute call per instantiation and device
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    MSG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        std::min(max_smem_optin(), 227 * 1024)));
    configured_dev = dev;
  }
  dim3 grid(pl.nrow_blocks, pl.S, pl.ncol_tiles);
  kern<<<grid, kThreads, pl.smem, s>>>(P);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

template <int D, typename XT, typename ET, bool SYM>
static int launch_fused_bc(const FusedPlan& pl, FusedParams& P, cudaStream_t s) {
  switch (pl.bc) {
    case 1: return launch_fused_t<D, XT, ET, 1, SYM, 32>(pl, P, s);
    case 2: return launch_fused_t<D, XT, ET, 2, SYM, 32>(pl, P, s);
    case 4: return launch_fused_t<D, XT, ET, 4, SYM, 32>(pl, P, s);
    case 8: return launch_fused_t<D, XT, ET, 8, SYM, 16>(pl, P, s);
  }
  return fail(MSG_ERR_UNSUPPORTED, "bad column tile %d", pl.bc);
}

template <int D, typename XT>
static int launch_fused_xt(const FusedPlan& pl, FusedParams& P, cudaStream_t s) {
  if (pl.f32_entries)
    return pl.sym ? launch_fused_bc<D, XT, float, true>(pl, P, s)
                  : launch_fused_bc<D, XT, float, false>(pl, P, s);
  return pl.sym ? launch_fused_bc<D, XT, __half, true>(pl, P, s)
                : launch_fused_bc<D, XT, __half, false>(pl, P, s);
}

template <int D>
static int launch_fused_d(const FusedPlan& pl, FusedParams& P, int x_dtype, cudaStream_t s) {
  if (x_dtype == MSG_F16) return launch_fused_xt<D, __half>(pl, P, s);
  return launch_fused_xt<D, float>(pl, P, s);
}

}  // namespace msg

using namespace msg;

extern "C" {

int64_t msg_repacked_bytes(int64_t m, int64_t k, int d, int layout) {
  if (layout == MSG_LAYOUT_NONE) return 0;
  if (layout != MSG_LAYOUT_QUAD || d < 1 || d > 3) return -1;
  return quad_layout(m, k, d).total;
}

int msg_repack(const uint8_t* packed, int64_t m, int64_t k, int d, int layout, int symmetric,
               uint8_t* out, void* stream) {
  if (layout != MSG_LAYOUT_QUAD)
    return fail(MSG_ERR_UNSUPPORTED, "unknown weight layout %d", layout);
  if (d < 1 || d > 3) return fail(MSG_ERR_UNSUPPORTED, "quad layout supports d in 1..3, got %d", d);
  QuadLayout L = quad_layout(m, k, d);
  int64_t total = L.nq * m;
  if (total == 0 && !(L.tail && m)) return MSG_OK;
  int64_t n = std::max<int64_t>(total, 1);
  int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)sm_count() * 16);
  if (total == 0) {
    // k < d: only a tail plane; handled by a degenerate launch over rows
    return fail(MSG_ERR_UNSUPPORTED, "quad layout needs at least one full group");
  }
  repack_quad_kernel<<<grid, 256, 0, as_stream(stream)>>>(packed, m, k, d, row_bytes(k, 4),
                                                         symmetric, L, out);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

static int validate_gemm(int64_t m, int64_t k, int width, int x_dtype, int64_t b, int d,
                         int scale_mode, int64_t group_size) {
  if (m < 0 || k < 0 || b < 0) return fail(MSG_ERR_VALUE, "matrix dimensions must be non-negative");
  if (d < 1) return fail(MSG_ERR_VALUE, "depth d must be >= 1");
  if (scale_mode == MSG_SCALE_PER_GROUP && (group_size < d || group_size % d != 0))
    return fail(MSG_ERR_VALUE,
                "per-group scaling needs group_size >= d and divisible by d; got group_size=%lld, d=%d",
                (long long)group_size, d);
  if (width < 2 || width > 8) return fail(MSG_ERR_VALUE, "width must be in 2..8, got %d", width);
  if (d * width > 32)
    return fail(MSG_ERR_VALUE, "d*width = %d exceeds 32-bit index limit", d * width);
  if (d * width > 28)
    return fail(MSG_ERR_UNSUPPORTED,
                "GPU tables are limited to 2^28 entries per block (d*width=%d)", d * width);
  if (dtype_size(x_dtype) == 0 || x_dtype == MSG_BF16)
    return fail(MSG_ERR_UNSUPPORTED, "activation dtype %d is not supported on the GPU path",
                x_dtype);
  return MSG_OK;
}

int msg_gemm_plan(int64_t m, int64_t k, int width, const double* values, int x_dtype, int64_t b,
                  int d, int scale_mode, int64_t group_size, int flags, int* layout_out,
                  int* symmetric_out, int64_t* ws_out) {
  if (int e = validate_gemm(m, k, width, x_dtype, b, d, scale_mode, group_size)) return e;
  FusedPlan p = fused_plan(m, k, width, values, x_dtype, b, d, scale_mode, flags);
  if (p.ok) {
    *layout_out = MSG_LAYOUT_QUAD;
    *symmetric_out = p.sym ? 1 : 0;
    *ws_out = p.partial_bytes + p.corr_bytes;
  } else {
    *layout_out = MSG_LAYOUT_NONE;
    *symmetric_out = 0;
    *ws_out = generic_workspace_bytes(m, k, width, x_dtype, b, d);
  }
  return MSG_OK;
}

int msg_gemm(const uint8_t* packed, const uint8_t* wrep, int64_t m, int64_t k, int width,
             const double* values, const void* x, int x_dtype, int64_t b, int d, int scale_mode,
             int64_t group_size, const void* q, int q_dtype, void* y, int y_dtype,
             void* workspace, int64_t ws_bytes, int flags, void* stream) {
  if (int e = validate_gemm(m, k, width, x_dtype, b, d, scale_mode, group_size)) return e;
  if (dtype_size(y_dtype) == 0) return fail(MSG_ERR_UNSUPPORTED, "bad output dtype %d", y_dtype);
  cudaStream_t s = as_stream(stream);
  CodebookParam cb = make_codebook(values, width);
  FusedPlan p = fused_plan(m, k, width, values, x_dtype, b, d, scale_mode, flags);
  if (!p.ok)
    return run_generic(packed, m, k, width, cb, x, x_dtype, b, d, scale_mode, group_size, q,
                       q_dtype, y, y_dtype, workspace, ws_bytes, s);
  if (!wrep) return fail(MSG_ERR_VALUE, "fused path needs the repacked (quad) weight layout");
  if (ws_bytes < p.partial_bytes + p.corr_bytes)
    return fail(MSG_ERR_WORKSPACE, "workspace too small: need %lld bytes",
                (long long)(p.partial_bytes + p.corr_bytes));
  double beta = 0;
  if (p.sym) codebook_antisymmetric(values, 16, &beta);
  FusedParams P{};
  P.wrep = wrep;
  P.lo_off = p.L.lo_off;
  P.hi_off = p.L.hi_off;
  P.m = m;
  P.nb = p.L.nb;
  P.nq = p.L.nq;
  P.x = x;
  P.b = b;
  P.d = d;
  for (int c = 0; c < 16; ++c) P.s[c] = (float)(values[c] - beta);
  P.beta = (float)beta;
  P.quads_per_slice = p.quads_per_slice;
  P.ql = p.ql;
  P.partial = reinterpret_cast<float*>(workspace);
  P.corr = reinterpret_cast<float*>((char*)workspace + p.partial_bytes);
  int e = MSG_OK;
  switch (d) {
    case 1: e = launch_fused_d<1>(p, P, x_dtype, s); break;
    case 2: e = launch_fused_d<2>(p, P, x_dtype, s); break;
    case 3: e = launch_fused_d<3>(p, P, x_dtype, s); break;
  }
  if (e) return e;
  if (flags & MSG_FLAG_LUT_PHASE_ONLY) return MSG_OK;
  TailVals tv;
  for (int c = 0; c < 16; ++c) tv.v[c] = (float)values[c];
  const int64_t total = m * b;
  const int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)sm_count() * 8);
  const uint16_t* tailp =
      p.L.tail ? reinterpret_cast<const uint16_t*>(wrep + p.L.tail_off) : nullptr;
  fused_finish_kernel<<<grid, 256, 0, s>>>(P.partial, p.sym ? P.corr : nullptr, p.S, m, b, k, d,
                                           tailp, tv, x, x_dtype, scale_mode, q, q_dtype, y,
                                           y_dtype);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

}  // extern "C"
