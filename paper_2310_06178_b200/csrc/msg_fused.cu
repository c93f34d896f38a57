// K3 (weight repack) and K1+K2 fused shared-memory LUT kernel for msGeMM.
//
// Reference semantics: gemm.py:89-153 (msgemm), gemm.py:70-86 (the column
// reduction, k%d tail, per-row scale), lut.py:59-72 (table entries),
// packing.py:201-228 (group index: first code least significant).
//
// Design (sm_100a, one 256-thread CTA per SM):
//   * K3 repacks the reference's row-major nibbles (packing.py:99-114) into
//     "quad planes": for every 4 consecutive d-groups and every row, a 32-bit
//     word of low index bytes (d=2,3; 16 bits for d=1) and, for d=3, a 16-bit
//     word of high index nibbles.  Density stays 4*d bits per group.  Plane
//     rows are padded to a multiple of 8 so a row block of a quad is one
//     16-byte-aligned contiguous span -> one TMA bulk copy.  For
//     antisymmetric codebooks (v[c] + v[~c] = 2*beta, e.g. two's-complement
//     int4 with beta = -1/2) K3 folds the sign symmetry into the stored index:
//     an index with the top bit set is stored complemented, plus a sign bit,
//     so tables hold only 2^(4d-1) entries and
//         L(idx) = +-H[f] + beta * (x_0 + .. + x_{d-1}).
//   * The fused kernel gives each CTA a block of R = 256*RPT rows, a k-slice
//     of quads and a tile of BC batch columns.  Per round it builds the
//     tables of QL quads (4*QL groups x ES entries x BC columns, batch
//     innermost so one vector LDS fetches all BC columns of an entry) into
//     shared memory and every thread gathers for its RPT rows, accumulating
//     fp32 in registers with packed FFMA2.  The weight words of round t+1 are
//     brought in by cp.async.bulk (TMA bulk copy) into a double-buffered
//     staging area while round t builds and gathers; the activations of round
//     t+1 are prefetched into registers.  Tables are built once per (row
//     block, k-slice) and amortised over R rows.
//   * k-slice partials go to a workspace [S][m][b] (fp32) and a second,
//     deterministic pass sums them in slice order, adds the k%d tail, the
//     symmetry correction and the per-row scale, and casts to Y's dtype.
#include <algorithm>
#include <cstring>

#include <cstdlib>

#include "msg_common.cuh"

namespace msg {

int run_generic(const uint8_t* packed, int64_t m, int64_t k, int width, const CodebookParam& cb,
                const void* x, int x_dtype, int64_t b, int d, int scale_mode, int64_t group_size,
                const void* q, int q_dtype, void* y, int y_dtype, void* ws, int64_t ws_bytes,
                cudaStream_t s);
int64_t generic_workspace_bytes(int64_t m, int64_t k, int width, int x_dtype, int64_t b, int d);
// b = 1 GEMV kernel (msg_lane.cu)
bool lane_eligible(int width, const double* values, double beta, int64_t k, int x_dtype,
                   int64_t b, int d, int scale_mode, bool sym, bool f32_entries);
int64_t lane_layout_bytes(int64_t m, int64_t k);
int64_t lane_workspace_bytes(int64_t m, int64_t k);
int lane_repack(const uint8_t* packed, int64_t m, int64_t k, uint8_t* out, cudaStream_t s);
int launch_lane(const uint8_t* wrep, int64_t m, int64_t k, const double* values, double beta,
                const void* x, int scale_mode, const void* q, int q_dtype, void* y, int y_dtype,
                void* ws, int64_t ws_bytes, bool early, bool lut_only, cudaStream_t s);
// batched d = 3 row-block kernel (msg_rowblock.cu)
struct TailVals;
int rb_group_count(int64_t b);
bool rb_eligible(int width, int x_dtype, int64_t b, int d, int scale_mode, bool sym,
                 bool f32_entries, bool s_exact16);
int64_t rb_layout_bytes(int64_t m, int64_t k, int G, int rpt);
int64_t rb_workspace_bytes(int64_t m, int64_t k, int64_t b, int rpt);
int rb_choose_rpt(int64_t m, int64_t b, int flags);
int rb_repack(const uint8_t* packed, int64_t m, int64_t k, int G, int rpt, uint8_t* out,
              cudaStream_t s);
int launch_rb(const uint8_t* wrep, int64_t m, int64_t k, const double* values, double beta,
              const void* x, int64_t b, int scale_mode, const void* q, int q_dtype, void* y,
              int y_dtype, void* ws, int64_t ws_bytes, bool early, bool lut_only,
              const TailVals& tv, int rpt, cudaStream_t s);
static int rb_layout_rpt(int layout) { return layout == MSG_LAYOUT_RB4S ? 8 : 16; }
static int rb_layout_groups(int layout) {
  return (layout == MSG_LAYOUT_RB4 || layout == MSG_LAYOUT_RB4S) ? 4
         : layout == MSG_LAYOUT_RB8 ? 8 : layout == MSG_LAYOUT_RB16 ? 16 : 0;
}

static inline int64_t align256(int64_t v) { return (v + 255) / 256 * 256; }

// ============================================================================
// K3: quad-plane repack
// ============================================================================
struct QuadLayout {
  int64_t nb, nq, tail, mp;  // mp: plane row stride (m rounded up to 8)
  int64_t lo_off, hi_off, tail_off, total;
  int lo_bytes;  // 4 for d=2,3 ; 2 for d=1
  bool has_hi;
};

static QuadLayout quad_layout(int64_t m, int64_t k, int d) {
  QuadLayout L{};
  L.nb = k / d;
  L.nq = (L.nb + 3) / 4;
  L.tail = k - L.nb * d;
  L.mp = (m + 7) / 8 * 8;
  L.lo_bytes = d == 1 ? 2 : 4;
  L.has_hi = d == 3;
  L.lo_off = 0;
  L.hi_off = align256(L.nq * L.mp * L.lo_bytes);
  L.tail_off = L.hi_off + (L.has_hi ? align256(L.nq * L.mp * 2) : 0);
  L.total = L.tail_off + (L.tail ? align256(m * 2) : 0);
  if (L.total == 0) L.total = 256;
  return L;
}

__device__ __forceinline__ uint32_t nib(const uint8_t* row, int64_t j) {
  return (row[j >> 1] >> ((j & 1) * 4)) & 0xF;
}

// One CTA per (32 rows, 16 quads): the tile's packed bytes (2d per quad and
// row) are staged with coalesced loads, then each thread forms (row, quad)
// records and writes them to the [quad][row] planes (consecutive rows ->
// coalesced stores).  Position g of row i holds group (g + i) % 4 of the quad
// (a warp's lanes hit 4 different tables at every step).
constexpr int kQrRows = 32, kQrQuads = 16;
__global__ void __launch_bounds__(256) repack_quad_kernel(const uint8_t* __restrict__ packed,
                                                          int64_t m, int64_t k, int d, int rb,
                                                          int symmetric, QuadLayout L,
                                                          uint8_t* __restrict__ out) {
  __shared__ uint8_t tile[kQrRows][kQrQuads * 6 + 4];
  const int bits = 4 * d, qb = 2 * d;  // bits per group, bytes per quad
  const uint32_t emask = (1u << bits) - 1;
  const uint32_t top = 1u << (bits - 1);
  const int64_t ntr = (L.mp + kQrRows - 1) / kQrRows, ntq = (L.nq + kQrQuads - 1) / kQrQuads;
  for (int64_t tt = blockIdx.x; tt < ntr * ntq; tt += gridDim.x) {
    const int64_t i0 = (tt % ntr) * kQrRows, q0 = (tt / ntr) * kQrQuads;
    const int64_t b0 = q0 * qb;
    const int tb = kQrQuads * qb;  // bytes per tile row
    __syncthreads();
    for (int e = threadIdx.x; e < kQrRows * tb; e += 256) {
      const int r = e / tb, c = e % tb;
      const int64_t i = i0 + r, by = b0 + c;
      tile[r][c] = (i < m && by < rb) ? __ldg(packed + i * rb + by) : 0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kQrRows * kQrQuads; e += 256) {
      const int r = e % kQrRows, qq = e / kQrRows;
      const int64_t i = i0 + r, q = q0 + qq;
      if (i >= L.mp || q >= L.nq) continue;
      uint32_t lo = 0, hi = 0;
      if (i < m) {
        for (int g = 0; g < 4; ++g) {
          const int gi = (int)((g + i) & 3);
          const int64_t j = q * 4 + gi;
          uint32_t st = 0;
          if (j < L.nb) {
            uint32_t idx = 0;
            for (int r2 = 0; r2 < d; ++r2) {
              const int cd = qq * 4 * d + gi * d + r2;  // code inside the tile row
              idx |= ((tile[r][cd >> 1] >> ((cd & 1) * 4)) & 0xF) << (4 * r2);
            }
            if (symmetric && (idx & top)) idx = (idx ^ emask) | top;  // complement + sign bit
            st = idx;
          }
          if (d == 1) lo |= st << (4 * g);
          else if (d == 2) lo |= st << (8 * g);
          else { lo |= (st & 0xFF) << (8 * g); hi |= (st >> 8) << (4 * g); }
        }
        if (L.tail && q == 0) {
          const uint8_t* row = packed + i * rb;
          uint32_t tc = 0;
          for (int64_t j = L.nb * d; j < k; ++j) tc |= nib(row, j) << (4 * (j - L.nb * d));
          reinterpret_cast<uint16_t*>(out + L.tail_off)[i] = (uint16_t)tc;
        }
      }
      const int64_t t = q * L.mp + i;
      if (d == 1) reinterpret_cast<uint16_t*>(out + L.lo_off)[t] = (uint16_t)lo;
      else reinterpret_cast<uint32_t*>(out + L.lo_off)[t] = lo;
      if (L.has_hi) reinterpret_cast<uint16_t*>(out + L.hi_off)[t] = (uint16_t)hi;
    }
  }
}

// ============================================================================
// async-copy and packed-math helpers (PTX)
// ============================================================================
// a0,a1 += x0*s, x1*s  (one FFMA2)
__device__ __forceinline__ void ffma2(float& a0, float& a1, float x0, float x1, float s) {
  unsigned long long acc, xv, sv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(xv) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(sv) : "f"(s));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(xv), "l"(sv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc));
}
// e0,e1 = s*x0 + b0, s*x1 + b1
__device__ __forceinline__ void fma2_to(float& e0, float& e1, float s, float x0, float x1,
                                        float b0, float b1) {
  unsigned long long acc, xv, sv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(b0), "f"(b1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(xv) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(sv) : "f"(s));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(xv), "l"(sv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(e0), "=f"(e1) : "l"(acc));
}

// ============================================================================
// fused LUT kernel
// ============================================================================
constexpr int kThreads = 256;

struct FusedParams {
  const uint8_t* wrep;
  int64_t lo_off, hi_off, mp;
  int64_t m, nb, nq;
  const void* x;  // (k, b) row-major, F16 or F32
  int64_t b;
  float s[16];  // per-code value used in tables: v[c] - beta (symmetric) or v[c]
  float beta;
  int s_exact16;        // every s[c] is exact in fp16 (fp16x2 table build allowed)
  int early;            // MSG_FLAG_STATIC_WEIGHTS: first weight copy before griddepcontrol.wait
  int quads_per_slice;  // k-slice length in quads
  int ql;               // quads per table round
  float* partial;       // [S][m][b]
};

template <typename XT> __device__ __forceinline__ float ldx(const void* p, int64_t i);
template <> __device__ __forceinline__ float ldx<float>(const void* p, int64_t i) {
  return __ldg(reinterpret_cast<const float*>(p) + i);
}
template <> __device__ __forceinline__ float ldx<__half>(const void* p, int64_t i) {
  return __half2float(reinterpret_cast<const __half*>(p)[i]);
}

__device__ __forceinline__ float h2f_lo(uint32_t w) {
  return __half2float(__ushort_as_half((unsigned short)(w & 0xFFFF)));
}
__device__ __forceinline__ float h2f_hi(uint32_t w) {
  return __half2float(__ushort_as_half((unsigned short)(w >> 16)));
}

// acc += h * s16 with h, s16 fp16 and acc fp32 (sm_100 FHFMA: one instruction,
// no separate f16->f32 conversion; the product is exact, one fp32 rounding)
__device__ __forceinline__ void fhfma(float& acc, unsigned short h, unsigned short s16) {
  asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(h), "h"(s16));
}
__device__ __forceinline__ void fhfma2w(float& a0, float& a1, uint32_t w, unsigned short s16) {
  unsigned short h0, h1;
  asm("mov.b32 {%0, %1}, %2;" : "=h"(h0), "=h"(h1) : "r"(w));
  fhfma(a0, h0, s16);
  fhfma(a1, h1, s16);
}

// acc[0..BC) += sign * entry (BC values of type ET at p); the sign is bit
// SBIT of the stored index st (symmetric tables) or +1.
template <typename ET, int BC, bool SYM, int SBIT>
__device__ __forceinline__ void gather_acc(const uint8_t* p, uint32_t st, float* acc) {
  if constexpr (sizeof(ET) == 2) {
    unsigned short s16 = 0x3C00;  // +1.0h
    if constexpr (SYM) s16 = (unsigned short)(0x3C00 | ((st >> SBIT) << 15));
    if constexpr (BC == 1) {
      fhfma(acc[0], *reinterpret_cast<const unsigned short*>(p), s16);
    } else if constexpr (BC == 2) {
      fhfma2w(acc[0], acc[1], *reinterpret_cast<const uint32_t*>(p), s16);
    } else if constexpr (BC == 4) {
      uint2 v = *reinterpret_cast<const uint2*>(p);
      fhfma2w(acc[0], acc[1], v.x, s16);
      fhfma2w(acc[2], acc[3], v.y, s16);
    } else {
      uint4 v = *reinterpret_cast<const uint4*>(p);
      fhfma2w(acc[0], acc[1], v.x, s16);
      fhfma2w(acc[2], acc[3], v.y, s16);
      fhfma2w(acc[4], acc[5], v.z, s16);
      fhfma2w(acc[6], acc[7], v.w, s16);
    }
  } else {
    float sg = 1.f;
    if constexpr (SYM) sg = ((st >> SBIT) & 1) ? -1.f : 1.f;
    if constexpr (BC == 1) {
      acc[0] = fmaf(sg, *reinterpret_cast<const float*>(p), acc[0]);
    } else if constexpr (BC == 2) {
      float2 v = *reinterpret_cast<const float2*>(p);
      ffma2(acc[0], acc[1], v.x, v.y, sg);
    } else {
#pragma unroll
      for (int i = 0; i < BC / 4; ++i) {
        float4 v = reinterpret_cast<const float4*>(p)[i];
        ffma2(acc[4 * i], acc[4 * i + 1], v.x, v.y, sg);
        ffma2(acc[4 * i + 2], acc[4 * i + 3], v.z, v.w, sg);
      }
    }
  }
}

template <typename ET, int BC> __device__ __forceinline__ void store_entry(uint8_t* p, const float* v) {
  if constexpr (sizeof(ET) == 4) {
    if constexpr (BC == 1) *reinterpret_cast<float*>(p) = v[0];
    else if constexpr (BC == 2) *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    else
#pragma unroll
      for (int i = 0; i < BC / 4; ++i)
        reinterpret_cast<float4*>(p)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  } else {
    if constexpr (BC == 1) {
      *reinterpret_cast<__half*>(p) = __float2half_rn(v[0]);
    } else {
      uint32_t w[BC / 2];
#pragma unroll
      for (int i = 0; i < BC / 2; ++i) {
        __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
        w[i] = *reinterpret_cast<uint32_t*>(&h);
      }
      if constexpr (BC == 2) *reinterpret_cast<uint32_t*>(p) = w[0];
      else if constexpr (BC == 4) *reinterpret_cast<uint2*>(p) = make_uint2(w[0], w[1]);
      else *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

// stored index of group g (0..3) from the quad words
template <int D>
__device__ __forceinline__ uint32_t stored_index(uint32_t lo, uint32_t hi, int g) {
  if constexpr (D == 1) return (lo >> (4 * g)) & 0xF;
  else if constexpr (D == 2) return (lo >> (8 * g)) & 0xFF;
  else return ((lo >> (8 * g)) & 0xFF) | (((hi >> (4 * g)) & 0xF) << 8);
}

// Table layout: the 4 tables of a quad are interleaved in 128-byte rows, each
// group owning a 32-byte slice (= 8 banks) of every row; entry f of group g
// sits at row f / SPG, slot f % SPG of that slice.  Lanes reading different
// groups therefore never share a bank.
template <int EB> struct TabLayout {
  static constexpr int SPG = 32 / EB;  // entries per group per 128-byte row
  static constexpr int LSPG = SPG == 1 ? 0 : SPG == 2 ? 1 : SPG == 4 ? 2 : SPG == 8 ? 3 : 4;
  static constexpr int LEB = EB == 2 ? 1 : EB == 4 ? 2 : EB == 8 ? 3 : EB == 16 ? 4 : 5;
  static __device__ __forceinline__ uint32_t off(uint32_t f, uint32_t gslot) {
    return ((f >> LSPG) << 7) | ((f & (SPG - 1)) << LEB) | gslot;
  }
};

template <int D> struct FusedShape {
  static constexpr int LOB = D == 1 ? 2 : 4;   // lo plane bytes per (quad,row)
  static constexpr int HIB = D == 3 ? 2 : 0;   // hi plane bytes per (quad,row)
};

template <int D, typename XT, typename ET, int BC, bool SYM, int RPT, int NT>
__global__ void __launch_bounds__(NT, 1) fused_lut_kernel(FusedParams P) {
  constexpr int ES = SYM ? (1 << (4 * D - 1)) : (1 << (4 * D));  // stored entries per group
  constexpr int EB = BC * (int)sizeof(ET);                        // bytes per entry
  constexpr int LOWN = D == 1 ? 1 : (D == 2 ? 16 : 256);          // combos of the low D-1 codes
  constexpr int HIN = SYM ? 8 : 16;                               // values of the top code
  constexpr int R = NT * RPT;
  constexpr int LOB = FusedShape<D>::LOB, HIB = FusedShape<D>::HIB;
  constexpr int XPT = 2;  // staged activation values per thread (<= 512 per round)
  constexpr int QUADB = 4 * ES * EB > 128 ? 4 * ES * EB : 128;  // table bytes per quad
  using TL = TabLayout<EB>;
  extern __shared__ __align__(128) uint8_t smem[];

  const int tid = threadIdx.x;
  const int64_t row0 = (int64_t)blockIdx.x * R;
  const int slice = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.z * BC;
  const int64_t q_begin = (int64_t)slice * P.quads_per_slice;
  const int64_t q_end = P.nq < q_begin + P.quads_per_slice ? P.nq : q_begin + P.quads_per_slice;
  const int rows_valid = (int)((P.m - row0) < R ? (P.m - row0) : R);
  const int rows_cp = (rows_valid + 7) & ~7;
  const int QL = P.ql;

  // ---- shared-memory carve-up
  uint8_t* tab = smem;                                                   // [QL*4][ES][BC] ET
  uint8_t* stage = tab + (size_t)QL * QUADB;                             // [2][QL][R] lo,hi
  const size_t stage_bytes = (size_t)QL * R * (LOB + HIB);
  constexpr int XN_MAX = 2 * NT;  // staged activations per round (QL*4*D*BC <= 2 NT)
  const int XN = QL * 4 * D * BC;
  float* xs0 = reinterpret_cast<float*>(stage + 2 * stage_bytes);       // [2][XN]
  uint64_t* bars = reinterpret_cast<uint64_t*>(xs0 + 2 * XN);           // [2]

  const uint8_t* lo_plane = P.wrep + P.lo_off;
  const uint8_t* hi_plane = P.wrep + P.hi_off;
  const int nrounds = (int)((q_end - q_begin + QL - 1) / QL);

  auto issue = [&](int t) {  // TMA bulk copies of round t's weight words (one thread)
    const int64_t qa = q_begin + (int64_t)t * QL;
    const int nql = (int)((q_end - qa) < QL ? (q_end - qa) : QL);
    uint8_t* buf = stage + (t & 1) * stage_bytes;
    uint64_t* bar = bars + (t & 1);
    fence_proxy_async();
    mbar_expect_tx(bar, (uint32_t)(nql * rows_cp * (LOB + HIB)));
    for (int qq = 0; qq < nql; ++qq) {
      const int64_t q = qa + qq;
      bulk_g2s(buf + (size_t)qq * R * LOB, lo_plane + (q * P.mp + row0) * LOB,
               (uint32_t)(rows_cp * LOB), bar);
      if constexpr (HIB > 0)
        bulk_g2s(buf + (size_t)QL * R * LOB + (size_t)qq * R * HIB,
                 hi_plane + (q * P.mp + row0) * HIB, (uint32_t)(rows_cp * HIB), bar);
    }
  };
  // activations of round t: element e -> (group row gr = e / BC, column c = e % BC)
  auto load_x = [&](int t, float (&xv)[XPT]) {
    const int64_t qa = q_begin + (int64_t)t * QL;
    const int64_t g_first = qa * 4;
    const int64_t qe = (qa + QL) < q_end ? (qa + QL) : q_end;
    const int64_t glast = (qe * 4) < P.nb ? qe * 4 : P.nb;
    const int nel = (int)(glast - g_first) * D * BC;
#pragma unroll
    for (int u = 0; u < XPT; ++u) {
      const int e = tid + u * NT;
      float v = 0.f;
      if (e < nel) {
        const int c = e % BC, gr = e / BC;
        if (c0 + c < P.b) v = ldx<XT>(P.x, (g_first * D + gr) * P.b + c0 + c);
      }
      xv[u] = v;
    }
  };

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  MSG_JITTER();
  __syncthreads();
  // Launched with PDL: the first weight copy may start before the wait only if
  // the preceding kernel did not write the repacked weights; x is read and the
  // partials are written only after it.  The finishing kernel may queue now.
  if (tid == 0 && nrounds > 0 && P.early) issue(0);
  griddep_wait();
  griddep_launch_dependents();
  if (tid == 0 && nrounds > 0 && !P.early) issue(0);
  // activations, double-buffered one round ahead: round t reads xs0[t & 1],
  // written during round t - 1 (or here), so no barrier sits between the
  // staging and the build
  float xnext[XPT];
  if (nrounds > 0) {
    load_x(0, xnext);
#pragma unroll
    for (int u = 0; u < XPT; ++u)
      if (tid + u * NT < XN) xs0[tid + u * NT] = xnext[u];
  }
  if (nrounds > 1) load_x(1, xnext);
  static_assert(XPT * NT >= XN_MAX, "staging capacity");

  float acc[RPT][BC];
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int c = 0; c < BC; ++c) acc[r][c] = 0.f;
  float corr = 0.f;  // thread tid < BC accumulates column tid's correction

  float sv[HIN];
#pragma unroll
  for (int h = 0; h < HIN; ++h) sv[h] = P.s[h];
  uint32_t gslot[4];  // table slice of the group at quad position g for this lane
#pragma unroll
  for (int g = 0; g < 4; ++g) gslot[g] = (uint32_t)((g + tid) & 3) << 5;

  for (int t = 0; t < nrounds; ++t) {
    const int64_t qa = q_begin + (int64_t)t * QL;
    const int nql = (int)((q_end - qa) < QL ? (q_end - qa) : QL);
    const int64_t g_first = qa * 4;
    const int ngroups = (int)((int64_t)nql * 4 < P.nb - g_first ? (int64_t)nql * 4 : P.nb - g_first);

    MSG_JITTER();
    __syncthreads();  // round t-1 finished with tab, xs0[(t+1)&1] and stage[(t+1)&1]
    if (tid == 0 && t + 1 < nrounds) issue(t + 1);
    float* xs = xs0 + (t & 1) * XN;
    if (t + 1 < nrounds) {
#pragma unroll
      for (int u = 0; u < XPT; ++u)
        if (tid + u * NT < XN) xs0[((t + 1) & 1) * XN + tid + u * NT] = xnext[u];
    }
    if (t + 2 < nrounds) load_x(t + 2, xnext);
    if (SYM && tid < BC) {
      float sacc = 0.f;
      for (int gr = 0; gr < ngroups * D; ++gr) sacc += xs[gr * BC + tid];
      corr += sacc;
    }
    // ---- build: entry(f) = sum_r s[nibble_r(f)] * x_r, top nibble < HIN.
    // Work item w -> (quad, group g = w % 4, low = (w / 4) % LOWN): the lanes of
    // one store wavefront fill one whole 128-byte table row (4 groups x SPG
    // consecutive entries), so the interleaved layout is written conflict-free.
    for (int w = tid; w < nql * 4 * LOWN; w += NT) {
      const int qq = w / (4 * LOWN), rem = w - qq * 4 * LOWN;
      const int g = rem & 3, low = rem >> 2;
      const int gl = qq * 4 + g;
      if (gl >= ngroups) continue;
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
      float xtop[BC];
#pragma unroll
      for (int c = 0; c < BC; ++c) xtop[c] = xt[c];
      uint8_t* dst = tab + (size_t)qq * QUADB;
      const uint32_t gslot_b = (uint32_t)g << 5;
      if (sizeof(ET) == 2 && BC >= 2 && P.s_exact16) {
        // fp16 entries: the low-code part and the top-code term rounded to
        // fp16 once each, then one HFMA2 per column pair (entry = base + s_h x_top)
        constexpr int NP = BC >= 2 ? BC / 2 : 1;
        __half2 b2[NP], t2[NP];
#pragma unroll
        for (int c = 0; c < BC; c += 2) {
          b2[c / 2] = __floats2half2_rn(base[c], base[c + 1]);
          t2[c / 2] = __floats2half2_rn(xtop[c], xtop[c + 1]);
        }
#pragma unroll
        for (int h = 0; h < HIN; ++h) {
          const __half2 s2 = __float2half2_rn(sv[h]);  // codebook values are exact in fp16
          uint32_t wv[NP];
#pragma unroll
          for (int c = 0; c < BC / 2; ++c) {
            __half2 e2 = __hfma2(s2, t2[c], b2[c]);
            wv[c] = *reinterpret_cast<uint32_t*>(&e2);
          }
          uint8_t* p = dst + TL::off((uint32_t)(low + h * LOWN), gslot_b);
          if constexpr (BC == 2) *reinterpret_cast<uint32_t*>(p) = wv[0];
          else if constexpr (BC == 4) *reinterpret_cast<uint2*>(p) = make_uint2(wv[0], wv[1]);
          else *reinterpret_cast<uint4*>(p) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      } else {
#pragma unroll
        for (int h = 0; h < HIN; ++h) {
          float e[BC];
          if constexpr (BC == 1) {
            e[0] = fmaf(sv[h], xtop[0], base[0]);
          } else {
#pragma unroll
            for (int c = 0; c < BC; c += 2)
              fma2_to(e[c], e[c + 1], sv[h], xtop[c], xtop[c + 1], base[c], base[c + 1]);
          }
          store_entry<ET, BC>(dst + TL::off((uint32_t)(low + h * LOWN), gslot_b), e);
        }
      }
    }
    MSG_JITTER();
    __syncthreads();
    mbar_wait(&bars[t & 1], (uint32_t)((t >> 1) & 1));
    // ---- gather
    const uint8_t* buf = stage + (t & 1) * stage_bytes;
    for (int qq = 0; qq < nql; ++qq) {
      const uint8_t* lo_s = buf + (size_t)qq * R * LOB;
      const uint16_t* hi_s =
          reinterpret_cast<const uint16_t*>(buf + (size_t)QL * R * LOB + (size_t)qq * R * HIB);
      const uint8_t* tq = tab + (size_t)qq * QUADB;
      const int gcount = ngroups - qq * 4;
      if (gcount >= 4) {
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int li = r * NT + tid;
          if (li < rows_valid) {
            uint32_t lo, hi = 0;
            if constexpr (LOB == 4) lo = reinterpret_cast<const uint32_t*>(lo_s)[li];
            else lo = reinterpret_cast<const uint16_t*>(lo_s)[li];
            if constexpr (HIB > 0) hi = hi_s[li];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const uint32_t st = stored_index<D>(lo, hi, g);
              const uint32_t f = SYM ? (st & (ES - 1)) : st;
              gather_acc<ET, BC, SYM, 4 * D - 1>(tq + TL::off(f, gslot[g]), st, acc[r]);
            }
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
          const int li = r * NT + tid;
          if (li < rows_valid) {
            uint32_t lo, hi = 0;
            if constexpr (LOB == 4) lo = reinterpret_cast<const uint32_t*>(lo_s)[li];
            else lo = reinterpret_cast<const uint16_t*>(lo_s)[li];
            if constexpr (HIB > 0) hi = hi_s[li];
            for (int g = 0; g < 4; ++g) {
              if (((g + tid) & 3) >= gcount) continue;
              const uint32_t st = stored_index<D>(lo, hi, g);
              const uint32_t f = SYM ? (st & (ES - 1)) : st;
              gather_acc<ET, BC, SYM, 4 * D - 1>(tq + TL::off(f, gslot[g]), st, acc[r]);
            }
          }
        }
      }
    }
  }
  // ---- fold this slice's symmetry correction beta * sum(x) into every row
  if constexpr (SYM) {
    MSG_JITTER();
    __syncthreads();
    if (tid < BC) xs0[tid] = P.beta * corr;
    MSG_JITTER();
    __syncthreads();
    float cv[BC];
#pragma unroll
    for (int c = 0; c < BC; ++c) cv[c] = xs0[c];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
#pragma unroll
      for (int c = 0; c < BC; ++c) acc[r][c] += cv[c];
  }
  // ---- write partials [slice][i][c]
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const int li = r * NT + tid;
    if (li < rows_valid) {
      float* dst = P.partial + ((int64_t)slice * P.m + row0 + li) * P.b + c0;
      if (c0 + BC <= P.b && BC >= 2 && (P.b % 2 == 0)) {
#pragma unroll
        for (int c = 0; c < BC; c += 2)
          *reinterpret_cast<float2*>(dst + c) = make_float2(acc[r][c], acc[r][c + 1]);
      } else {
#pragma unroll
        for (int c = 0; c < BC; ++c)
          if (c0 + c < P.b) dst[c] = acc[r][c];
      }
    }
  }
}

// ============================================================================
// epilogue: deterministic slice reduction + tail + correction + per-row scale
// ============================================================================
struct TailVals {
  float v[16];
};

// A 256-thread block reduces 256/SG consecutive outputs: slice group g (of SG)
// sums slices g, g+SG, ... in order for each output (lanes = consecutive
// outputs, so every load is a coalesced 128-byte row), then the SG partial
// sums are combined in fixed order -- deterministic run to run.
template <int SG>
__global__ void __launch_bounds__(256) fused_finish_kernel(
    const float* __restrict__ partial, int S, int64_t m, int64_t b, int64_t k, int d,
    const uint16_t* __restrict__ tailp, TailVals vals, const void* x, int x_dtype, int scale_mode,
    const void* q, int q_dtype, void* y, int y_dtype, YFan fan) {
  constexpr int OPB = 256 / SG;  // outputs per block
  __shared__ float red[SG][OPB];
  const int64_t nb = k / d;
  const int tail = (int)(k - nb * d);  // < d <= 3 on the fused paths
  const int64_t total = m * b;
  const int og = threadIdx.x % OPB, sg = threadIdx.x / OPB;
  // Operands that do not depend on the partials (tail weights and activations,
  // per-row scale) are loaded before griddepcontrol.wait: the LUT kernel only
  // writes the partials, and x / wrep / q were final before it started.
  float tw[2] = {0.f, 0.f}, tx[2] = {0.f, 0.f}, qs = 1.f;
  auto extras = [&](int64_t t) {
    const int64_t i = t / b, c = t - i * b;
    if (tail) {
      const uint32_t tc = tailp[i];
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (u < tail) {
          tw[u] = vals.v[(tc >> (4 * u)) & 0xF];
          tx[u] = load_as<float>(x, x_dtype, (nb * d + u) * b + c);
        }
    }
    if (scale_mode == MSG_SCALE_PER_ROW) qs = load_as<float>(q, q_dtype, i);
  };
  {
    const int64_t t = (int64_t)blockIdx.x * OPB + og;
    if (t < total && sg == 0) extras(t);
  }
  // PDL: let the next kernel on the stream (e.g. the next layer's LUT kernel)
  // start its prologue now; then wait until the LUT kernel's partials are complete
  griddep_launch_dependents();
  griddep_wait();
  for (int64_t t0 = (int64_t)blockIdx.x * OPB; t0 < total; t0 += (int64_t)gridDim.x * OPB) {
    const int64_t t = t0 + og;
    float s = 0.f;
    if (t < total) {
      if (scale_mode == MSG_SCALE_PER_GROUP) {
        // slice sl is scale group sl: q is (m, S) row-major (packing.py:29-36)
        const int64_t qi = (t / b) * S;
#pragma unroll 4
        for (int sl = sg; sl < S; sl += SG)
          s = fmaf(load_as<float>(q, q_dtype, qi + sl), __ldcg(partial + (int64_t)sl * total + t), s);
      } else {
#pragma unroll 8
        for (int sl = sg; sl < S; sl += SG) s += __ldcg(partial + (int64_t)sl * total + t);
      }
    }
    if constexpr (SG > 1) {
      red[sg][og] = s;
      MSG_JITTER();
      __syncthreads();
      if (sg == 0) {
#pragma unroll
        for (int g = 1; g < SG; ++g) s += red[g][og];
      }
      MSG_JITTER();
      __syncthreads();
    }
    if (t < total && sg == 0) {
      if (t0 != (int64_t)blockIdx.x * OPB) extras(t);
#pragma unroll
      for (int u = 0; u < 2; ++u)
        if (u < tail) s = fmaf(tw[u], tx[u], s);
      if (scale_mode == MSG_SCALE_PER_ROW) s *= qs;
      store_as<float>(y, y_dtype, t, s);
      if (fan.n) {  // compile-time indices: a dynamic index would move the parameter block to local memory
#pragma unroll
        for (int pr = 0; pr < kMaxFan; ++pr)
          if (pr < fan.n) store_as<float>(fan.p[pr], y_dtype, t, s);
      }
    }
  }
}

// Four consecutive outputs of one row per thread group (b % 4 == 0): float4
// loads, slice group g (of SG) sums slices g, g+SG, ... in order, the SG
// partial sums are combined in fixed order through shared memory --
// deterministic run to run.  SG = 1 is the plain slice-order sum.
template <int SG>
__global__ void __launch_bounds__(256) finish_vec4_kernel(
    const float* __restrict__ partial, int S, int64_t m, int64_t b, int64_t k, int d,
    const uint16_t* __restrict__ tailp, TailVals vals, const void* x, int x_dtype, int scale_mode,
    const void* q, int q_dtype, void* y, int y_dtype, YFan fan) {
  constexpr int OPB = 256 / SG;  // float4 outputs per block
  __shared__ float4 red[SG > 1 ? SG : 1][OPB];
  const int64_t total = m * b, total4 = total / 4;
  const int64_t nb = k / d;
  const int tail = (int)(k - nb * d);
  const int og = threadIdx.x % OPB, sg = threadIdx.x / OPB;
  griddep_launch_dependents();
  griddep_wait();
  for (int64_t v0 = (int64_t)blockIdx.x * OPB; v0 < total4; v0 += (int64_t)gridDim.x * OPB) {
    const int64_t v = v0 + og;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (v < total4) {
      const float4* src = reinterpret_cast<const float4*>(partial) + v;
      int sl = sg;
      for (; sl + 2 * SG < S; sl += 3 * SG) {
        const float4 p0 = __ldcg(src + sl * total4), p1 = __ldcg(src + (sl + SG) * total4),
                     p2 = __ldcg(src + (sl + 2 * SG) * total4);
        a.x += p0.x; a.y += p0.y; a.z += p0.z; a.w += p0.w;
        a.x += p1.x; a.y += p1.y; a.z += p1.z; a.w += p1.w;
        a.x += p2.x; a.y += p2.y; a.z += p2.z; a.w += p2.w;
      }
      for (; sl < S; sl += SG) {
        const float4 p0 = __ldcg(src + sl * total4);
        a.x += p0.x; a.y += p0.y; a.z += p0.z; a.w += p0.w;
      }
    }
    if constexpr (SG > 1) {
      red[sg][og] = a;
      MSG_JITTER();
      __syncthreads();
      if (sg == 0) {
#pragma unroll
        for (int g = 1; g < SG; ++g) {
          const float4 r = red[g][og];
          a.x += r.x; a.y += r.y; a.z += r.z; a.w += r.w;
        }
      }
      MSG_JITTER();
      __syncthreads();
    }
    if (sg != 0 || v >= total4) continue;
    const int64_t t = v * 4, i = t / b, c = t - i * b;
    if (b % 4 == 0) {  // the four outputs share row i
      if (tail) {
        const uint32_t tc = tailp[i];
        for (int u = 0; u < tail; ++u) {
          const float w = vals.v[(tc >> (4 * u)) & 0xF];
          const int64_t xo = (nb * d + u) * b + c;
          a.x = fmaf(w, load_as<float>(x, x_dtype, xo), a.x);
          a.y = fmaf(w, load_as<float>(x, x_dtype, xo + 1), a.y);
          a.z = fmaf(w, load_as<float>(x, x_dtype, xo + 2), a.z);
          a.w = fmaf(w, load_as<float>(x, x_dtype, xo + 3), a.w);
        }
      }
      if (scale_mode == MSG_SCALE_PER_ROW) {
        const float qs = load_as<float>(q, q_dtype, i);
        a.x *= qs; a.y *= qs; a.z *= qs; a.w *= qs;
      }
    } else {           // b % 4 != 0 (m b % 4 == 0): the four outputs may span rows
      float* av[4] = {&a.x, &a.y, &a.z, &a.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t ie = (t + e) / b, ce = (t + e) - ie * b;
        float r = *av[e];
        if (tail) {
          const uint32_t tc = tailp[ie];
          for (int u = 0; u < tail; ++u)
            r = fmaf(vals.v[(tc >> (4 * u)) & 0xF], load_as<float>(x, x_dtype, (nb * d + u) * b + ce), r);
        }
        if (scale_mode == MSG_SCALE_PER_ROW) r *= load_as<float>(q, q_dtype, ie);
        *av[e] = r;
      }
    }
    auto put = [&](void* yy) {
      if (y_dtype == MSG_F16) {
        __half2 h0 = __floats2half2_rn(a.x, a.y), h1 = __floats2half2_rn(a.z, a.w);
        *reinterpret_cast<uint2*>(reinterpret_cast<__half*>(yy) + t) =
            make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
      } else if (y_dtype == MSG_F32) {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(yy) + t) = a;
      } else {
        store_as<float>(yy, y_dtype, t, a.x);
        store_as<float>(yy, y_dtype, t + 1, a.y);
        store_as<float>(yy, y_dtype, t + 2, a.z);
        store_as<float>(yy, y_dtype, t + 3, a.w);
      }
    };
    put(y);
    if (fan.n) {  // compile-time indices (see fused_finish_kernel)
#pragma unroll
      for (int pr = 0; pr < kMaxFan; ++pr)
        if (pr < fan.n) put(fan.p[pr]);
    }
  }
}

// ============================================================================
// host planning / dispatch
// ============================================================================
struct FusedPlan {
  bool ok, lane, rb;
  int rb_groups;
  int rb_rpt;
  int bc, rpt, ql, S, nrow_blocks, ncol_tiles, quads_per_slice;
  bool sym, f32_entries;
  int64_t smem, partial_bytes;
  QuadLayout L;
};

static bool codebook_antisymmetric(const double* v, int n, double* beta) {
  double twob = v[0] + v[n - 1];
  for (int c = 0; c < n; ++c)
    if (v[c] + v[c ^ (n - 1)] != twob) return false;
  *beta = twob / 2;
  return true;
}

// Per-group scales (gemm.py:75-79) run on the row-block kernels when every
// scale group is a whole number of quads: each k-slice is then exactly one
// scale group and the finish kernel weights slice s of row i by q[i, s].
static bool per_group_quads(int64_t k, int d, int64_t group_size) {
  return group_size > 0 && k % group_size == 0 && group_size % d == 0 &&
         (group_size / d) % 4 == 0;
}

static bool fused_eligible(int width, int x_dtype, int64_t k, int d, int scale_mode,
                           int64_t group_size) {
  return width == 4 && (x_dtype == MSG_F16 || x_dtype == MSG_F32) && d >= 1 && d <= 3 &&
         (scale_mode != MSG_SCALE_PER_GROUP || per_group_quads(k, d, group_size));
}

static int rpt_for(int bc) { return bc == 8 ? 16 : 32; }

static FusedPlan fused_plan(int64_t m, int64_t k, int width, const double* values, int x_dtype,
                            int64_t b, int d, int scale_mode, int64_t group_size, int flags) {
  FusedPlan p{};
  p.ok = false;
  if (flags & MSG_FLAG_FORCE_GENERIC) return p;
  if (!fused_eligible(width, x_dtype, k, d, scale_mode, group_size)) return p;
  if (m <= 0 || b <= 0 || k / d == 0) return p;
  double beta = 0;
  p.sym = !(flags & MSG_FLAG_NO_SYMMETRY) && codebook_antisymmetric(values, 16, &beta);
  p.f32_entries = (x_dtype == MSG_F32) || (flags & MSG_FLAG_F32_ENTRIES);
  if (!(flags & MSG_FLAG_NO_LANE) &&
      lane_eligible(width, values, beta, k, x_dtype, b, d, scale_mode, p.sym, p.f32_entries)) {
    // one kernel; its workspace (int64 row sums + tile counters) must be zero on
    // entry and is left zero on exit
    p.lane = true;
    p.S = 0;
    p.partial_bytes = lane_workspace_bytes(m, k);
    p.ok = true;
    return p;
  }
  bool s_exact16 = true;
  for (int c = 0; c < 16; ++c) {
    const float sc = (float)(values[c] - beta);
    if ((double)__half2float(__float2half_rn(sc)) != values[c] - beta) s_exact16 = false;
  }
  if (!(flags & MSG_FLAG_NO_ROWBLOCK) &&
      rb_eligible(width, x_dtype, b, d, scale_mode, p.sym, p.f32_entries, s_exact16)) {
    p.rb = true;
    p.rb_groups = rb_group_count(b);
    p.rb_rpt = rb_choose_rpt(m, b, flags);
    p.partial_bytes = rb_workspace_bytes(m, k, b, p.rb_rpt);
    p.ok = true;
    return p;
  }
  const int esize = p.f32_entries ? 4 : 2;
  const int64_t ES = p.sym ? (1 << (4 * d - 1)) : (1 << (4 * d));
  const int64_t budget = std::min<int64_t>(max_smem_optin(), 227 * 1024) - 2 * 1024;
  const int lob = d == 1 ? 2 : 4, hib = d == 3 ? 2 : 0;
  int bc = b >= 8 ? 8 : (b >= 4 ? 4 : (b >= 2 ? 2 : 1));
  if (b == 3) bc = 4;
  if (b > 4 && b < 8) bc = 8;
  auto quad_bytes = [&](int bcx) {  // tables + 2 staging buffers + staged x, per quad
    return std::max<int64_t>(4 * ES * bcx * esize, 128) +
           2 * (int64_t)kThreads * rpt_for(bcx) * (lob + hib) + 4 * d * bcx * 4;
  };
  while (bc > 1 && quad_bytes(bc) > budget) bc /= 2;
  if (quad_bytes(bc) > budget) return p;
  p.bc = bc;
  p.rpt = rpt_for(bc);
  p.L = quad_layout(m, k, d);
  p.nrow_blocks = (int)ceil_div(m, (int64_t)kThreads * p.rpt);
  p.ncol_tiles = (int)ceil_div(b, bc);
  const int64_t base = (int64_t)p.nrow_blocks * p.ncol_tiles;
  int64_t S = std::max<int64_t>(1, sm_count() / std::max<int64_t>(1, base));
  S = std::min<int64_t>(S, p.L.nq);
  p.quads_per_slice = (int)ceil_div(p.L.nq, S);
  if (scale_mode == MSG_SCALE_PER_GROUP) p.quads_per_slice = (int)(group_size / d / 4);
  p.S = (int)ceil_div(p.L.nq, p.quads_per_slice);
  int64_t ql = std::max<int64_t>(1, std::min<int64_t>(budget / quad_bytes(bc), p.quads_per_slice));
  // staged activations: at most 2 per thread per round
  while (ql > 1 && ql * 4 * d * bc > 2 * kThreads) --ql;
  p.ql = (int)ql;
  p.smem = p.ql * quad_bytes(bc) + p.ql * 4 * d * bc * 4 + 16;  // + second activation buffer
  p.partial_bytes = align256((int64_t)p.S * m * b * 4);
  p.ok = true;
  return p;
}

// Column tiles of <= 4 run the row-block kernel with 512 threads x RPT/2 rows
// (same R = 256 * RPT rows per CTA): twice the warps to hide the gather's
// shared-memory latency, half the accumulator registers.  At BC = 8 the
// gather saturates the shared-memory pipe already and 256 x RPT measured
// faster (config 5: 334 vs 341 us).
template <int BC> constexpr int fused_nt() { return BC <= 4 ? 512 : kThreads; }

template <int D, typename XT, typename ET, int BC, bool SYM, int RPT>
static int launch_fused_t(const FusedPlan& pl, FusedParams& P, cudaStream_t s) {
  constexpr int NT = fused_nt<BC>();
  auto kern = fused_lut_kernel<D, XT, ET, BC, SYM, RPT * kThreads / NT, NT>;
  static int configured_dev = -1;  // one attribute call per kernel and device
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    MSG_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        std::min(max_smem_optin(), 227 * 1024)));
    configured_dev = dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.nrow_blocks, pl.S, pl.ncol_tiles);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MSG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, P));
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

int launch_finish(const float* partial, int S, int64_t m, int64_t b, int64_t k, int d,
                  const uint16_t* tailp, const TailVals& tv, const void* x, int x_dtype,
                  int scale_mode, const void* q, int q_dtype, void* y, int y_dtype,
                  cudaStream_t s);

}  // namespace msg

using namespace msg;

extern "C" {

int64_t msg_repacked_bytes(int64_t m, int64_t k, int d, int layout) {
  if (layout == MSG_LAYOUT_NONE) return 0;
  if (layout == MSG_LAYOUT_LANE) return d == 3 ? lane_layout_bytes(m, k) : -1;
  if (rb_layout_groups(layout))
    return d == 3 ? rb_layout_bytes(m, k, rb_layout_groups(layout), rb_layout_rpt(layout)) : -1;
  if (layout != MSG_LAYOUT_QUAD || d < 1 || d > 3) return -1;
  return quad_layout(m, k, d).total;
}

int msg_repack(const uint8_t* packed, int64_t m, int64_t k, int d, int layout, int symmetric,
               uint8_t* out, void* stream) {
  if (layout == MSG_LAYOUT_LANE) {
    if (d != 3 || !symmetric)
      return fail(MSG_ERR_UNSUPPORTED, "lane layout is for d=3 with an antisymmetric codebook");
    return lane_repack(packed, m, k, out, as_stream(stream));
  }
  if (rb_layout_groups(layout)) {
    if (d != 3 || !symmetric)
      return fail(MSG_ERR_UNSUPPORTED, "row-block layout is for d=3 with an antisymmetric codebook");
    return rb_repack(packed, m, k, rb_layout_groups(layout), rb_layout_rpt(layout), out,
                     as_stream(stream));
  }
  if (layout != MSG_LAYOUT_QUAD)
    return fail(MSG_ERR_UNSUPPORTED, "unknown weight layout %d", layout);
  if (d < 1 || d > 3) return fail(MSG_ERR_UNSUPPORTED, "quad layout supports d in 1..3, got %d", d);
  QuadLayout L = quad_layout(m, k, d);
  int64_t total = L.nq * L.mp;
  if (total == 0) return fail(MSG_ERR_UNSUPPORTED, "quad layout needs at least one full group");
  const int64_t tiles = ceil_div(L.mp, kQrRows) * ceil_div(L.nq, kQrQuads);
  int grid = (int)std::min<int64_t>(tiles, (int64_t)sm_count() * 8);
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
  FusedPlan p = fused_plan(m, k, width, values, x_dtype, b, d, scale_mode, group_size, flags);
  if (p.ok) {
    *layout_out = p.lane ? MSG_LAYOUT_LANE
                : p.rb ? (p.rb_groups == 4 ? (p.rb_rpt == 8 ? MSG_LAYOUT_RB4S : MSG_LAYOUT_RB4)
                                           : p.rb_groups == 8 ? MSG_LAYOUT_RB8 : MSG_LAYOUT_RB16)
                       : MSG_LAYOUT_QUAD;
    *symmetric_out = p.sym ? 1 : 0;
    *ws_out = p.partial_bytes;
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
  FusedPlan p = fused_plan(m, k, width, values, x_dtype, b, d, scale_mode, group_size, flags);
  if (!p.ok) {
    if (current_fan().n) return fail(MSG_ERR_UNSUPPORTED, "the generic path has no Y fan-out");
    const CodebookParam cb = make_codebook(values, width);  // 2 KiB block: generic path only
    return run_generic(packed, m, k, width, cb, x, x_dtype, b, d, scale_mode, group_size, q,
                       q_dtype, y, y_dtype, workspace, ws_bytes, s);
  }
  if (!wrep) return fail(MSG_ERR_VALUE, "fused path needs the repacked (quad) weight layout");
  if (ws_bytes < p.partial_bytes)
    return fail(MSG_ERR_WORKSPACE, "workspace too small: need %lld bytes",
                (long long)(p.partial_bytes));
  double beta = 0;
  if (p.sym) codebook_antisymmetric(values, 16, &beta);
  TailVals tv;
  for (int c = 0; c < 16; ++c) tv.v[c] = (float)values[c];
  const bool early = (flags & MSG_FLAG_STATIC_WEIGHTS) != 0;
  const bool lut_only = (flags & MSG_FLAG_LUT_PHASE_ONLY) != 0;
  if (p.lane)  // LUT_PHASE_ONLY: the LUT kernel alone (its sums stay in the workspace)
    return launch_lane(wrep, m, k, values, beta, x, scale_mode, q, q_dtype, y, y_dtype,
                       workspace, ws_bytes, early, lut_only, s);
  if (p.rb)
    return launch_rb(wrep, m, k, values, beta, x, b, scale_mode, q, q_dtype, y, y_dtype,
                     workspace, ws_bytes, early, lut_only, tv, p.rb_rpt, s);
  FusedParams P{};
  P.wrep = wrep;
  P.lo_off = p.L.lo_off;
  P.hi_off = p.L.hi_off;
  P.mp = p.L.mp;
  P.m = m;
  P.nb = p.L.nb;
  P.nq = p.L.nq;
  P.x = x;
  P.b = b;
  P.s_exact16 = 1;
  for (int c = 0; c < 16; ++c) {
    P.s[c] = (float)(values[c] - beta);
    if ((double)__half2float(__float2half_rn(P.s[c])) != values[c] - beta) P.s_exact16 = 0;
  }
  P.beta = (float)beta;
  P.early = early ? 1 : 0;
  P.quads_per_slice = p.quads_per_slice;
  P.ql = p.ql;
  P.partial = reinterpret_cast<float*>(workspace);
  int e = MSG_OK;
  switch (d) {
    case 1: e = launch_fused_d<1>(p, P, x_dtype, s); break;
    case 2: e = launch_fused_d<2>(p, P, x_dtype, s); break;
    case 3: e = launch_fused_d<3>(p, P, x_dtype, s); break;
  }
  if (e) return e;
  if (lut_only) return MSG_OK;
  const uint16_t* tailp =
      p.L.tail ? reinterpret_cast<const uint16_t*>(wrep + p.L.tail_off) : nullptr;
  return launch_finish(P.partial, p.S, m, b, k, d, tailp, tv, x, x_dtype, scale_mode, q, q_dtype,
                       y, y_dtype, s);
}

int msg_gemm_fanout(const uint8_t* packed, const uint8_t* wrep, int64_t m, int64_t k, int width,
                    const double* values, const void* x, int x_dtype, int64_t b, int d,
                    int scale_mode, int64_t group_size, const void* q, int q_dtype, void* y,
                    int y_dtype, void* workspace, int64_t ws_bytes, int flags, void* stream,
                    void* const* y_peers, int n_peers) {
  if (n_peers < 0 || n_peers > kMaxFan)
    return fail(MSG_ERR_VALUE, "fan-out takes 0..%d peer buffers (got %d)", kMaxFan, n_peers);
  if (n_peers && !y_peers) return fail(MSG_ERR_VALUE, "y_peers is NULL");
  if (flags & MSG_FLAG_LUT_PHASE_ONLY) n_peers = 0;
  YFan& fan = current_fan();
  fan.n = n_peers;
  for (int i = 0; i < n_peers; ++i) fan.p[i] = y_peers[i];
  const int e = msg_gemm(packed, wrep, m, k, width, values, x, x_dtype, b, d, scale_mode, group_size,
                         q, q_dtype, y, y_dtype, workspace, ws_bytes, flags, stream);
  fan.n = 0;
  return e;
}

}  // extern "C"

namespace msg {
int launch_finish(const float* partial, int S, int64_t m, int64_t b, int64_t k, int d,
                  const uint16_t* tailp, const TailVals& tv, const void* x, int x_dtype,
                  int scale_mode, const void* q, int q_dtype, void* y, int y_dtype,
                  cudaStream_t s) {
  const int64_t total = m * b;
  const YFan fan = current_fan();
  bool fan_aligned = true;  // the vectorised kernel stores 16 / 8 bytes at a time
  for (int i = 0; i < fan.n; ++i) fan_aligned = fan_aligned && (reinterpret_cast<uintptr_t>(fan.p[i]) & 15) == 0;
  // four outputs per thread group; slices split over SG groups when there are
  // few outputs per SM (e.g. 137 slices x 8192 x 4)
  // (float4 / uint2 stores of Y: a caller-supplied Y must be 16-byte aligned)
  // (b % 4 != 0 works as long as m b % 4 == 0: the flat output index is
  // vectorised and every element finds its own row -- worth it with enough
  // outputs to fill the GPU: for a GEMV-sized m b the scalar kernel keeps
  // four times more threads busy.  Measured crossover, tools/batch_sweep.py
  // with MSG_FIN_VEC_MIN: m b = 16384 (8192^2 b = 2) 26.5 -> 22.0 us vectorised,
  // m b = 12288 (4096^2 b = 3) 15.5 -> 16.8 us: vectorise from 16384 outputs)
  static const int64_t vec_min = [] {
    const char* e = std::getenv("MSG_FIN_VEC_MIN");
    return e ? (int64_t)std::atoll(e) : (int64_t)16384;
  }();
  // the slice-group count fixes the fp32 summation order: a shape the
  // vectorised kernel can take uses ITS count in the scalar kernel too, so Y
  // does not depend on where the caller's buffer happens to be aligned
  const bool vec_shape = total % 4 == 0 && (b % 4 == 0 || total >= vec_min) &&
                         scale_mode != MSG_SCALE_PER_GROUP && S >= 2;
  int sg_vec = 1;
  while (sg_vec < 16 && 2 * sg_vec <= S && (total / 4) * sg_vec < (int64_t)sm_count() * 512) sg_vec *= 2;
  if (vec_shape && (reinterpret_cast<uintptr_t>(y) & 15) == 0 && fan_aligned) {
    const int sg = sg_vec;
    const int opb = 256 / sg;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(total / 4, opb), (int64_t)sm_count() * 8)));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#define MSG_FIN4(G)                                                                            \
  MSG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, finish_vec4_kernel<G>, partial, S, m, b, k, d, tailp, \
                                    tv, x, x_dtype, scale_mode, q, q_dtype, y, y_dtype, fan))
    switch (sg) {
      case 1: MSG_FIN4(1); break;
      case 2: MSG_FIN4(2); break;
      case 4: MSG_FIN4(4); break;
      case 8: MSG_FIN4(8); break;
      default: MSG_FIN4(16); break;
    }
#undef MSG_FIN4
    return MSG_OK;
  }
  // slice groups per output: enough loads in flight to cover the SMs
  int sg = 1;
  while (sg < 32 && 2 * sg <= S && total * sg < (int64_t)sm_count() * 2048) sg *= 2;
  if (vec_shape) sg = sg_vec;
  const int opb = 256 / sg;
  const int grid =
      (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, opb), (int64_t)sm_count() * 16));
  // Programmatic dependent launch: the finish grid is set up while the LUT
  // kernel drains and waits (griddepcontrol.wait) for its results.
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#define MSG_FIN(G)                                                                            \
  MSG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, fused_finish_kernel<G>, partial, S, m, b, k, d,    \
                                    tailp, tv, x, x_dtype, scale_mode, q, q_dtype, y, y_dtype, fan))
  switch (sg) {
    case 1: MSG_FIN(1); break;
    case 2: MSG_FIN(2); break;
    case 4: MSG_FIN(4); break;
    case 8: MSG_FIN(8); break;
    case 16: MSG_FIN(16); break;
    default: MSG_FIN(32); break;
  }
#undef MSG_FIN
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

int launch_finish_plain(const float* partial, int S, int64_t m, int64_t b, void* y, int y_dtype,
                        cudaStream_t s) {
  TailVals tv{};
  return launch_finish(partial, S, m, b, 0, 1, nullptr, tv, nullptr, MSG_F32, MSG_SCALE_NONE,
                       nullptr, MSG_F32, y, y_dtype, s);
}

}  // namespace msg
