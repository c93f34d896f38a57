// msGeMM GEMV kernel (b = 1, d = 3, fp16 sign-symmetric tables): bank-private
// tables and a lane-rotated weight layout.
//
// Reference semantics as in msg_fused.cu (gemm.py:70-153, lut.py:59-72,
// packing.py:201-228); results go through the same deterministic finish
// kernel.
//
// Why a separate kernel: at b = 1 every table lookup returns 2 bytes, so the
// gather is bound by instruction issue and shared-memory bank conflicts,
// not by bytes.  Here
//   * a chunk of 32 groups has its 32 half tables (2048 fp16 entries each,
//     128 KiB total) laid out bank-private: group j lives only in bank j
//     (word (row, j) holds entries row and row+1024 of group j);
//   * lane l of a warp owns row 32*tile + l and, at step t, looks up group
//     (t + l) mod 32 -- all 32 lanes hit 32 different banks, every LDS is a
//     single wavefront, and each lane accumulates its own row (no cross-lane
//     reduction);
//   * K3 stores each row's 32 indices in that rotated order, split into a
//     10-bit "row" stream (one funnel shift + one LOP3 gives the table byte
//     offset) and a 2-bit stream (half select, sign), 12 bits per group as in
//     the reference layout; a warp reads a 32-row tile as three coalesced
//     512-byte requests;
//   * accumulation is FHFMA (fp32 += fp16 * +-1, one instruction).
// Work is the (chunk, row tile) grid linearised chunk-major and split evenly
// over one persistent CTA per SM, so each table is built by at most two CTAs
// more than the minimum.
#include <algorithm>

#include "msg_common.cuh"

namespace msg {

static inline int64_t align256l(int64_t v) { return (v + 255) / 256 * 256; }

struct LaneLayout {
  int64_t nb, nchunk, ntiles, tail;
  int64_t body_off, tail_off, total;  // body: [chunk][tile][3][32 lanes][16 B]
};

static LaneLayout lane_layout(int64_t m, int64_t k) {
  LaneLayout L{};
  L.nb = k / 3;
  L.nchunk = (L.nb + 31) / 32;
  L.ntiles = (m + 31) / 32;
  L.tail = k - L.nb * 3;
  L.body_off = 0;
  L.tail_off = align256l(L.nchunk * L.ntiles * 1536);
  L.total = L.tail_off + (L.tail ? align256l(m * 2) : 0);
  if (L.total == 0) L.total = 256;
  return L;
}

int64_t lane_layout_bytes(int64_t m, int64_t k) { return lane_layout(m, k).total; }
int64_t lane_tail_offset(int64_t m, int64_t k) { return lane_layout(m, k).tail_off; }

__device__ __forceinline__ uint32_t nib_l(const uint8_t* row, int64_t j) {
  return (row[j >> 1] >> ((j & 1) * 4)) & 0xF;
}

// One thread per (chunk, row): 48 bytes = 10 words of 10-bit "row" fields
// (position t at bit 10t), one word of signs (positions 2q, 2q+1 at bits
// 15-q, 31-q, so one shift + LOP3 yields two fp16 +-1 multipliers) and one
// word of half-select bits (position t at bit t).  Position t of row i holds
// group t ^ (i % 32) of the chunk.  Stored in the coalesced tile order
// [chunk][tile][v][lane][4 words].
__global__ void repack_lane_kernel(const uint8_t* __restrict__ packed, int64_t m, int64_t k,
                                   int rb, LaneLayout L, uint8_t* __restrict__ out) {
  const int64_t total = L.nchunk * L.ntiles * 32;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / (L.ntiles * 32);
    const int64_t i = t - c * (L.ntiles * 32);  // padded row
    uint32_t w[12] = {0};
    if (i < m) {
      const uint8_t* row = packed + i * rb;
      for (int p = 0; p < 32; ++p) {
        const int64_t j = c * 32 + (p ^ (i & 31));
        uint32_t f = 0, sign = 0;
        if (j < L.nb) {
          uint32_t idx = nib_l(row, 3 * j) | (nib_l(row, 3 * j + 1) << 4) | (nib_l(row, 3 * j + 2) << 8);
          if (idx & 0x800) { idx ^= 0xFFF; sign = 1; }  // sign symmetry: complement
          f = idx;                                       // 11 bits
        }
        const uint32_t rowf = f & 0x3FF, half = f >> 10;
        const int bit = 10 * p;
        w[bit >> 5] |= rowf << (bit & 31);
        if ((bit & 31) > 22) w[(bit >> 5) + 1] |= rowf >> (32 - (bit & 31));
        // signs of positions 2q, 2q+1 at bits 15-q, 31-q; half select of p at bit p
        w[10] |= sign << ((p & 1) ? 31 - (p >> 1) : 15 - (p >> 1));
        w[11] |= half << p;
      }
      if (L.tail && c == 0) {
        uint32_t tc = 0;
        for (int64_t j = L.nb * 3; j < k; ++j) tc |= nib_l(row, j) << (4 * (j - L.nb * 3));
        reinterpret_cast<uint16_t*>(out + L.tail_off)[i] = (uint16_t)tc;
      }
    }
    const int64_t tile = i >> 5, lane = i & 31;
    uint4* base = reinterpret_cast<uint4*>(out + L.body_off) + (c * L.ntiles + tile) * 96;
    base[0 * 32 + lane] = make_uint4(w[0], w[1], w[2], w[3]);
    base[1 * 32 + lane] = make_uint4(w[4], w[5], w[6], w[7]);
    base[2 * 32 + lane] = make_uint4(w[8], w[9], w[10], w[11]);
  }
}

__device__ __forceinline__ void fhfma_l(float& acc, unsigned short h, unsigned short s16) {
  asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(h), "h"(s16));
}

__device__ __forceinline__ uint32_t mul_hi_u32(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

template <int N>
__device__ __forceinline__ uint32_t funnel_r(uint32_t lo, uint32_t hi) {
  uint32_t r;
  asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(lo), "r"(hi), "n"(N));
  return r;
}

struct LaneParams {
  const uint8_t* body;
  int64_t m, nb, nchunk, ntiles;
  const void* x;  // (k,) fp16 or fp32
  float s[16];    // v[c] - beta
  float beta;
  float* partial;  // [nchunk][m]
  TraceRec* trace;  // per-CTA trace records or nullptr
  uint32_t ones;    // 0x3C003C00: two fp16 +1.0
  int early;        // MSG_FLAG_STATIC_WEIGHTS: stream weights before griddepcontrol.wait
};

constexpr int kLaneThreads = 512;

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__half v) { return __half2float(v); }

// One lookup at position T: the 10-bit row field lands at byte-offset bits
// 7..16 via one funnel shift, the half select at bit 1, the bank offset
// (T ^ lane) * 4 at bits 2..6; the fp16 entry is accumulated with FHFMA.
template <int T>
__device__ __forceinline__ void lookup(const uint32_t (&w)[12], uint32_t xt, uint32_t S,
                                       float& acc) {
  // The row field occupies stream bits [10T, 10T+10) and must land at bits
  // 7..16.  Shifts that stay inside one word use the FMA pipe (IMAD.SHL /
  // IMAD.HI as >>) so the ALU pipe -- the bound of this kernel -- only does the
  // masking and the final 3-input add.
  constexpr int S0 = (10 * T) & 31, K = (10 * T) >> 5;
  uint32_t d;
  if constexpr (S0 + 10 <= 32) {
    if constexpr (S0 == 7) d = w[K];
    else if constexpr (S0 < 7) d = w[K] << (7 - S0);
    else d = mul_hi_u32(w[K], 1u << (39 - S0));  // == w[K] >> (S0 - 7)
  } else {
    constexpr int B = 10 * T - 7;
    d = funnel_r<(B & 31)>(w[B >> 5], w[(B >> 5) + 1]);
  }
  uint32_t hb;  // half-select bit T of w[11] moved to bit 1
  if constexpr (T == 0) hb = w[11] << 1;
  else if constexpr (T == 1) hb = w[11];
  else hb = mul_hi_u32(w[11], 1u << (33 - T));  // == w[11] >> (T - 1)
  // xt already holds table base + bank offset; the three fields do not overlap
  uint32_t addr;
  asm("add.u32 %0, %1, %2;" : "=r"(addr) : "r"(d & 0x1FF80u), "r"(hb & 2u));
  addr += xt;
  // gather one fp16 entry and accumulate +-entry into fp32; the multiplier is
  // the low (even T) or high (odd T) half of S
  if constexpr (T & 1)
    asm volatile(
        "{\n\t.reg .b16 h, lo, hi;\n\t"
        "ld.shared.u16 h, [%1];\n\t"
        "mov.b32 {lo, hi}, %2;\n\t"
        "fma.rn.f32.f16 %0, h, hi, %0;\n\t}"
        : "+f"(acc) : "r"(addr), "r"(S));
  else
    asm volatile(
        "{\n\t.reg .b16 h, lo, hi;\n\t"
        "ld.shared.u16 h, [%1];\n\t"
        "mov.b32 {lo, hi}, %2;\n\t"
        "fma.rn.f32.f16 %0, h, lo, %0;\n\t}"
        : "+f"(acc) : "r"(addr), "r"(S));
}

template <int T, int TPW>
__device__ __forceinline__ void steps(const uint32_t (&w)[TPW][12], uint32_t tab,
                                      uint32_t lane4, uint32_t ones, float (&acc)[TPW]) {
  if constexpr (T < 32) {
    const uint32_t xt = tab + (lane4 ^ (uint32_t)(T << 2));  // base + bank of group T ^ lane
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
      // +-1.0h multipliers of positions 2q, 2q+1 (sign bits at 15-q, 31-q)
      const uint32_t S = ((w[u][10] << (T >> 1)) & 0x80008000u) | ones;
      lookup<T>(w[u], xt, S, acc[u]);
    }
    steps<T + 1, TPW>(w, tab, lane4, ones, acc);
  }
}

constexpr int kTableBytes = 128 * 1024;
constexpr int kTileBytes = 1536;             // one 32-row tile of one chunk
constexpr int kRing = 4;                     // tiles in flight per warp (TMA ring)
constexpr int kNW = kLaneThreads / 32;
constexpr int kLaneSmem = kTableBytes + kNW * kRing * kTileBytes + kNW * kRing * 8;

// Work unit = "superbatch": TPW*kNW consecutive row tiles of one chunk, so that
// every warp gets exactly one batch of TPW tiles per superbatch; superbatches
// (chunk-major) are split evenly over one CTA per SM.  Each warp streams its
// tiles through a kRing-deep ring of shared-memory slots filled by
// cp.async.bulk (lane 0 issues, one mbarrier per slot), so the weight stream
// has kNW*kRing*1.5 KB in flight per SM independently of the table build.
template <typename XT, int TPW>
__global__ void __launch_bounds__(kLaneThreads, 1) lane_lut_kernel(LaneParams P) {
  extern __shared__ __align__(128) uint8_t smem[];  // table | rings | mbarriers
  constexpr int SB = TPW * kNW;                     // tiles per superbatch
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint8_t* ring = smem + kTableBytes + warp * kRing * kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kTableBytes + kNW * kRing * kTileBytes) +
                   warp * kRing;
  const int64_t nsb = (P.ntiles + SB - 1) / SB;  // superbatches per chunk
  const int64_t U = P.nchunk * nsb;
  const int64_t u_begin = U * blockIdx.x / gridDim.x;
  const int64_t u_end = U * (blockIdx.x + 1) / gridDim.x;
  __shared__ float corr_s;
  const unsigned long long t_start = P.trace ? global_ns() : 0ull;

  if (lane == 0)
    for (int i = 0; i < kRing; ++i) mbar_init(&bars[i], 1);
  fence_mbar_init();
  __syncwarp();

  // Issue cursor (lane-uniform, no division on the hot path): chunk nc,
  // superbatch ns within it, tile nq of this warp's batch; nu = linear unit.
  // Tile of this warp for (ns, nq) is ns*SB + warp*TPW + nq.
  uint32_t issued = 0, consumed = 0;  // per-warp ring counters (lane-uniform)
  int64_t nu = u_begin, nc = u_begin / nsb, ns = u_begin - (u_begin / nsb) * nsb;
  int nq = 0;
  // keep kRing tiles of this warp in flight, in consumption order (lane 0 issues)
  auto refill = [&]() {
    while (issued - consumed < (uint32_t)kRing && nu < u_end) {
      const int64_t t = ns * SB + warp * TPW + nq;
      if (t < P.ntiles) {
        if (lane == 0) {
          const int slot = issued % kRing;
          fence_proxy_async();
          mbar_expect_tx(&bars[slot], kTileBytes);
          bulk_g2s(ring + slot * kTileBytes, P.body + (nc * P.ntiles + t) * kTileBytes,
                   kTileBytes, &bars[slot]);
        }
        ++issued;
      }
      if (++nq == TPW) {
        nq = 0;
        ++nu;
        if (++ns == nsb) { ns = 0; ++nc; }
      }
    }
  };

  // activations are prefetched as raw XT values and converted at the build,
  // so the load latency is not exposed where the prefetch is issued
  auto load_x = [&](int64_t c, XT& x0, XT& x1, XT& x2) {
    x0 = x1 = x2 = XT(0.f);
    const int64_t g = c * 32 + lane;
    if (c < P.nchunk && g < P.nb) {
      const XT* xp = reinterpret_cast<const XT*>(P.x) + 3 * g;
      x0 = xp[0];
      x1 = xp[1];
      x2 = xp[2];
    }
  };
  XT xn0, xn1, xn2;
  // Launched with PDL: the prologue overlaps the previous kernel's tail.  The
  // weight stream may start before the wait only if the previous kernel did
  // not write it; x and the partials are touched only after the wait.
  if (P.early) refill();
  griddep_wait();
  griddep_launch_dependents();  // the finish kernel may queue behind this grid
  if (!P.early) refill();
  load_x(u_begin / nsb, xn0, xn1, xn2);

  int64_t u = u_begin;
  while (u < u_end) {
    const int64_t c = u / nsb;
    const int64_t sb_end = std::min<int64_t>(u_end, (c + 1) * nsb);  // this chunk's share
    const float x0 = to_f(xn0), x1 = to_f(xn1), x2 = to_f(xn2);
    load_x(c + 1, xn0, xn1, xn2);  // prefetch the next chunk's activations
    // ---- build chunk c's 32 bank-private half tables (groups beyond nb get
    // x = 0, i.e. all-zero tables, so padded positions contribute nothing)
    __syncthreads();
    {
      const int j = lane;
      float a[16];
#pragma unroll
      for (int v = 0; v < 16; ++v) a[v] = P.s[v] * x0;
      if (warp == 0) {
        float sx = x0 + x1 + x2;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
        if (lane == 0) corr_s = P.beta * sx;
      }
      // warp w (of 16) builds rows u0 | u1<<4 | u2lo<<8 with u2lo = w/4 and
      // u1 in [4(w%4), 4(w%4)+4); the high half of word (row, j) is entry
      // row + 1024 (u2 = u2lo + 4)
      static_assert(kLaneThreads == 512, "build split assumes 16 warps");
      const int u2lo = warp >> 2;
      const float c0 = P.s[u2lo] * x2, c1 = P.s[u2lo + 4] * x2;
      uint32_t* tw = reinterpret_cast<uint32_t*>(smem);
#pragma unroll 2
      for (int hh = 0; hh < 4; ++hh) {
        const int u1 = (warp & 3) * 4 + hh;
        const float bv = P.s[u1] * x1;
        const float bc0 = bv + c0, bc1 = bv + c1;
        uint32_t* dst = tw + ((u1 << 4) | (u2lo << 8)) * 32 + j;
#pragma unroll
        for (int u0 = 0; u0 < 16; ++u0) {
          __half2 h2 = __floats2half2_rn(a[u0] + bc0, a[u0] + bc1);
          dst[u0 * 32] = *reinterpret_cast<uint32_t*>(&h2);
        }
      }
    }
    __syncthreads();
    const float corr = corr_s;
    const uint32_t lane4 = (uint32_t)lane << 2;
    const uint32_t tab32 = smem_u32(smem);
    const uint32_t ones = P.ones;  // 0x3C003C00 from the parameter block (one LOP3 for S)
    for (; u < sb_end; ++u) {
      const int64_t sb = u - c * nsb;
      const int64_t t0 = sb * SB + warp * TPW;
      uint32_t w[TPW][12];
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        if (t0 + q < P.ntiles) {
          const int slot = consumed % kRing;
          mbar_wait(&bars[slot], (consumed / kRing) & 1);
          const uint4* tb = reinterpret_cast<const uint4*>(ring + slot * kTileBytes);
          uint4 v0 = tb[lane], v1 = tb[32 + lane], v2 = tb[64 + lane];
          w[q][0] = v0.x; w[q][1] = v0.y; w[q][2] = v0.z; w[q][3] = v0.w;
          w[q][4] = v1.x; w[q][5] = v1.y; w[q][6] = v1.z; w[q][7] = v1.w;
          w[q][8] = v2.x; w[q][9] = v2.y; w[q][10] = v2.z; w[q][11] = v2.w;
          ++consumed;
        } else {
#pragma unroll
          for (int e = 0; e < 12; ++e) w[q][e] = 0;
        }
      }
      __syncwarp();  // every lane has copied its words out of the consumed slots
      refill();
      float acc[TPW];
#pragma unroll
      for (int q = 0; q < TPW; ++q) acc[q] = corr;
      steps<0, TPW>(w, tab32, lane4, ones, acc);
#pragma unroll
      for (int q = 0; q < TPW; ++q) {
        const int64_t row = (t0 + q) * 32 + lane;
        if (t0 + q < P.ntiles && row < P.m) P.partial[c * P.m + row] = acc[q];
      }
    }
  }
  if (P.trace) {
    __syncthreads();
    if (tid == 0 && blockIdx.x < kTraceMax)
      P.trace[blockIdx.x] =
          TraceRec{sm_id(), t_start, global_ns(), (unsigned long long)(u_end - u_begin)};
  }
}

bool lane_eligible(int width, int x_dtype, int64_t b, int d, int scale_mode, bool sym,
                   bool f32_entries) {
  return width == 4 && d == 3 && b == 1 && sym && !f32_entries &&
         (x_dtype == MSG_F16 || x_dtype == MSG_F32) && scale_mode != MSG_SCALE_PER_GROUP;
}

int lane_repack(const uint8_t* packed, int64_t m, int64_t k, uint8_t* out, cudaStream_t s) {
  LaneLayout L = lane_layout(m, k);
  const int64_t total = L.nchunk * L.ntiles * 32;
  if (total == 0) return fail(MSG_ERR_UNSUPPORTED, "lane layout needs at least one group");
  int grid = (int)std::min<int64_t>(ceil_div(total, 256), (int64_t)sm_count() * 16);
  repack_lane_kernel<<<grid, 256, 0, s>>>(packed, m, k, row_bytes(k, 4), L, out);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

int64_t lane_partial_slices(int64_t m, int64_t k) { return lane_layout(m, k).nchunk; }

template <typename XT, int TPW>
static int launch_lane_t(const LaneParams& P, cudaStream_t s) {
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    MSG_CUDA_CHECK(cudaFuncSetAttribute(lane_lut_kernel<XT, TPW>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, kLaneSmem));
    configured_dev = dev;
  }
  const int64_t nsb = (P.ntiles + TPW * kNW - 1) / (TPW * kNW);
  const int64_t U = P.nchunk * nsb;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(U, sm_count()));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kLaneThreads);
  cfg.dynamicSmemBytes = kLaneSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MSG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, lane_lut_kernel<XT, TPW>, P));
  return MSG_OK;
}

template <typename XT>
static int launch_lane_x(const LaneParams& P, cudaStream_t s) {
  // superbatch granularity: 2 tiles per warp when every SM gets several
  // superbatches, else 1 (finer split, better balance on small problems)
  const int64_t sb2 = P.nchunk * ((P.ntiles + 2 * kNW - 1) / (2 * kNW));
  if (sb2 >= 4 * (int64_t)sm_count()) return launch_lane_t<XT, 2>(P, s);
  return launch_lane_t<XT, 1>(P, s);
}

int launch_lane(const uint8_t* wrep, int64_t m, int64_t k, const double* values, double beta,
                const void* x, int x_dtype, float* partial, bool early, cudaStream_t s) {
  LaneLayout L = lane_layout(m, k);
  LaneParams P{};
  P.body = wrep + L.body_off;
  P.m = m;
  P.nb = L.nb;
  P.nchunk = L.nchunk;
  P.ntiles = L.ntiles;
  P.x = x;
  for (int c = 0; c < 16; ++c) P.s[c] = (float)(values[c] - beta);
  P.beta = (float)beta;
  P.partial = partial;
  P.trace = trace_buffer();
  P.ones = 0x3C003C00u;
  P.early = early ? 1 : 0;
  if (x_dtype == MSG_F16) return launch_lane_x<__half>(P, s);
  return launch_lane_x<float>(P, s);
}

}  // namespace msg
