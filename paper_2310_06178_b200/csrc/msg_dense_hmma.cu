// Dense comparison baseline for 1 <= b <= 16: a weight-streaming kernel that
// dequantises int4 in registers and multiplies on the tensor cores with
// mma.sync (m16n8k16, fp16 x fp16 -> fp32), reading the reference's own packed
// layout (no repack, no X preparation kernel, no split-k finishing kernel).
//
// Spec: naive_gemm(dense(pwm), X) (gemm.py:206-216, packing.py:191-198) for
// int4 / uint4 codebooks and fp16 X.  At these batch sizes the dense product
// is bound by the weight stream (m k / 2 bytes from HBM); the CUDA-core GEMV
// (msg_dense.cu) spends ~2.3 issue slots per weight on dequantise + FMA, and
// the tcgen05 kernel (msg_mma.cu) pays a TMA/TMEM pipeline built for
// M128 x N x K64 tiles.  Here the multiply costs one HMMA per 256 weights and
// the columns 2..8 (9..16: a second n-tile) ride for free, so the issue cost
// is the dequantise alone (~1.1 slots per weight).
//
// CTA = 8 warps x 16 rows; a warp streams its 16 rows in chunks of 256
// weights: quad lane t of row g / g + 8 (the two rows a thread holds in an
// m16n8k16 A fragment) loads bytes [128 c + 32 t, +32) of the row -- a quad
// reads whole 128-byte lines (tools/microbench/stream_pattern.cu: 64-byte
// pieces per row stream ~20 % slower) -- four chunks ahead.  One 32-bit word of 8 nibbles
// k0..k7 becomes the fp16 pairs (k0,k4) (k1,k5) (k2,k6) (k3,k7) with one LOP3
// and one HSUB2 / HFMA2 each (magic numbers 1024 + u, as msg_dense.cu); pairs
// 0/1 are the A registers of one HMMA and 2/3 of the next, so the MMA's k
// slots (2t, 2t+1 | 2t+8, 2t+9) stand for the activations (k0,k4 | k1,k5):
// the k order inside an MMA is free as long as B agrees.  X is staged per
// CTA and k sub-slice in shared memory directly in that B-fragment order
// ([chunk][n-tile][column g][t][16 words], the four 16-byte units of a lane
// XOR-swizzled so every LDS.128 phase is conflict-free).
//
// Split k: the S CTAs of a thread-block cluster (1, S, 1) take k slices of
// the same 128 rows and meet in distributed shared memory -- every CTA sums
// 128 / S rows over the S partial tiles in rank order (deterministic) and
// writes Y.  Products int4 x fp16 are exact in fp32; for integer-valued X
// with partial sums below 2^24 the result is bit-exact.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "msg_common.cuh"

namespace cg = cooperative_groups;

namespace msg {

constexpr int kDhThreads = 256, kDhWarps = kDhThreads / 32;
constexpr int kDhRows = kDhWarps * 16;  // rows per CTA
constexpr int kDhNV = 2;                // 16-byte loads per thread, row and chunk
constexpr int kDhJ = 4 * kDhNV;         // 32-bit weight words per thread, row and chunk
constexpr int kDhChunk = 128 * kDhNV;   // weights per (row, warp iteration): a full 128-byte line per quad
#ifndef MSG_DH_DEPTH
#define MSG_DH_DEPTH 4
#endif
constexpr int kDhDepth = MSG_DH_DEPTH;  // chunks in flight per warp
#ifndef MSG_DH_SUBK
#define MSG_DH_SUBK 2048
#endif
constexpr int kDhSubK = MSG_DH_SUBK;    // activation rows per staged X sub-slice
constexpr int kDhSub = kDhSubK / kDhChunk;
static_assert(kDhSub % kDhDepth == 0, "sub-slices hold whole pipeline rounds");

struct DhConsts {
  uint32_t magic, magic_hi, sub2, sub_hi;
};

struct DhParams {
  const uint8_t* packed;
  int64_t m, k, rb;
  const __half* x;
  int b;
  int nchunks, chunks_per_cta;
  DhConsts c;
  void* y;
  int y_dtype;
};

// 8 nibbles -> 4 half2 registers (k0,k4) (k1,k5) (k2,k6) (k3,k7), exact
__device__ __forceinline__ void dh_dequant(uint32_t wd, const DhConsts& c, uint32_t (&h)[4]) {
  const uint32_t w8 = wd >> 8;
  uint32_t t0, t1, t2, t3;
  asm("lop3.b32 %0, %1, 0x000F000F, %2, 0x6A;" : "=r"(t0) : "r"(wd), "r"(c.magic));  // (a & b) ^ c
  asm("lop3.b32 %0, %1, 0x00F000F0, %2, 0x6A;" : "=r"(t1) : "r"(wd), "r"(c.magic_hi));
  asm("lop3.b32 %0, %1, 0x000F000F, %2, 0x6A;" : "=r"(t2) : "r"(w8), "r"(c.magic));
  asm("lop3.b32 %0, %1, 0x00F000F0, %2, 0x6A;" : "=r"(t3) : "r"(w8), "r"(c.magic_hi));
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(h[0]) : "r"(t0), "r"(c.sub2));
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(h[1]) : "r"(t1), "r"(0x2C002C00u), "r"(c.sub_hi));
  asm("sub.rn.f16x2 %0, %1, %2;" : "=r"(h[2]) : "r"(t2), "r"(c.sub2));
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(h[3]) : "r"(t3), "r"(0x2C002C00u), "r"(c.sub_hi));
}

__device__ __forceinline__ void dh_mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                       uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint4 dh_ldw(const uint8_t* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// bytes of staged X per chunk and n-tile: 8 columns x 4 quad lanes x (16 kDhJ) B
constexpr int kDhLaneBytes = 16 * kDhJ;
constexpr int kDhTileBytes = 8 * 4 * kDhLaneBytes;

template <int NT>
__global__ void __launch_bounds__(kDhThreads, (NT == 1 && kDhDepth <= 2) ? 3 : 2) dq_hmma_kernel(DhParams P) {
  extern __shared__ __align__(128) uint8_t smem[];  // [kDhSub][NT][8][4][kDhLaneBytes]; later the partial tile
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const uint32_t swz = (uint32_t)(lane & (kDhJ - 1));
  const int64_t row0 = (int64_t)blockIdx.x * kDhRows;
  // chunks [c_begin, c_end) of this k slice; c_end is c_begin plus a multiple
  // of kDhDepth (the host rounds chunks_per_cta): chunks past the matrix read
  // clamped (in-bounds) weight bytes against zero activations
  const int c_begin = (int)blockIdx.y * P.chunks_per_cta;
  const int c_end = c_begin + P.chunks_per_cta;

  // this thread's two rows, clamped for the loads: rows >= m accumulate
  // another row's weights and are never stored
  const int64_t ra = row0 + warp * 16 + g, rbw = ra + 8;
  const uint8_t* pa = P.packed + min(ra, P.m - 1) * P.rb;
  const uint8_t* pb = P.packed + min(rbw, P.m - 1) * P.rb;
  const uint32_t last = (uint32_t)P.rb - 16u;
  auto load_w = [&](int c, uint4 (&wa)[kDhNV], uint4 (&wb)[kDhNV]) {
#pragma unroll
    for (int v = 0; v < kDhNV; ++v) {
      const uint32_t o = min((uint32_t)c * (kDhChunk / 2) + (uint32_t)(16 * kDhNV * t + 16 * v), last);
      wa[v] = dh_ldw(pa + o);
      wb[v] = dh_ldw(pb + o);
    }
  };
  uint4 wa[kDhDepth][kDhNV], wb[kDhDepth][kDhNV];
  // weights never depend on the preceding kernel: in flight before the PDL wait
#pragma unroll
  for (int u = 0; u < kDhDepth; ++u) load_w(c_begin + u, wa[u], wb[u]);
  const int kk = (int)P.k, bb = P.b;
  if (bb < NT * 8) {  // columns >= b of the staged X are never written: zero them once
    for (int i = tid; i < kDhSub * NT * kDhTileBytes / 16; i += kDhThreads)
      reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
  }
  griddep_wait();
  griddep_launch_dependents();

  float d[NT][2][4];  // two accumulator chains per n-tile (even / odd HMMAs)
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) d[nt][0][i] = d[nt][1][i] = 0.f;
  const uint32_t xs_lane = smem_u32(smem) + (uint32_t)((g * 4 + t) * kDhLaneBytes);
  const bool xvec = (P.b & 7) == 0 && (reinterpret_cast<uintptr_t>(P.x) & 15) == 0;

  for (int sub = c_begin; sub < c_end; sub += kDhSub) {
    const int sub_end = min(c_end, sub + kDhSub);
    if (sub != c_begin) __syncthreads();  // the previous sub-slice's X is consumed
    // ---- stage X rows [kDhChunk sub, kDhChunk sub_end) in B-fragment order:
    // item = (chunk lc, quad lane tt, word group j, word w) holds the
    // activation rows k_lo = kDhChunk c + 8 kDhJ tt + 8 j + w and k_lo + 4 of
    // every column (columns >= b hold zeros: their products land in Y columns
    // that are not stored)
    constexpr int kItemsPerChunk = 4 * kDhJ * 4;
    constexpr int kItems = kDhSub * kItemsPerChunk / kDhThreads;
    const int nit = (sub_end - sub) * kItemsPerChunk;
    auto item_k = [&](int it) {
      return (sub + it / kItemsPerChunk) * kDhChunk + 8 * kDhJ * ((it / (4 * kDhJ)) & 3) + 8 * ((it >> 2) & (kDhJ - 1)) + (it & 3);
    };
    auto item_dst = [&](int it, int gg) {  // word (x[k_lo], x[k_lo + 4]) of column gg (n-tile 0)
      const int w = it & 3, j = (it >> 2) & (kDhJ - 1), tt = (it / (4 * kDhJ)) & 3, lc = it / kItemsPerChunk;
      const uint32_t sw = (uint32_t)((gg * 4 + tt) & (kDhJ - 1));
      MSG_DASSERT(lc >= 0 && lc < kDhSub && gg >= 0 && gg < 8);
      return reinterpret_cast<uint32_t*>(smem + (size_t)lc * NT * kDhTileBytes + (gg * 4 + tt) * kDhLaneBytes +
                                         16 * (j ^ sw) + 4 * w);
    };
    if (xvec) {
#pragma unroll
      for (int i0 = 0; i0 < kItems; i0 += 2) {  // two items' loads in flight
        uint4 lo[2][NT], hi[2][NT];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int it = tid + (i0 + i) * kDhThreads;
          const int k_lo = item_k(it);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const bool colsv = nt * 8 < bb && it < nit;
            lo[i][nt] = (colsv && k_lo < kk)
                            ? __ldg(reinterpret_cast<const uint4*>(P.x + (int64_t)k_lo * bb + nt * 8))
                            : make_uint4(0, 0, 0, 0);
            hi[i][nt] = (colsv && k_lo + 4 < kk)
                            ? __ldg(reinterpret_cast<const uint4*>(P.x + (int64_t)(k_lo + 4) * bb + nt * 8))
                            : make_uint4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int it = tid + (i0 + i) * kDhThreads;
          if (it >= nit) break;
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            if (nt * 8 >= bb) break;
            const uint32_t l4[4] = {lo[i][nt].x, lo[i][nt].y, lo[i][nt].z, lo[i][nt].w};
            const uint32_t h4[4] = {hi[i][nt].x, hi[i][nt].y, hi[i][nt].z, hi[i][nt].w};
#pragma unroll
            for (int cc = 0; cc < 8; ++cc) {
              const uint32_t lv = (cc & 1) ? (l4[cc >> 1] >> 16) : (l4[cc >> 1] & 0xFFFFu);
              const uint32_t hv = (cc & 1) ? (h4[cc >> 1] & 0xFFFF0000u) : (h4[cc >> 1] << 16);
              item_dst(it, cc)[nt * (kDhTileBytes / 4)] = lv | hv;
            }
          }
        }
      }
    } else {
      const unsigned short* xu = reinterpret_cast<const unsigned short*>(P.x);
      if (bb == 1) {  // a vector: all of a thread's loads first
        uint32_t lv[kItems], hv[kItems];
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
          const int it = tid + i * kDhThreads;
          const int k_lo = item_k(it);
          lv[i] = (it < nit && k_lo < kk) ? __ldg(xu + k_lo) : 0u;
          hv[i] = (it < nit && k_lo + 4 < kk) ? __ldg(xu + k_lo + 4) : 0u;
        }
#pragma unroll
        for (int i = 0; i < kItems; ++i) {
          const int it = tid + i * kDhThreads;
          if (it < nit) *item_dst(it, 0) = lv[i] | (hv[i] << 16);
        }
      } else {
#pragma unroll 1
        for (int i = 0; i < kItems; ++i) {
          const int it = tid + i * kDhThreads;
          if (it >= nit) break;
          const int k_lo = item_k(it), k_hi = k_lo + 4;
          const unsigned short* xl = xu + (int64_t)k_lo * bb;
          const unsigned short* xh = xu + (int64_t)k_hi * bb;
          for (int cc = 0; cc < bb; ++cc) {
            const uint32_t lv = k_lo < kk ? __ldg(xl + cc) : 0u;
            const uint32_t hv = k_hi < kk ? __ldg(xh + cc) : 0u;
            item_dst(it, cc & 7)[(cc >> 3) * (kDhTileBytes / 4)] = lv | (hv << 16);
          }
        }
      }
    }
    MSG_JITTER();
    __syncthreads();
    // ---- stream the chunks of this sub-slice, kDhDepth in flight
    for (int c = sub; c < sub_end; c += kDhDepth) {
#pragma unroll
      for (int u = 0; u < kDhDepth; ++u) {
        MSG_DASSERT(c + u - sub >= 0 && c + u - sub < kDhSub);
        const uint32_t xb = xs_lane + (uint32_t)((c + u - sub) * NT * kDhTileBytes);
#pragma unroll
        for (int v = 0; v < kDhNV; ++v) {
          const uint32_t wwa[4] = {wa[u][v].x, wa[u][v].y, wa[u][v].z, wa[u][v].w};
          const uint32_t wwb[4] = {wb[u][v].x, wb[u][v].y, wb[u][v].z, wb[u][v].w};
#pragma unroll
          for (int j4 = 0; j4 < 4; ++j4) {
            const int j = 4 * v + j4;
            uint4 xq[NT];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
              asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(xq[nt].x), "=r"(xq[nt].y), "=r"(xq[nt].z), "=r"(xq[nt].w)
                           : "r"(xb + nt * kDhTileBytes + 16 * ((uint32_t)j ^ swz)));
            uint32_t ha[4], hb[4];
            dh_dequant(wwa[j4], P.c, ha);
            dh_dequant(wwb[j4], P.c, hb);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              dh_mma(d[nt][0], ha[0], hb[0], ha[1], hb[1], xq[nt].x, xq[nt].y);
              dh_mma(d[nt][1], ha[2], hb[2], ha[3], hb[3], xq[nt].z, xq[nt].w);
            }
          }
        }
        if (c + u + kDhDepth < c_end) load_w(c + u + kDhDepth, wa[u], wb[u]);  // may belong to the next sub-slice
      }
    }
  }
  float dd[NT][4];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt)
#pragma unroll
    for (int i = 0; i < 4; ++i) dd[nt][i] = d[nt][0][i] + d[nt][1][i];

  // ---- output: direct from the fragments, or summed over the cluster's k slices
  const int S = (int)gridDim.y;
  auto store_y = [&](int64_t row, int col, float v) {
    if (row < P.m && col < P.b) {
      if (P.y_dtype == MSG_F16) reinterpret_cast<__half*>(P.y)[row * P.b + col] = __float2half_rn(v);
      else reinterpret_cast<float*>(P.y)[row * P.b + col] = v;
    }
  };
  if (S == 1) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      store_y(ra, nt * 8 + 2 * t, dd[nt][0]);
      store_y(ra, nt * 8 + 2 * t + 1, dd[nt][1]);
      store_y(rbw, nt * 8 + 2 * t, dd[nt][2]);
      store_y(rbw, nt * 8 + 2 * t + 1, dd[nt][3]);
    }
    return;
  }
  cg::cluster_group cl = cg::this_cluster();
  constexpr int NC = NT * 8;
  float* tile = reinterpret_cast<float*>(smem);  // [kDhRows][NC]
  MSG_JITTER();
  __syncthreads();  // X staging is consumed by every warp
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    float* r0 = tile + (warp * 16 + g) * NC + nt * 8 + 2 * t;
    *reinterpret_cast<float2*>(r0) = make_float2(dd[nt][0], dd[nt][1]);
    *reinterpret_cast<float2*>(r0 + 8 * NC) = make_float2(dd[nt][2], dd[nt][3]);
  }
  cl.sync();
  const int rows_per = (kDhRows + S - 1) / S;
  const int rank = (int)cl.block_rank();
  for (int i = tid; i < rows_per * NC; i += kDhThreads) {
    const int r = rank * rows_per + i / NC, col = i % NC;
    if (r >= kDhRows) break;
    MSG_DASSERT(r >= 0 && r < kDhRows && col < NC);
    float sum = 0.f;
    for (int s = 0; s < S; ++s) sum += cl.map_shared_rank(tile, s)[r * NC + col];
    store_y(row0 + r, col, sum);
  }
  cl.sync();  // no CTA exits while its tile may still be read
}

template <int NT>
static int launch_dh(DhParams& P, int S, cudaStream_t s) {
  const int smem = std::max(kDhSub * NT * kDhTileBytes, kDhRows * NT * 8 * 4);
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    MSG_CUDA_CHECK(cudaFuncSetAttribute(dq_hmma_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured_dev = dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)ceil_div(P.m, kDhRows), S, 1);
  cfg.blockDim = dim3(kDhThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = 1;
  attr[1].val.clusterDim.y = S;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = S > 1 ? 2 : 1;
  MSG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, dq_hmma_kernel<NT>, P));
  return MSG_OK;
}

// k slices per row block (cluster size): the smallest power of two <= 8 that
// puts about two CTAs on every SM (one wave: every warp's first kDhDepth
// chunks are in flight from the start), each slice at least one pipeline
// round.  Measured on one B200 (tools/dense_probe.py, MSG_DH_SPLIT forces a
// size): 8192^2 b = 1: S = 1 / 2 / 4 / 8 -> 22.7 / 14.7 / 11.9 / 15.8 us;
// 65536 x 8192 b = 8: 68.4 / 70.2 / 79.6 us for S = 1 / 2 / 4.
static int dh_choose_split(int64_t m, int nchunks) {
  if (const char* e = std::getenv("MSG_DH_SPLIT")) {
    const int S = std::atoi(e);
    if (S >= 1 && S <= 8) return std::min(S, std::max(1, nchunks));
  }
  const int64_t want = (int64_t)sm_count() * 3 / 2, rbk = ceil_div(m, kDhRows);
  int S = 1;
  while (S < 8 && rbk * S < want && nchunks / (2 * S) >= kDhDepth) S *= 2;
  return S;
}

}  // namespace msg

using namespace msg;

extern "C" int msg_dequant_hmma(const uint8_t* packed, int64_t m, int64_t k, const double* values,
                                const void* x, int x_dtype, int64_t b, void* y, int y_dtype,
                                void* stream) {
  if (x_dtype != MSG_F16)
    return fail(MSG_ERR_UNSUPPORTED, "the dense HMMA baseline takes fp16 activations");
  if (b < 1 || b > 16)
    return fail(MSG_ERR_UNSUPPORTED, "the dense HMMA baseline supports 1 <= b <= 16 (got %lld)", (long long)b);
  if (y_dtype != MSG_F32 && y_dtype != MSG_F16)
    return fail(MSG_ERR_UNSUPPORTED, "the dense HMMA baseline writes fp32 or fp16 Y");
  bool int4 = true, uint4 = true;
  for (int c = 0; c < 16; ++c) {
    int4 = int4 && values[c] == (double)(c < 8 ? c : c - 16);
    uint4 = uint4 && values[c] == (double)c;
  }
  if (!int4 && !uint4) return fail(MSG_ERR_UNSUPPORTED, "the dense HMMA baseline supports int4/uint4");
  if (row_bytes(k, 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(packed) & 15) != 0)
    return fail(MSG_ERR_UNSUPPORTED, "the dense HMMA baseline needs 16-byte aligned rows (k %% 32 == 0)");
  if (m == 0 || k == 0) return MSG_OK;
  if (k > (int64_t)1 << 30) return fail(MSG_ERR_UNSUPPORTED, "the dense HMMA baseline indexes k with 32 bits");
  DhParams P{};
  P.packed = packed;
  P.m = m;
  P.k = k;
  P.rb = row_bytes(k, 4);
  P.x = reinterpret_cast<const __half*>(x);
  P.b = (int)b;
  P.nchunks = (int)ceil_div(k, kDhChunk);
  const int S = dh_choose_split(m, P.nchunks);
  P.chunks_per_cta = (int)(ceil_div(ceil_div(P.nchunks, S), kDhDepth) * kDhDepth);
  // fp16 magic numbers as msg_dequant_gemv (msg_dense.cu)
  P.c.magic = int4 ? 0x64086408u : 0x64006400u;
  P.c.magic_hi = int4 ? 0x64806480u : 0x64006400u;
  const __half hs = __float2half_rn(int4 ? 1032.0f : 1024.0f);
  const __half hh = __float2half_rn(int4 ? -72.0f : -64.0f);
  P.c.sub2 = (uint32_t)__half_as_ushort(hs) * 0x10001u;
  P.c.sub_hi = (uint32_t)__half_as_ushort(hh) * 0x10001u;
  P.y = y;
  P.y_dtype = y_dtype;
  cudaStream_t s = as_stream(stream);
  return b <= 8 ? launch_dh<1>(P, S, s) : launch_dh<2>(P, S, s);
}
