// K4: dequantise-then-tcgen05.mma comparison kernel.
//
// The dense baseline the paper argues msGeMM against:
// Y = dequant(W) @ X with W int4 and X fp16, on the 5th-generation tensor
// cores.  Spec: naive_gemm(dense(pwm), X) (gemm.py:206-216,
// packing.py:191-198); the int4 -> fp16 dequantisation is exact and the
// tensor core accumulates in fp32.
//
// Per CTA: a 128-row tile of W (M = 128), the whole (padded) batch N = b,
// and a slice of K.  Each 64-wide K step:
//   * TMA bulk copies bring the repacked 128x64 int4 tile (4 KiB) and the
//     pre-swizzled fp16 X^T tile (N x 128 B) into a NS-deep smem ring;
//   * the 128 threads dequantise their row (magic-number fp16 conversion:
//     8 nibbles -> 4 half2 in 4 LOP3 + 4 HFMA2, K3 pre-permutes the nibbles)
//     straight into tensor memory (tcgen05.st, 32 columns per row per k
//     step): the A operand never touches shared memory, so at small b the
//     kernel is bound by the int4 weight stream, not by a 4x-inflated fp16
//     smem round trip;
//   * one thread issues 4 tcgen05.mma.kind::f16 (M128 x N x K16) with A from
//     TMEM, B (X^T, SW128 K-major) from smem and the fp32 accumulator in TMEM,
//     and commits to mbarriers that release the A buffer and the ring slot.
// The epilogue reads TMEM with tcgen05.ld (one warp per 32 rows) and writes
// fp32 k-split partials, reduced by the shared deterministic finish kernel.
#include <algorithm>

#include "msg_common.cuh"

namespace msg {

int launch_finish_plain(const float* partial, int S, int64_t m, int64_t b, void* y, int y_dtype,
                        cudaStream_t s);

constexpr int kMmaBM = 128, kMmaBK = 64;
constexpr int kMmaTileA = kMmaBM * kMmaBK / 2;  // 4096 packed bytes

static inline int64_t al256(int64_t v) { return (v + 255) / 256 * 256; }

struct MmaShape {
  int64_t mt, kt, npad;  // 128-row tiles, 64-wide k tiles, padded batch
};
static MmaShape mma_shape(int64_t m, int64_t k, int64_t b) {
  MmaShape s{};
  s.mt = (m + kMmaBM - 1) / kMmaBM;
  s.kt = (k + kMmaBK - 1) / kMmaBK;
  int64_t n = 16;
  while (n < b) n *= 2;
  s.npad = n;
  return s;
}

}  // namespace msg

extern "C" int64_t msg_mma_layout_bytes(int64_t m, int64_t k) {
  msg::MmaShape s = msg::mma_shape(m, k, 1);
  return s.mt * s.kt * msg::kMmaTileA;
}

namespace msg {

// repacked W: [mt][kt][128 rows][32 bytes]; within each 32-bit word the 8
// nibbles of k = 8q..8q+7 sit at positions (0,4,1,5,2,6,3,7) and are XORed
// with `xmask` (8 for two's-complement int4, so stored u = v + 8; 0 for uint4)
__global__ void repack_mma_kernel(const uint8_t* __restrict__ packed, int64_t m, int64_t k,
                                  int rb, int xmask, MmaShape S, uint8_t* __restrict__ out) {
  const int64_t nwords = S.mt * S.kt * kMmaBM * 8;  // 8 words per row per k tile
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nwords;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(t & 7);
    const int64_t rt = t >> 3;  // (mt, kt, row)
    const int r = (int)(rt % kMmaBM);
    const int64_t tile = rt / kMmaBM;
    const int64_t kti = tile % S.kt, mti = tile / S.kt;
    const int64_t i = mti * kMmaBM + r;
    uint32_t w = 0;
    const int pos[8] = {0, 4, 1, 5, 2, 6, 3, 7};
    for (int e = 0; e < 8; ++e) {
      const int64_t j = kti * kMmaBK + q * 8 + e;
      uint32_t c = 0;
      if (i < m && j < k) c = (packed[i * rb + (j >> 1)] >> ((j & 1) * 4)) & 0xF;
      w |= ((c ^ (uint32_t)xmask) & 0xF) << (4 * pos[e]);
    }
    reinterpret_cast<uint32_t*>(out)[t] = w;
  }
}

// X (k, b) fp16 row-major -> per k tile the K-major SWIZZLE_128B image of X^T:
// row n, 16-byte chunk c at (n/8)*1024 + (n%8)*128 + ((c ^ n%8) * 16)
__global__ void prep_xt_kernel(const __half* __restrict__ x, int64_t k, int64_t b, MmaShape S,
                               uint8_t* __restrict__ out) {
  const int64_t tile_bytes = S.npad * 128;
  const int64_t nchunks = S.kt * S.npad * 8;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nchunks;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(t & 7);
    const int64_t n = (t >> 3) % S.npad;
    const int64_t kti = (t >> 3) / S.npad;
    uint32_t wv[4];
    for (int e = 0; e < 4; ++e) {
      __half lo = __float2half(0.f), hi = __float2half(0.f);
      const int64_t j = kti * kMmaBK + c * 8 + 2 * e;
      if (n < b && j < k) lo = x[j * b + n];
      if (n < b && j + 1 < k) hi = x[(j + 1) * b + n];
      __half2 h2 = __halves2half2(lo, hi);
      wv[e] = *reinterpret_cast<uint32_t*>(&h2);
    }
    const int64_t off = kti * tile_bytes + (n >> 3) * 1024 + (n & 7) * 128 + ((c ^ (n & 7)) * 16);
    *reinterpret_cast<uint4*>(out + off) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
}

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)1 << 16) |  // start, LBO = 16 B
         ((uint64_t)(1024 >> 4) << 32) |                            // SBO = 1024 B (8-row group)
         ((uint64_t)1 << 46) |                                       // descriptor version (sm_100)
         ((uint64_t)2 << 61);                                        // SWIZZLE_128B
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::
                   "r"(smem_u32(bar))
               : "memory");
}
// A from tensor memory ("TS" form): [d], [a], b-desc
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// 32 consecutive columns of this thread's TMEM lane (warp-collective)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
      "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
      "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
      "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

struct MmaParams {
  const uint8_t* wt;   // repacked W tiles
  const uint8_t* xt;   // swizzled X^T tiles
  float* partial;      // [S][m][b]
  int64_t m, b, kt_total, kt_per_split;
  float sub_lo, sub_hi;  // dequant constants: v = h - sub (lo lanes), v = h/16 - sub (hi lanes)
};

constexpr int kNA = 3;  // dequantised A operand buffers (TMEM, 32 columns each; 3 keeps N<=32 at 128 columns = 4 CTAs/SM)

template <int N> constexpr uint32_t dq_acc_cols() { return N < 32 ? 32 : N; }
template <int N> constexpr uint32_t dq_tmem_cols() {
  constexpr uint32_t need = dq_acc_cols<N>() + kNA * 32;
  return need <= 32 ? 32 : need <= 64 ? 64 : need <= 128 ? 128 : need <= 256 ? 256 : 512;
}

// Warp-specialised pipeline (256 threads):
//   warp 0 lane 0  : TMA producer -- packed W tile + swizzled X^T tile per k step
//                    into an NS-deep ring (full/empty mbarriers);
//   warp 1 lane 0  : MMA issuer   -- 4 x tcgen05.mma (K=16, A from TMEM) per k
//                    step, commits release the A buffer and the ring slot;
//   warp 2         : TMEM allocator;
//   warps 4..7     : dequantisers -- one row each (TMEM lane = row), int4 -> fp16
//                    (magic numbers) into one of kNA TMEM A buffers; afterwards
//                    the TMEM -> register -> global epilogue (warp w owns TMEM
//                    lanes 32*(w%4)..+31).
template <int N, int NS>
__global__ void __launch_bounds__(256, 1) dq_mma_kernel(MmaParams P) {
  constexpr int TB = N * 128;  // B tile bytes
  constexpr uint32_t kA0 = dq_acc_cols<N>();  // first A column (accumulator: [0, N))
  constexpr uint32_t kCols = dq_tmem_cols<N>();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* stB = smem;                              // [NS][TB]
  uint8_t* stA = stB + NS * TB;                     // [NS][4 KiB]
  uint64_t* full = reinterpret_cast<uint64_t*>(stA + NS * kMmaTileA);  // [NS] TMA landed
  uint64_t* empty = full + NS;                      // [NS] slot consumed (MMA + dequant)
  uint64_t* afull = empty + NS;                     // [kNA] operand written
  uint64_t* aempty = afull + kNA;                   // [kNA] operand consumed by MMA
  uint64_t* accf = aempty + kNA;                    // accumulator complete
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t mt = blockIdx.x, split = blockIdx.y;
  const int64_t kt0 = split * P.kt_per_split;
  const int64_t kt1 = std::min<int64_t>(P.kt_total, kt0 + P.kt_per_split);
  const int nloc = (int)std::max<int64_t>(0, kt1 - kt0);

  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1 + 128);  // MMA commit + 128 dequant threads
    }
    for (int i = 0; i < kNA; ++i) {
      mbar_init(&afull[i], 128);
      mbar_init(&aempty[i], 1);
    }
    mbar_init(accf, 1);
    fence_mbar_init();
  }
  tc_fence_before();
  MSG_JITTER();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      for (int i = 0; i < nloc; ++i) {
        const int slot = i % NS;
        if (i >= NS) mbar_wait(&empty[slot], (uint32_t)(((i / NS) - 1) & 1));
        const int64_t kt = kt0 + i;
        mbar_expect_tx(&full[slot], kMmaTileA + TB);
        bulk_g2s(stA + slot * kMmaTileA, P.wt + (mt * P.kt_total + kt) * kMmaTileA, kMmaTileA,
                 &full[slot]);
        bulk_g2s(stB + slot * TB, P.xt + kt * TB, TB, &full[slot]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc =
          (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      for (int i = 0; i < nloc; ++i) {
        const int slot = i % NS, buf = i % kNA;
        mbar_wait(&full[slot], (uint32_t)((i / NS) & 1));  // B tile landed (TMA)
        mbar_wait(&afull[buf], (uint32_t)((i / kNA) & 1));  // A written to TMEM
        tc_fence_after();
        const uint32_t ta = tmem + kA0 + (uint32_t)buf * 32;
        const uint64_t bd = umma_desc_sw128(smem_u32(stB + slot * TB));
#pragma unroll
        for (int ks = 0; ks < kMmaBK / 16; ++ks)  // K = 16 per instruction = 8 TMEM columns
          mma_f16_ts(tmem, ta + 8 * ks, bd + 2 * ks, idesc, (i > 0 || ks > 0) ? 1u : 0u);
        mma_commit(&aempty[buf]);
        mma_commit(&empty[slot]);
      }
      if (nloc > 0) mma_commit(accf);
    }
  } else if (warp >= 4) {
    // ---------------- dequantisers, then epilogue
    const int quarter = warp & 3;
    const int r = tid - 128;  // tile row = TMEM lane
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const __half2 sub_lo = __float2half2_rn(P.sub_lo);
    const __half2 sub_hi = __float2half2_rn(P.sub_hi);
    const __half2 sixteenth = __float2half2_rn(1.0f / 16.0f);
    for (int i = 0; i < nloc; ++i) {
      const int slot = i % NS, buf = i % kNA;
      mbar_wait(&full[slot], (uint32_t)((i / NS) & 1));
      const uint4* src = reinterpret_cast<const uint4*>(stA + slot * kMmaTileA + r * 32);
      const uint4 p0 = src[0], p1 = src[1];
      mbar_arrive(&empty[slot]);  // packed A copied out
      const uint32_t words[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
      uint32_t o[32];  // column 4c + j holds k = 8c + 2j, 8c + 2j + 1 (lo, hi)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t w = words[c];
        uint32_t h[4];
        h[0] = (w & 0x000F000Fu) | 0x64006400u;
        h[1] = (w & 0x00F000F0u) | 0x64006400u;
        w >>= 8;
        h[2] = (w & 0x000F000Fu) | 0x64006400u;
        h[3] = (w & 0x00F000F0u) | 0x64006400u;
        __half2 v0 = __hsub2(*reinterpret_cast<__half2*>(&h[0]), sub_lo);
        __half2 v1 = __hfma2(*reinterpret_cast<__half2*>(&h[1]), sixteenth, sub_hi);
        __half2 v2 = __hsub2(*reinterpret_cast<__half2*>(&h[2]), sub_lo);
        __half2 v3 = __hfma2(*reinterpret_cast<__half2*>(&h[3]), sixteenth, sub_hi);
        o[4 * c + 0] = *reinterpret_cast<uint32_t*>(&v0);
        o[4 * c + 1] = *reinterpret_cast<uint32_t*>(&v1);
        o[4 * c + 2] = *reinterpret_cast<uint32_t*>(&v2);
        o[4 * c + 3] = *reinterpret_cast<uint32_t*>(&v3);
      }
      if (i >= kNA) mbar_wait(&aempty[buf], (uint32_t)(((i / kNA) - 1) & 1));
      tc_fence_after();
      tmem_st32(tmem + lane_base + kA0 + (uint32_t)buf * 32, o);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&afull[buf]);
    }
    // ---------------- epilogue: TMEM -> registers -> fp32 partials
    const int64_t row = mt * kMmaBM + quarter * 32 + lane;
    float* dst = P.partial + (split * P.m + row) * P.b;
    if (nloc > 0) {
      mbar_wait(accf, 0);
      tc_fence_after();
#pragma unroll
      for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + lane_base + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"
            "%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
              "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
              "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < P.m) {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (c0 + e < P.b) dst[c0 + e] = __uint_as_float(v[e]);
        }
      }
    } else if (row < P.m) {
      for (int64_t e = 0; e < P.b; ++e) dst[e] = 0.f;
    }
  }
  tc_fence_before();
  MSG_JITTER();
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
}

template <int N, int NS>
constexpr int dq_smem() {
  return 1024 + NS * (N * 128 + kMmaTileA) + (2 * NS + 2 * kNA + 1) * 8 + 16;
}

// CTAs per SM: shared memory and tensor memory (512 columns) both bound it
template <int N, int NS>
constexpr int dq_per_sm() {
  const int by_smem = (227 * 1024) / dq_smem<N, NS>();
  const int by_tmem = 512 / (int)dq_tmem_cols<N>();
  const int v = by_smem < by_tmem ? by_smem : by_tmem;
  return v < 1 ? 1 : (v > 4 ? 4 : v);
}

template <int N, int NS>
static int launch_dq(const MmaParams& P, const MmaShape& S, int splits, cudaStream_t s) {
  // request enough shared memory that no more CTAs than TMEM can serve are resident
  const int smem = std::max(dq_smem<N, NS>(), (227 * 1024) / (dq_per_sm<N, NS>() + 1) + 1024);
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    MSG_CUDA_CHECK(cudaFuncSetAttribute(dq_mma_kernel<N, NS>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured_dev = dev;
  }
  dim3 grid((unsigned)S.mt, (unsigned)splits);
  dq_mma_kernel<N, NS><<<grid, 256, smem, s>>>(P);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}

constexpr int kDqStages = 6;

static int dq_per_sm_for(int64_t npad) {
  switch (npad) {
    case 16: return dq_per_sm<16, kDqStages>();
    case 32: return dq_per_sm<32, kDqStages>();
    case 64: return dq_per_sm<64, kDqStages>();
    case 128: return dq_per_sm<128, kDqStages>();
  }
  return dq_per_sm<256, kDqStages>();
}

// k-splits: enough CTAs to fill every SM with as many resident CTAs as shared
// memory allows (up to 4), each split at least 4 k tiles long
static int mma_splits(const MmaShape& S) {
  const int per_sm = dq_per_sm_for(S.npad);
  int64_t sp = std::max<int64_t>(1, (int64_t)sm_count() * per_sm / std::max<int64_t>(1, S.mt));
  return (int)std::min<int64_t>(sp, std::max<int64_t>(1, S.kt / 4));
}

}  // namespace msg

using namespace msg;

extern "C" int64_t msg_dequant_mma_workspace_bytes(int64_t m, int64_t k, int64_t b) {
  MmaShape S = mma_shape(m, k, b);
  const int sp = mma_splits(S);
  return al256(S.kt * S.npad * 128) + al256((int64_t)sp * m * b * 4);
}

extern "C" int msg_dequant_mma(const uint8_t* wmma, int64_t m, int64_t k, const double* values,
                               const void* x, int x_dtype, int64_t b, void* y, int y_dtype,
                               void* workspace, int64_t ws_bytes, void* stream) {
  if (x_dtype != MSG_F16)
    return fail(MSG_ERR_UNSUPPORTED, "the dequant-MMA comparison kernel takes fp16 activations");
  if (b < 1 || b > 256)
    return fail(MSG_ERR_UNSUPPORTED, "dequant-MMA supports 1 <= b <= 256 (got %lld)", (long long)b);
  // int4 (two's complement) or uint4 alphabets: v = u - off with u the stored nibble
  double off;
  bool int4 = true, uint4 = true;
  for (int c = 0; c < 16; ++c) {
    int4 = int4 && values[c] == (double)(c < 8 ? c : c - 16);
    uint4 = uint4 && values[c] == (double)c;
  }
  if (int4) off = 8.0;
  else if (uint4) off = 0.0;
  else return fail(MSG_ERR_UNSUPPORTED, "dequant-MMA supports the int4/uint4 codebooks");
  if (ws_bytes < msg_dequant_mma_workspace_bytes(m, k, b))
    return fail(MSG_ERR_WORKSPACE, "workspace too small for dequant-MMA");
  if (m == 0) return MSG_OK;
  cudaStream_t s = as_stream(stream);
  MmaShape S = mma_shape(m, k, b);
  const int splits = mma_splits(S);
  uint8_t* xt = reinterpret_cast<uint8_t*>(workspace);
  float* partial = reinterpret_cast<float*>((char*)workspace + al256(S.kt * S.npad * 128));
  {
    const int64_t n = S.kt * S.npad * 8;
    const int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)sm_count() * 8);
    prep_xt_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const __half*>(x), k, b, S, xt);
    MSG_LAUNCH_CHECK();
  }
  MmaParams P{};
  P.wt = wmma;
  P.xt = xt;
  P.partial = partial;
  P.m = m;
  P.b = b;
  P.kt_total = S.kt;
  P.kt_per_split = ceil_div(S.kt, splits);
  // magic-number dequant: (1024 + u) - (1024 + off); (1024*16 + 16u)/16 - (1024 + off)
  P.sub_lo = (float)(1024.0 + off);
  P.sub_hi = (float)(-(64.0 + off));
  int e;
  switch (S.npad) {
    case 16: e = launch_dq<16, kDqStages>(P, S, splits, s); break;
    case 32: e = launch_dq<32, kDqStages>(P, S, splits, s); break;
    case 64: e = launch_dq<64, kDqStages>(P, S, splits, s); break;
    case 128: e = launch_dq<128, kDqStages>(P, S, splits, s); break;
    default: e = launch_dq<256, kDqStages>(P, S, splits, s); break;
  }
  if (e) return e;
  return launch_finish_plain(partial, splits, m, b, y, y_dtype, s);
}

extern "C" int msg_repack_mma(const uint8_t* packed, int64_t m, int64_t k,
                              const double* values, uint8_t* out, void* stream) {
  bool int4 = true, uint4 = true;
  for (int c = 0; c < 16; ++c) {
    int4 = int4 && values[c] == (double)(c < 8 ? c : c - 16);
    uint4 = uint4 && values[c] == (double)c;
  }
  if (!int4 && !uint4)
    return fail(MSG_ERR_UNSUPPORTED, "dequant-MMA supports the int4/uint4 codebooks");
  const int xmask = int4 ? 8 : 0;
  cudaStream_t s = as_stream(stream);
  MmaShape S = mma_shape(m, k, 1);
  const int64_t n = S.mt * S.kt * kMmaBM * 8;
  if (n == 0) return MSG_OK;
  const int grid = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)sm_count() * 16);
  repack_mma_kernel<<<grid, 256, 0, s>>>(packed, m, k, row_bytes(k, 4), xmask, S, out);
  MSG_LAUNCH_CHECK();
  return MSG_OK;
}
