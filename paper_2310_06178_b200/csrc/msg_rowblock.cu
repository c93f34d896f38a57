// Row-block msGeMM kernel for the batched case: d = 3, fp16 activations,
// sign-symmetric fp16 half tables, 2 <= b (column tiles of BC = 2, 4, 8).
//
// Reference semantics: gemm.py:89-153 (msgemm), gemm.py:70-86 (row sum, k%d
// tail, per-row scale -- the tail and scales are applied by the finish
// kernel of msg_fused.cu), lut.py:59-72 (table entries), packing.py:201-228
// (group index, first code least significant).
//
// Design (sm_100a, one 512-thread CTA per SM, 128 KiB of tables):
//   * A round holds G = 32 / BC groups.  Their G half tables (2048 fp16
//     entries of BC columns each, H[f] = sum_r (v[c_r] - beta) x_r for the
//     folded 11-bit index f) are interleaved so that entry f of table t sits
//     at byte 64 f + t EB (EB = 2 BC bytes): table t owns two bank slots of
//     every 128-byte row, and one shared-memory wavefront phase (8 lanes for
//     LDS.128, 16 for LDS.64, 32 for LDS.32) reaches G tables with 2 lanes
//     each -- measured (tools/microbench/lds_conflicts.cu) 1.94 wavefronts per
//     phase for random entries, against 2.6 for an unstructured table.
//   * K3 (repack_rb_kernel) stores, per row and quad of groups, 48 bits:
//     four 11-bit folded indices (the sign-symmetry complement folded in) and
//     four sign bits, ordered so that position p of row i holds group
//     (p + i) mod G of its round -- lane l of a phase hits table (p + l) mod G
//     -- and so that every byte address is one shift (or funnel shift) and one
//     LOP3: ((word >> s) & 0x1FFC0) | slot.
//   * Weight words go HBM -> registers with coalesced loads (lanes own
//     consecutive rows), prefetched one round ahead in place: no staging
//     buffer, so shared memory only carries the table build (STS) and the
//     gathers (LDS).
//   * The gather accumulates fp32 += fp16 * (+-1) with FHFMA; k-slice
//     partials go to the workspace [S][m][b] and msg_fused.cu's finish kernel
//     sums them in slice order (deterministic), adds the k%d tail and the
//     per-row scale and casts to Y's dtype.
#include <algorithm>

#include "msg_common.cuh"

namespace msg {

struct TailVals;
int launch_finish(const float* partial, int S, int64_t m, int64_t b, int64_t k, int d,
                  const uint16_t* tailp, const TailVals& tv, const void* x, int x_dtype,
                  int scale_mode, const void* q, int q_dtype, void* y, int y_dtype,
                  cudaStream_t s);

static inline int64_t al256(int64_t v) { return (v + 255) / 256 * 256; }

// ============================================================================
// K3: row-block layout
// ============================================================================
struct RbLayout {
  int64_t nb, nq, nqp, mp;              // groups, quads, quads padded to rounds, row stride
  int64_t lo_off, hi_off, rot_off, tail_off, total;
  int G, tail;
  int rpt;                              // G = 4: rows per thread of the kernel (16 or 8)
};

// G = 4 comes in two variants: 16 rows per thread (8192 rows per CTA) or 8
// (4096 rows per CTA, for row counts that would leave most of an 8192-row
// block idle or whose fixed k-slice partial traffic would dominate)
RbLayout rb_layout(int64_t m, int64_t k, int G, int rpt = 16) {
  RbLayout L{};
  L.G = G;
  L.rpt = rpt;
  L.nb = k / 3;
  L.nq = (L.nb + 3) / 4;
  const int qr = G / 4;
  L.nqp = (L.nq + qr - 1) / qr * qr;
  L.mp = (m + 31) / 32 * 32;
  L.tail = (int)(k - L.nb * 3);
  L.lo_off = 0;
  L.hi_off = al256(L.nqp * L.mp * 4);
  L.rot_off = L.hi_off + al256(L.nqp * L.mp * 2);
  // G = 4: per (quad, rpt-row group) the rotations chosen by K3 (2 bits per row)
  L.tail_off = L.rot_off + (G == 4 ? al256(L.nqp * (L.mp / rpt) * 4) : 0);
  L.total = L.tail_off + (L.tail ? al256(m * 2) : 0);
  if (L.total == 0) L.total = 256;
  return L;
}

constexpr int kRpTileRows = 32, kRpTileQuads = 16;  // K3 tile: 32 rows x 16 quads (96 B per row)
constexpr int kRbThreads = 512;
// rows per thread: rounds of 4 groups keep their accumulators in tensor
// memory (16 rows x 8 columns per thread, 8192 rows per CTA); the others in
// registers
__host__ __device__ constexpr int rb_rows_per_thread(int G) { return G == 4 ? 16 : (G == 16 ? 4 : 8); }

// One CTA per (32-row, 16-quad) tile: the tile's packed bytes are read with
// coalesced loads into shared memory, then every thread forms two (row, quad)
// records and writes them to the [quad][row] planes (consecutive rows ->
// coalesced stores).  Position p of row i holds group (p + i) mod G of its
// round; indices with the top bit set are stored complemented + sign bit.
__global__ void __launch_bounds__(256) repack_rb_kernel(const uint8_t* __restrict__ packed,
                                                        int64_t m, int64_t k, int rb, RbLayout L,
                                                        uint8_t* __restrict__ out) {
  __shared__ uint8_t tile[kRpTileRows][kRpTileQuads * 6 + 4];
  const int64_t ntr = (m + kRpTileRows - 1) / kRpTileRows;
  const int64_t ntq = (L.nqp + kRpTileQuads - 1) / kRpTileQuads;
  const int G = L.G;
  for (int64_t tt = blockIdx.x; tt < ntr * ntq; tt += gridDim.x) {
    const int64_t i0 = (tt % ntr) * kRpTileRows, q0 = (tt / ntr) * kRpTileQuads;
    const int64_t b0 = q0 * 6;  // first byte of the tile in a row
    MSG_JITTER();
    __syncthreads();
    if ((rb & 3) == 0) {  // 4-byte loads (b0 is a multiple of 4: q0 is a multiple of 16)
      for (int e = threadIdx.x; e < kRpTileRows * 24; e += 256) {
        const int r = e / 24, w = e % 24;
        const int64_t i = i0 + r, by = b0 + 4 * w;
        uint32_t v = 0;
        if (i < m && by < rb) v = *reinterpret_cast<const uint32_t*>(packed + i * rb + by);
        *reinterpret_cast<uint32_t*>(&tile[r][4 * w]) = v;
      }
    } else {
      for (int e = threadIdx.x; e < kRpTileRows * 96; e += 256) {
        const int r = e / 96, c = e % 96;
        const int64_t i = i0 + r, by = b0 + c;
        tile[r][c] = (i < m && by < rb) ? packed[i * rb + by] : 0;
      }
    }
    MSG_JITTER();
    __syncthreads();
    for (int e = threadIdx.x; e < kRpTileRows * kRpTileQuads; e += 256) {
      const int r = e % kRpTileRows, qq = e / kRpTileRows;
      const int64_t i = i0 + r, q = q0 + qq;
      if (i >= L.mp || q >= L.nqp) continue;
      // G, rows per thread and rows per CTA are powers of two: shifts and masks
      const int lg = G == 8 ? 3 : 4;                   // log2 G (G = 8 or 16 here)
      const int lrpt = G == 8 ? 3 : 2;                 // log2 rb_rows_per_thread(G)
      const int64_t round = q >> (lg - 2);
      const int qin = (int)(q & ((G >> 2) - 1));
      // lanes own rows: thread tid of a CTA holds rows tid * RPT .. + RPT - 1 of
      // its row block, and its position p looks up group (p + tid) mod G
      const int lane = (int)((i & ((int64_t)kRbThreads << lrpt) - 1) >> lrpt);
      uint32_t f[4] = {0, 0, 0, 0}, sg[4] = {0, 0, 0, 0};
      if (i < m) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const int p = 4 * qin + s;
          const int g = (p + lane) & (G - 1);          // group of this position in the round
          const int64_t j = round * G + g;             // global group
          if (j >= L.nb) continue;
          const int lq = (int)(j / 4 - q0);            // its quad inside this tile
          const int c0 = (int)(j % 4) * 3;             // first code inside that quad
          uint32_t idx = 0;
          for (int t = 0; t < 3; ++t) {
            const int c = c0 + t;
            idx |= ((tile[r][lq * 6 + (c >> 1)] >> ((c & 1) * 4)) & 0xF) << (4 * t);
          }
          if (idx & 0x800) { idx ^= 0xFFF; sg[s] = 1; }
          f[s] = idx;
        }
      }
      const uint32_t lo = f[0] | (f[1] << 11) | ((f[2] & 0x3FF) << 22);
      const uint32_t hi = (f[2] >> 10) | (f[3] << 1) | (sg[0] << 12) | (sg[1] << 13) |
                          (sg[2] << 14) | (sg[3] << 15);
      reinterpret_cast<uint32_t*>(out + L.lo_off)[q * L.mp + i] = lo;
      reinterpret_cast<uint16_t*>(out + L.hi_off)[q * L.mp + i] = (uint16_t)hi;
    }
  }
}

// ---------------------------------------------------------------------------
// K3 for rounds of 4 groups (b >= 8): conflict-aware rotations.  One LDS.128
// wavefront phase is 8 lanes (a quarter warp) = 8 threads holding rows
// i_u = base + 16 u + r (u = 0..7) at row step r.  Table t occupies bank slots
// {t, t + 4} of every 128-byte row, chosen by the parity of the folded index,
// so a phase is conflict-free when every table is hit by two lanes of
// opposite parity.  Lane u reads group (s + rho_u) mod 4 at position s; K3
// picks the rotations per (octet, row step, quad): lanes are paired (105
// pairings), each pair gets its own rotation (24 permutations), and the
// chosen assignment minimises the positions at which some pair reads its
// table with equal parities (the 8 pairings with the fewest equal-parity
// tables are searched; measured by simulation 1.55 wavefronts per phase on
// uniform random weights against 1.94 for the fixed rotation rho_u = u mod 4).
__constant__ uint32_t kPairings[105] = {
    0x76543210u, 0x75643210u, 0x65743210u, 0x76534210u, 0x75634210u, 0x65734210u,
    0x76435210u, 0x74635210u, 0x64735210u, 0x75436210u, 0x74536210u, 0x54736210u,
    0x65437210u, 0x64537210u, 0x54637210u, 0x76543120u, 0x75643120u, 0x65743120u,
    0x76534120u, 0x75634120u, 0x65734120u, 0x76435120u, 0x74635120u, 0x64735120u,
    0x75436120u, 0x74536120u, 0x54736120u, 0x65437120u, 0x64537120u, 0x54637120u,
    0x76542130u, 0x75642130u, 0x65742130u, 0x76524130u, 0x75624130u, 0x65724130u,
    0x76425130u, 0x74625130u, 0x64725130u, 0x75426130u, 0x74526130u, 0x54726130u,
    0x65427130u, 0x64527130u, 0x54627130u, 0x76532140u, 0x75632140u, 0x65732140u,
    0x76523140u, 0x75623140u, 0x65723140u, 0x76325140u, 0x73625140u, 0x63725140u,
    0x75326140u, 0x73526140u, 0x53726140u, 0x65327140u, 0x63527140u, 0x53627140u,
    0x76432150u, 0x74632150u, 0x64732150u, 0x76423150u, 0x74623150u, 0x64723150u,
    0x76324150u, 0x73624150u, 0x63724150u, 0x74326150u, 0x73426150u, 0x43726150u,
    0x64327150u, 0x63427150u, 0x43627150u, 0x75432160u, 0x74532160u, 0x54732160u,
    0x75423160u, 0x74523160u, 0x54723160u, 0x75324160u, 0x73524160u, 0x53724160u,
    0x74325160u, 0x73425160u, 0x43725160u, 0x54327160u, 0x53427160u, 0x43527160u,
    0x65432170u, 0x64532170u, 0x54632170u, 0x65423170u, 0x64523170u, 0x54623170u,
    0x65324170u, 0x63524170u, 0x53624170u, 0x64325170u, 0x63425170u, 0x43625170u,
    0x54326170u, 0x53426170u, 0x43526170u,
};
__constant__ uint8_t kPerms[24] = {0xe4, 0xb4, 0xd8, 0x78, 0x9c, 0x6c, 0xe1, 0xb1, 0xc9, 0x39, 0x8d, 0x2d,
                                   0xd2, 0x72, 0xc6, 0x36, 0x4e, 0x1e, 0x93, 0x63, 0x87, 0x27, 0x4b, 0x1b};

__device__ __forceinline__ uint32_t rotr4(uint32_t m, int r) { return ((m >> r) | (m << (4 - r))) & 0xF; }

constexpr int kRb4Cands = 4;  // pairings searched (simulated: top-4 matches top-8, 1.55 wavefronts)

// rotations (2 bits per lane) of one octet from the lanes' 4-bit parity masks
// pmw (lane u at bits 4u..4u+3).  The kRb4Cands pairings with the fewest
// equal-parity (pair, table) incidences are searched over the 24 rotation
// permutations (ties: earlier pairings first).
//
// the 4 lane pairs of every pairing as indices into the 28 pairs (a < b),
// pair (a, b) -> a (15 - a) / 2 + b - a - 1 (compile-time copy of kPairings)
__host__ __device__ constexpr int pair_idx(int p, int i) {
  constexpr uint8_t t[105][4] = {
    {0, 13, 22, 27}, {0, 13, 23, 26}, {0, 13, 24, 25}, {0, 14, 19, 27}, {0, 14, 20, 26}, {0, 14, 21, 25},
    {0, 15, 18, 27}, {0, 15, 20, 24}, {0, 15, 21, 23}, {0, 16, 18, 26}, {0, 16, 19, 24}, {0, 16, 21, 22},
    {0, 17, 18, 25}, {0, 17, 19, 23}, {0, 17, 20, 22}, {1, 8, 22, 27}, {1, 8, 23, 26}, {1, 8, 24, 25},
    {1, 9, 19, 27}, {1, 9, 20, 26}, {1, 9, 21, 25}, {1, 10, 18, 27}, {1, 10, 20, 24}, {1, 10, 21, 23},
    {1, 11, 18, 26}, {1, 11, 19, 24}, {1, 11, 21, 22}, {1, 12, 18, 25}, {1, 12, 19, 23}, {1, 12, 20, 22},
    {2, 7, 22, 27}, {2, 7, 23, 26}, {2, 7, 24, 25}, {2, 9, 15, 27}, {2, 9, 16, 26}, {2, 9, 17, 25},
    {2, 10, 14, 27}, {2, 10, 16, 24}, {2, 10, 17, 23}, {2, 11, 14, 26}, {2, 11, 15, 24}, {2, 11, 17, 22},
    {2, 12, 14, 25}, {2, 12, 15, 23}, {2, 12, 16, 22}, {3, 7, 19, 27}, {3, 7, 20, 26}, {3, 7, 21, 25},
    {3, 8, 15, 27}, {3, 8, 16, 26}, {3, 8, 17, 25}, {3, 10, 13, 27}, {3, 10, 16, 21}, {3, 10, 17, 20},
    {3, 11, 13, 26}, {3, 11, 15, 21}, {3, 11, 17, 19}, {3, 12, 13, 25}, {3, 12, 15, 20}, {3, 12, 16, 19},
    {4, 7, 18, 27}, {4, 7, 20, 24}, {4, 7, 21, 23}, {4, 8, 14, 27}, {4, 8, 16, 24}, {4, 8, 17, 23},
    {4, 9, 13, 27}, {4, 9, 16, 21}, {4, 9, 17, 20}, {4, 11, 13, 24}, {4, 11, 14, 21}, {4, 11, 17, 18},
    {4, 12, 13, 23}, {4, 12, 14, 20}, {4, 12, 16, 18}, {5, 7, 18, 26}, {5, 7, 19, 24}, {5, 7, 21, 22},
    {5, 8, 14, 26}, {5, 8, 15, 24}, {5, 8, 17, 22}, {5, 9, 13, 26}, {5, 9, 15, 21}, {5, 9, 17, 19},
    {5, 10, 13, 24}, {5, 10, 14, 21}, {5, 10, 17, 18}, {5, 12, 13, 22}, {5, 12, 14, 19}, {5, 12, 15, 18},
    {6, 7, 18, 25}, {6, 7, 19, 23}, {6, 7, 20, 22}, {6, 8, 14, 25}, {6, 8, 15, 23}, {6, 8, 16, 22},
    {6, 9, 13, 25}, {6, 9, 15, 20}, {6, 9, 16, 19}, {6, 10, 13, 23}, {6, 10, 14, 20}, {6, 10, 16, 18},
    {6, 11, 13, 22}, {6, 11, 14, 19}, {6, 11, 15, 18}};
  return t[p][i];
}
__host__ __device__ constexpr uint32_t perm_code(int q) {
  constexpr uint8_t t[24] = {0xe4, 0xb4, 0xd8, 0x78, 0x9c, 0x6c, 0xe1, 0xb1, 0xc9, 0x39, 0x8d, 0x2d, 0xd2, 0x72, 0xc6, 0x36, 0x4e, 0x1e, 0x93, 0x63, 0x87, 0x27, 0x4b, 0x1b};
  return t[q];
}

// pairing P's score (equal-parity incidences) into the running top 4, kept
// in registers sorted by score (ties: earlier pairings first) with predicated
// compare-and-swaps -- no shared memory, no divergent insertion loop; template
// recursion so every pair index is a compile-time constant (pc stays in registers)
struct Top4 { int s0, s1, s2, s3, c0, c1, c2, c3; };
template <int P>
__device__ __forceinline__ void score_pairings(const int (&pc)[28], Top4& t) {
  if constexpr (P < 105) {
    const int sc = pc[pair_idx(P, 0)] + pc[pair_idx(P, 1)] + pc[pair_idx(P, 2)] + pc[pair_idx(P, 3)];
    if (sc < t.s3) {
      t.s3 = sc; t.c3 = P;
      if (t.s3 < t.s2) {
        int x = t.s2; t.s2 = t.s3; t.s3 = x; x = t.c2; t.c2 = t.c3; t.c3 = x;
        if (t.s2 < t.s1) {
          x = t.s1; t.s1 = t.s2; t.s2 = x; x = t.c1; t.c1 = t.c2; t.c2 = x;
          if (t.s1 < t.s0) { x = t.s0; t.s0 = t.s1; t.s1 = x; x = t.c0; t.c0 = t.c1; t.c1 = x; }
        }
      }
    }
    score_pairings<P + 1>(pc, t);
  }
}

template <int Q>
__device__ __forceinline__ void best_perm(const uint32_t (&rm)[4], int& cbest, int& qbest) {
  if constexpr (Q < 24) {
    constexpr uint32_t pr = perm_code(Q);
    const uint32_t u = (rm[0] >> (4 * (pr & 3))) | (rm[1] >> (4 * ((pr >> 2) & 3))) |
                       (rm[2] >> (4 * ((pr >> 4) & 3))) | (rm[3] >> (4 * (pr >> 6)));
    const int cost = __popc(u & 0xF);
    if (cost < cbest) { cbest = cost; qbest = Q; }
    best_perm<Q + 1>(rm, cbest, qbest);
  }
}

__device__ uint32_t choose_rotations(uint32_t pmw) {
  // equal-parity count of every lane pair, once (the 105 pairings reuse them)
  int pc[28];
#pragma unroll
  for (int a = 0, n = 0; a < 8; ++a)
#pragma unroll
    for (int b = a + 1; b < 8; ++b, ++n) pc[n] = __popc(~((pmw >> (4 * a)) ^ (pmw >> (4 * b))) & 0xF);
  static_assert(kRb4Cands == 4, "the register top-K keeps 4 candidates");
  Top4 t{99, 99, 99, 99, 0, 0, 0, 0};
  score_pairings<0>(pc, t);
  const int cand[4] = {t.c0, t.c1, t.c2, t.c3};
  int best = 99;
  uint32_t best_rho = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t code = kPairings[cand[c]];
    uint32_t rm[4];  // the pair's bad-position mask under rotation r at bits 4r..4r+3
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t a = (code >> (8 * i)) & 0xF, b = (code >> (8 * i + 4)) & 0xF;
      const uint32_t bad = ~((pmw >> (4 * a)) ^ (pmw >> (4 * b))) & 0xF;
      rm[i] = bad | (rotr4(bad, 1) << 4) | (rotr4(bad, 2) << 8) | (rotr4(bad, 3) << 12);
    }
    int cbest = 99, qbest = 0;
    best_perm<0>(rm, cbest, qbest);
    if (cbest < best) {
      best = cbest;
      const uint32_t pr = kPerms[qbest];
      uint32_t rho = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t a = (code >> (8 * i)) & 0xF, b = (code >> (8 * i + 4)) & 0xF;
        const uint32_t ri = (pr >> (2 * i)) & 3;
        rho |= (ri << (2 * a)) | (ri << (2 * b));
      }
      best_rho = rho;
    }
  }
  return best_rho;
}

// K3 for rounds of 4 groups.  One CTA per (128-row block, 8 quads): the
// block's packed bytes (48 per row) are staged with coalesced loads, then
// thread (r, sub, qq) takes row step r of quad qq for the octet of rows
// base + 8 RPT sub + RPT u + r (u < 8) -- the 8 lanes of one LDS.128 phase of
// the kernel, whose thread t holds rows RPT t .. RPT t + RPT - 1 -- its
// rotations and its 8 (lo, hi) records; the per-(quad, RPT-row group)
// rotation words are assembled from shared memory.
constexpr int kRb4Rows = 128, kRb4Quads = 8;
template <int RPT>
__global__ void __launch_bounds__(128) repack_rb4_kernel(const uint8_t* __restrict__ packed,
                                                         int64_t m, int64_t k, int rb, RbLayout L,
                                                         uint8_t* __restrict__ out) {
  constexpr int NSUB = 16 / RPT;                    // octet blocks per 128 rows
  constexpr int NGRP = kRb4Rows / RPT;              // RPT-row groups per 128 rows
  __shared__ uint8_t tile[kRb4Rows][kRb4Quads * 6 + 4];
  __shared__ uint16_t rho_s[kRb4Quads][NSUB][RPT];
  const int tid = threadIdx.x;
  uint32_t* lo_p = reinterpret_cast<uint32_t*>(out + L.lo_off);
  uint16_t* hi_p = reinterpret_cast<uint16_t*>(out + L.hi_off);
  uint32_t* rot_p = reinterpret_cast<uint32_t*>(out + L.rot_off);
  const int64_t nrb = L.mp / kRb4Rows + (L.mp % kRb4Rows ? 1 : 0);
  const int64_t nqt = (L.nqp + kRb4Quads - 1) / kRb4Quads;
  for (int64_t t = blockIdx.x; t < nrb * nqt; t += gridDim.x) {
    const int64_t base = (t % nrb) * kRb4Rows, q0 = (t / nrb) * kRb4Quads;
    const int64_t b0 = q0 * 6;  // first byte of the tile in a row
    __syncthreads();
    if ((rb & 3) == 0) {  // b0 = 48 (q0 / 8): 4-byte aligned
      for (int e = tid; e < kRb4Rows * 12; e += 128) {
        const int r = e / 12, w = e % 12;
        const int64_t i = base + r, by = b0 + 4 * w;
        uint32_t v = 0;
        if (i < m && by < rb) v = __ldg(reinterpret_cast<const uint32_t*>(packed + i * rb + by));
        *reinterpret_cast<uint32_t*>(&tile[r][4 * w]) = v;
      }
    } else {
      for (int e = tid; e < kRb4Rows * 48; e += 128) {
        const int r = e / 48, c = e % 48;
        const int64_t i = base + r, by = b0 + c;
        tile[r][c] = (i < m && by < rb) ? __ldg(packed + i * rb + by) : 0;
      }
    }
    __syncthreads();
    const int r = tid % RPT, sub = (tid / RPT) % NSUB, qq = tid / 16;
    const int64_t q = q0 + qq;
    if (q < L.nqp) {
      // folded index / sign of group g (of quad q) for tile row tr
      auto rec = [&](int tr, int g, uint32_t& sign) -> uint32_t {
        const int64_t j = q * 4 + g;
        sign = 0;
        if (base + tr >= m || j >= L.nb) return 0;
        uint32_t idx = 0;
#pragma unroll
        for (int c3 = 0; c3 < 3; ++c3) {
          const int c = 12 * qq + 3 * g + c3;  // code inside the tile row
          idx |= ((tile[tr][c >> 1] >> ((c & 1) * 4)) & 0xF) << (4 * c3);
        }
        if (idx & 0x800) { idx ^= 0xFFF; sign = 1; }
        return idx;
      };
      const int tr0 = 8 * RPT * sub + r;               // tile row of lane u = 0
      // each lane's 4 records (11-bit folded index | sign << 11) at bits 12 g,
      // extracted once and reused for the rotated writes (64-bit shifts, no
      // dynamically indexed arrays)
      uint64_t recs[8];
      uint32_t pmw = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        uint64_t rw = 0;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint32_t sg;
          const uint32_t f = rec(tr0 + RPT * u, g, sg);
          pmw |= (f & 1) << (4 * u + g);
          rw |= (uint64_t)(f | (sg << 11)) << (12 * g);
        }
        recs[u] = rw;
      }
      const uint32_t rho = choose_rotations(pmw);
      rho_s[qq][sub][r] = (uint16_t)rho;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int tr = tr0 + RPT * u;
        const int64_t i = base + tr;
        if (i >= L.mp) continue;
        const uint32_t ru = (rho >> (2 * u)) & 3;
        // position s2 holds group (s2 + ru) mod 4: rotate the 48-bit record set
        const uint64_t rw = recs[u];
        const uint64_t rot = ((rw >> (12 * ru)) | (rw << (48 - 12 * ru))) & 0xFFFFFFFFFFFFull;
        uint32_t ff[4], ss[4];
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) {
          const uint32_t v = (uint32_t)(rot >> (12 * s2)) & 0xFFF;
          ff[s2] = v & 0x7FF;
          ss[s2] = v >> 11;
        }
        lo_p[q * L.mp + i] = ff[0] | (ff[1] << 11) | ((ff[2] & 0x3FF) << 22);
        hi_p[q * L.mp + i] = (uint16_t)((ff[2] >> 10) | (ff[3] << 1) | (ss[0] << 12) |
                                        (ss[1] << 13) | (ss[2] << 14) | (ss[3] << 15));
      }
    }
    __syncthreads();
    if (tid < kRb4Quads * NGRP) {  // rotation word of (quad qq2, RPT-row group g2): 2 bits per row step
      const int qq2 = tid / NGRP, g2 = tid % NGRP, sub2 = g2 / 8, u2 = g2 % 8;
      const int64_t q2 = q0 + qq2, i0 = base + RPT * g2;
      if (q2 < L.nqp && i0 < L.mp) {
        uint32_t w = 0;
#pragma unroll
        for (int r2 = 0; r2 < RPT; ++r2) w |= ((uint32_t)(rho_s[qq2][sub2][r2] >> (2 * u2)) & 3) << (2 * r2);
        rot_p[q2 * (L.mp / RPT) + i0 / RPT] = w;
      }
    }
  }
}

// k % 3 tail codes per row (16 bits) for the finish kernel
__global__ void repack_rb_tail_kernel(const uint8_t* __restrict__ packed, int64_t m, int64_t k,
                                      int rb, RbLayout L, uint8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t tc = 0;
    for (int64_t j = L.nb * 3; j < k; ++j)
      tc |= ((packed[i * rb + (j >> 1)] >> ((j & 1) * 4)) & 0xF) << (4 * (j - L.nb * 3));
    reinterpret_cast<uint16_t*>(out + L.tail_off)[i] = (uint16_t)tc;
  }
}

// ============================================================================
// the row-block LUT kernel
// ============================================================================
constexpr int kRbTableBytes = 128 * 1024;
constexpr int kRbXN = 96;                        // staged activations per round (3 G BC)
// shared memory after the tables: [2][kRbXN] staged x | 8 corrections | TMEM slot | 16 half2 offsets s
constexpr int kRbCsOff = kRbTableBytes + 2 * kRbXN * 2, kRbS2Off = kRbCsOff + 64;

struct RbParams {
  const uint32_t* lo;     // [nqp][mp]
  const uint16_t* hi;     // [nqp][mp]
  const uint32_t* rot;    // [nqp][mp / 16] row rotations (rounds of 4 groups)
  int64_t mp, m, nb;
  const __half* x;        // (k, b) row-major
  int64_t b;
  float s[16];            // v[c] - beta
  float beta;
  int rounds_per_slice, nrounds;
  int rpb;                // rows per CTA of the rounds-of-4 kernel: whole warps (a multiple of 32 RPT), <= 512 RPT
  int early;              // weights may be read before griddepcontrol.wait
  float* partial;         // [S][m][b]
};

__device__ __forceinline__ uint32_t ldg_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ldg_u16(const uint16_t* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t mask, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(a), "r"(mask), "r"(c));  // (a & b) | c
  return r;
}
__device__ __forceinline__ uint32_t funnel16(uint32_t lo, uint32_t hi) {
  uint32_t r;
  asm("shf.r.wrap.b32 %0, %1, %2, 16;" : "=r"(r) : "r"(lo), "r"(hi));
  return r;
}

// acc[0..BC) += m * entry at shared byte address a, m = +-1.0h in the low
// (H == 0) or high half of mw
template <int BC, int H>
__device__ __forceinline__ void gather(uint32_t a, uint32_t mw, float* acc) {
  if constexpr (BC == 8) {
    uint32_t w0, w1, w2, w3;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(w0), "=r"(w1), "=r"(w2), "=r"(w3) : "r"(a));
    const uint32_t w[4] = {w0, w1, w2, w3};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (H == 0)
        asm("{\n\t.reg .b16 l, h, m0, m1;\n\tmov.b32 {l, h}, %2;\n\tmov.b32 {m0, m1}, %3;\n\t"
            "fma.rn.f32.f16 %0, l, m0, %0;\n\tfma.rn.f32.f16 %1, h, m0, %1;\n\t}"
            : "+f"(acc[2 * i]), "+f"(acc[2 * i + 1]) : "r"(w[i]), "r"(mw));
      else
        asm("{\n\t.reg .b16 l, h, m0, m1;\n\tmov.b32 {l, h}, %2;\n\tmov.b32 {m0, m1}, %3;\n\t"
            "fma.rn.f32.f16 %0, l, m1, %0;\n\tfma.rn.f32.f16 %1, h, m1, %1;\n\t}"
            : "+f"(acc[2 * i]), "+f"(acc[2 * i + 1]) : "r"(w[i]), "r"(mw));
    }
  } else if constexpr (BC == 4) {
    uint32_t w0, w1;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(w0), "=r"(w1) : "r"(a));
    const uint32_t w[2] = {w0, w1};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if constexpr (H == 0)
        asm("{\n\t.reg .b16 l, h, m0, m1;\n\tmov.b32 {l, h}, %2;\n\tmov.b32 {m0, m1}, %3;\n\t"
            "fma.rn.f32.f16 %0, l, m0, %0;\n\tfma.rn.f32.f16 %1, h, m0, %1;\n\t}"
            : "+f"(acc[2 * i]), "+f"(acc[2 * i + 1]) : "r"(w[i]), "r"(mw));
      else
        asm("{\n\t.reg .b16 l, h, m0, m1;\n\tmov.b32 {l, h}, %2;\n\tmov.b32 {m0, m1}, %3;\n\t"
            "fma.rn.f32.f16 %0, l, m1, %0;\n\tfma.rn.f32.f16 %1, h, m1, %1;\n\t}"
            : "+f"(acc[2 * i]), "+f"(acc[2 * i + 1]) : "r"(w[i]), "r"(mw));
    }
  } else {
    uint32_t w0;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w0) : "r"(a));
    if constexpr (H == 0)
      asm("{\n\t.reg .b16 l, h, m0, m1;\n\tmov.b32 {l, h}, %2;\n\tmov.b32 {m0, m1}, %3;\n\t"
          "fma.rn.f32.f16 %0, l, m0, %0;\n\tfma.rn.f32.f16 %1, h, m0, %1;\n\t}"
          : "+f"(acc[0]), "+f"(acc[1]) : "r"(w0), "r"(mw));
    else
      asm("{\n\t.reg .b16 l, h, m0, m1;\n\tmov.b32 {l, h}, %2;\n\tmov.b32 {m0, m1}, %3;\n\t"
          "fma.rn.f32.f16 %0, l, m1, %0;\n\tfma.rn.f32.f16 %1, h, m1, %1;\n\t}"
          : "+f"(acc[0]), "+f"(acc[1]) : "r"(w0), "r"(mw));
  }
}

// beta * (sum of this slice's activations of column c0 + c), c < BC, into
// cs[c] (the sign-symmetric tables' per-column correction, DESIGN.md "Sign
// symmetry"): computed once after the last round by all threads, in a fixed
// order (deterministic), with red[] (kRbThreads floats) as scratch -- instead
// of a serial per-round sum on one warp, which held that warp back at every
// round's barrier.
template <int BC, int G>
__device__ __forceinline__ void slice_correction(const RbParams& P, int r_begin, int r_end,
                                                 int64_t c0, float* red, float* cs) {
  const int tid = threadIdx.x;
  constexpr int NR = kRbThreads / BC;
  const int c = tid % BC, lr = tid / BC;
  const int64_t e0 = (int64_t)r_begin * G * 3;
  const int64_t e1 = min((int64_t)r_end * G, P.nb) * 3;
  float sum = 0.f;
  if (c0 + c < P.b)
    for (int64_t e = e0 + lr; e < e1; e += NR) sum += __half2float(P.x[e * P.b + c0 + c]);
  red[tid] = sum;
  MSG_JITTER();
  __syncthreads();
  if (tid < BC) {
    float t = 0.f;
    for (int i = 0; i < NR; ++i) t += red[i * BC + tid];
    cs[tid] = P.beta * t;
  }
  MSG_JITTER();
  __syncthreads();
}

// one row's partials of a column tile: the widest aligned stores the tile
// allows (float4 when the row stride b and the valid columns are multiples of
// 4, float2 for multiples of 2; a partly filled last tile of b = 6, 12, ...
// otherwise fell back to strided scalar stores, measured 25 % slower kernels)
template <int BC>
__device__ __forceinline__ void store_partial_row(float* dst, const float* v, int64_t b, int64_t c0) {
  const int64_t nvc = b - c0 < BC ? b - c0 : BC;   // valid columns of this tile
  if ((b & 3) == 0 && (nvc & 3) == 0) {
#pragma unroll
    for (int c = 0; c < BC; c += 4)
      if (c < nvc) *reinterpret_cast<float4*>(dst + c) = make_float4(v[c], v[c + 1], v[c + 2], v[c + 3]);
  } else if ((b & 1) == 0 && (nvc & 1) == 0) {
#pragma unroll
    for (int c = 0; c < BC; c += 2)
      if (c < nvc) *reinterpret_cast<float2*>(dst + c) = make_float2(v[c], v[c + 1]);
  } else {
#pragma unroll
    for (int c = 0; c < BC; ++c)
      if (c < nvc) dst[c] = v[c];
  }
}

// (a & b) | (c & ~b): the table slot bits come from c, the entry bits from a
__device__ __forceinline__ uint32_t lop3_mux(uint32_t a, uint32_t mask, uint32_t c) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE2;" : "=r"(r) : "r"(a), "r"(mask), "r"(c));
  return r;
}

// the four lookups of one (row, quad) record: addresses from lo/hi, +-1.0h
// multipliers from the sign bits (hi bits 12..15) -- sign 0 / 2 land at bits
// 15 / 31 of one word and 1 / 3 of another (one IMAD each, no carries: the
// masked bits map to distinct positions)
template <int BC>
__device__ __forceinline__ void quad_lookups(uint32_t lo, uint32_t hi, uint32_t tab,
                                             const uint32_t (&slot)[4], float* acc) {
  const uint32_t hm = hi & 0xF000u;
  const uint32_t m02 = lop3_and_or(hm * 0x20008u, 0x80008000u, 0x3C003C00u);
  const uint32_t m13 = lop3_and_or(hm * 0x10004u, 0x80008000u, 0x3C003C00u);
  const uint32_t a0 = lop3_and_or(lo << 6, 0x1FFC0u, slot[0]);
  const uint32_t a1 = lop3_and_or(lo >> 5, 0x1FFC0u, slot[1]);
  const uint32_t a2 = lop3_and_or(funnel16(lo, hi), 0x1FFC0u, slot[2]);
  const uint32_t a3 = lop3_and_or(hi << 5, 0x1FFC0u, slot[3]);
  MSG_DASSERT(a0 < kRbTableBytes && a1 < kRbTableBytes && a2 < kRbTableBytes && a3 < kRbTableBytes);
  gather<BC, 0>(a0 + tab, m02, acc);
  gather<BC, 0>(a1 + tab, m13, acc);
  gather<BC, 1>(a2 + tab, m02, acc);
  gather<BC, 1>(a3 + tab, m13, acc);
}

// One round's weight words of one thread: RPT consecutive rows per quad
// plane, read with 16-byte loads (lo: RPT words, hi: RPT 16-bit halves).
template <int QR, int RPT>
struct WSet {
  uint32_t lo[QR][RPT];
  uint32_t hi[QR][RPT / 2];
};

template <int QR, int RPT>
__device__ __forceinline__ void load_wset(WSet<QR, RPT>& w, const uint32_t* lo, const uint16_t* hi,
                                          int64_t mp, bool ok) {

#pragma unroll
  for (int u = 0; u < QR; ++u) {
    if (ok) {
#pragma unroll
      for (int v = 0; v < RPT / 4; ++v) {
        uint32_t a, b, c, d;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(lo + u * mp + 4 * v));
        w.lo[u][4 * v] = a; w.lo[u][4 * v + 1] = b; w.lo[u][4 * v + 2] = c; w.lo[u][4 * v + 3] = d;
      }
      if constexpr (RPT == 8) {
        uint32_t a, b, c, d;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(hi + u * mp));
        w.hi[u][0] = a; w.hi[u][1] = b; w.hi[u][2] = c; w.hi[u][3] = d;
      } else {
        uint32_t a, b;
        asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                     : "=r"(a), "=r"(b) : "l"(hi + u * mp));
        w.hi[u][0] = a; w.hi[u][1] = b;
      }
    } else {
#pragma unroll
      for (int r = 0; r < RPT; ++r) w.lo[u][r] = 0;
#pragma unroll
      for (int r = 0; r < RPT / 2; ++r) w.hi[u][r] = 0;
    }
  }
}

// rounds of 4 groups: position s of a row reads table (s + rho) mod 4, rho
// chosen per row by K3 (2 bits of the round's rotation word); the slot base
// t0 = 16 rho and t0 + 16 s carry the slot at bits 4-5 (a carry into bit 6 is
// masked off by the mux)
template <int BC>
__device__ __forceinline__ void quad_lookups_rot(uint32_t lo, uint32_t hi, uint32_t t0,
                                                 uint32_t tab, float* acc) {
  const uint32_t hm = hi & 0xF000u;
  const uint32_t m02 = lop3_and_or(hm * 0x20008u, 0x80008000u, 0x3C003C00u);
  const uint32_t m13 = lop3_and_or(hm * 0x10004u, 0x80008000u, 0x3C003C00u);
  const uint32_t a0 = lop3_mux(lo << 6, 0x1FFC0u, t0);
  const uint32_t a1 = lop3_mux(lo >> 5, 0x1FFC0u, t0 + 16);
  const uint32_t a2 = lop3_mux(funnel16(lo, hi), 0x1FFC0u, t0 + 32);
  const uint32_t a3 = lop3_mux(hi << 5, 0x1FFC0u, t0 + 48);
  MSG_DASSERT(a0 < kRbTableBytes && a1 < kRbTableBytes && a2 < kRbTableBytes && a3 < kRbTableBytes);
  gather<BC, 0>(a0 + tab, m02, acc);
  gather<BC, 0>(a1 + tab, m13, acc);
  gather<BC, 1>(a2 + tab, m02, acc);
  gather<BC, 1>(a3 + tab, m13, acc);
}

template <int BC>
__global__ void __launch_bounds__(kRbThreads, 1) rb_lut_kernel(RbParams P) {
  constexpr int G = 32 / BC;          // groups (tables) per round
  constexpr int QR = G / 4;           // quads per round
  constexpr int EB = 2 * BC;          // bytes per entry
  constexpr int RPT = rb_rows_per_thread(G);
  constexpr int R = kRbThreads * RPT;       // rows per CTA
  constexpr int NI = G * 256 / kRbThreads;  // build work items per thread
  extern __shared__ __align__(128) uint8_t smem[];
  __half* xs0 = reinterpret_cast<__half*>(smem + kRbTableBytes);  // [2][96] staged activations
  float* cs = reinterpret_cast<float*>(smem + kRbCsOff);  // [BC] corrections
  uint32_t* s2h = reinterpret_cast<uint32_t*>(smem + kRbS2Off);  // half2 (s[c], s[c])

  const int tid = threadIdx.x;
  if (tid < 16) {
    const __half2 h2 = __float2half2_rn(P.s[tid]);
    s2h[tid] = *reinterpret_cast<const uint32_t*>(&h2);
  }
  const int64_t row0 = (int64_t)blockIdx.x * R;
  const int slice = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.z * BC;
  const int r_begin = slice * P.rounds_per_slice;
  const int r_end = min(P.nrounds, r_begin + P.rounds_per_slice);
  const int nr = r_end - r_begin;
  const int64_t my_row = row0 + (int64_t)tid * RPT;     // this thread's first row
  const int64_t left = P.m - my_row;
  const int nvalid = left <= 0 ? 0 : (left < RPT ? (int)left : RPT);  // rows < m
  const bool has_words = my_row < P.mp;                 // its rows exist in the (padded) planes
  const uint32_t tab = smem_u32(smem);

  // activations of round t: element e -> (group gr = e / (3 BC), code r, column c)
  auto load_x = [&](int t) -> __half {
    __half v = __ushort_as_half((unsigned short)0);
    if (tid < kRbXN && t < nr) {
      const int gl = tid / (3 * BC), rem = tid % (3 * BC), r = rem / BC, c = rem % BC;
      const int64_t j = (int64_t)(r_begin + t) * G + gl;
      if (j < P.nb && c0 + c < P.b) v = P.x[(j * 3 + r) * P.b + c0 + c];
    }
    return v;
  };

  const int64_t wstep = (int64_t)QR * P.mp;  // plane elements per round
  const uint32_t* plo = P.lo + (int64_t)r_begin * wstep + my_row;
  const uint16_t* phi = P.hi + (int64_t)r_begin * wstep + my_row;
  WSet<QR, RPT> wa;
  if (nr > 0 && P.early) load_wset(wa, plo, phi, P.mp, has_words);
  griddep_wait();
  griddep_launch_dependents();
  if (nr > 0 && !P.early) load_wset(wa, plo, phi, P.mp, has_words);
  if (tid < kRbXN) xs0[tid] = load_x(0);
  __half xnext = load_x(1);

  float acc[RPT][BC];
#pragma unroll
  for (int r = 0; r < RPT; ++r)
#pragma unroll
    for (int c = 0; c < BC; ++c) acc[r][c] = 0.f;

  // table slot (byte offset) of position p: group (p + tid) mod G
  uint32_t slot[QR][4];
#pragma unroll
  for (int u = 0; u < QR; ++u)
#pragma unroll
    for (int s = 0; s < 4; ++s) slot[u][s] = (uint32_t)(((4 * u + s + tid) % G) * EB);
  // build work: this thread fills table tt = tid % G at low code pairs
  // lw = tid / G + i * (512 / G), entries lw + 256 h for the 8 top codes h
  const int tt = tid % G;
  uint8_t* const bdst = smem + (uint32_t)(tid / G) * 64 + (uint32_t)tt * EB;

  // one round: build the tables from xs[t & 1], prefetch round t+1's words into
  // `nxt`, gather with `cur` (two register sets, so no copies between rounds)
  auto round = [&](int t, WSet<QR, RPT>& cur, WSet<QR, RPT>& nxt) {
    const __half* xs = xs0 + (t & 1) * kRbXN;
    MSG_JITTER();
    __syncthreads();  // the gathers of round t-1 are done with the tables; xs[t&1] written
    if (t + 1 < nr && tid < kRbXN) xs0[((t + 1) & 1) * kRbXN + tid] = xnext;
    xnext = load_x(t + 2);
    // ---- build, all in fp16x2 (the codebook offsets s are exact in fp16):
    // entry(lw + 256 h) = (s[lw & 15] x0 + s[lw >> 4] x1) + s[h] x2, one
    // rounding per operation as in the reference's table (lut.py:59-72)
    {
      const __half2* xg = reinterpret_cast<const __half2*>(xs + tt * 3 * BC);
      __half2 x0[BC / 2], x1[BC / 2], t2[BC / 2];
#pragma unroll
      for (int c = 0; c < BC / 2; ++c) { x0[c] = xg[c]; x1[c] = xg[BC / 2 + c]; t2[c] = xg[BC + c]; }
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int lw = tid / G + i * (kRbThreads / G);
        const __half2 sa = *reinterpret_cast<const __half2*>(&s2h[lw & 15]);
        const __half2 sb = *reinterpret_cast<const __half2*>(&s2h[lw >> 4]);
        __half2 b2[BC / 2];
#pragma unroll
        for (int c = 0; c < BC / 2; ++c) b2[c] = __hfma2(sb, x1[c], __hmul2(sa, x0[c]));
        uint8_t* dst = bdst + i * (kRbThreads / G) * 64;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const __half2 s2 = *reinterpret_cast<const __half2*>(&s2h[h]);
          uint32_t wv[BC / 2];
#pragma unroll
          for (int c = 0; c < BC / 2; ++c) {
            const __half2 e2 = __hfma2(s2, t2[c], b2[c]);
            wv[c] = *reinterpret_cast<const uint32_t*>(&e2);
          }
          uint8_t* p = dst + h * 256 * 64;
          MSG_DASSERT(p + EB <= smem + kRbTableBytes);
          if constexpr (BC == 2) *reinterpret_cast<uint32_t*>(p) = wv[0];
          else if constexpr (BC == 4) *reinterpret_cast<uint2*>(p) = make_uint2(wv[0], wv[1]);
          else *reinterpret_cast<uint4*>(p) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      }
    }
    MSG_JITTER();
    __syncthreads();
    // the next round's words are loaded into the registers of this round's
    // words right after their last use (one register set, no copies): the
    // loads have the rest of this round and the next build to land
    const bool more = t + 1 < nr;
    const uint32_t* nlo = plo + (int64_t)(t + 1) * wstep;
    const uint16_t* nhi = phi + (int64_t)(t + 1) * wstep;
    if (has_words) {
#pragma unroll
      for (int r = 0; r < RPT; ++r) {
#pragma unroll
        for (int u = 0; u < QR; ++u) {
          const uint32_t hw = cur.hi[u][r >> 1];
          quad_lookups<BC>(cur.lo[u][r], (r & 1) ? (hw >> 16) : hw, tab, slot[u], acc[r]);
          if (more && (r & 3) == 3) {
            uint32_t a, b, c, d;
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(nlo + u * P.mp + r - 3));
            cur.lo[u][r - 3] = a; cur.lo[u][r - 2] = b; cur.lo[u][r - 1] = c; cur.lo[u][r] = d;
          }
          if (more && r == RPT - 1) {
            if constexpr (RPT == 8) {
              uint32_t a, b, c, d;
              asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(nhi + u * P.mp));
              cur.hi[u][0] = a; cur.hi[u][1] = b; cur.hi[u][2] = c; cur.hi[u][3] = d;
            } else {
              uint32_t a, b;
              asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                           : "=r"(a), "=r"(b) : "l"(nhi + u * P.mp));
              cur.hi[u][0] = a; cur.hi[u][1] = b;
            }
          }
        }
      }
    }
  };
  for (int t = 0; t < nr; ++t) round(t, wa, wa);
  // ---- fold this slice's symmetry correction beta * sum(x) into every row
  MSG_JITTER();
  __syncthreads();  // the tables are free: scratch for the correction sum
  slice_correction<BC, G>(P, r_begin, r_end, c0, reinterpret_cast<float*>(smem), cs);
  float cv[BC];
#pragma unroll
  for (int c = 0; c < BC; ++c) cv[c] = cs[c];
  // ---- write partials [slice][i][c]
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    if (r >= nvalid) continue;
    float* dst = P.partial + ((int64_t)slice * P.m + my_row + r) * P.b + c0;
    float v[BC];
#pragma unroll
    for (int c = 0; c < BC; ++c) v[c] = acc[r][c] + cv[c];
    store_partial_row<BC>(dst, v, P.b, c0);
  }
}

// ============================================================================
// rounds of 4 groups (b >= 8): accumulators in tensor memory
// ============================================================================
// 16 rows x 8 fp32 columns per thread live in TMEM (512 columns x 128 lanes =
// 8192 rows per CTA, twice the register kernel's rows per table build, and
// 64 registers freed for loads in flight).  Thread (warp w, lane l) owns TMEM
// lane 32 (w mod 4) + l (the lanes a warp may access) and columns
// 128 (w / 4) .. + 127; per round it streams its rows two at a time through
// registers: tcgen05.ld (32x32b.x16: two rows), 8 lookups, tcgen05.st, with
// the next pair's load in flight.
// (RPT = 16: 8192 rows per CTA, all 512 TMEM columns; RPT = 8: 4096 rows,
// 256 columns)

__device__ __forceinline__ void tm_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tm_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tm_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void ldg_v4(const void* p, uint32_t& a, uint32_t& b, uint32_t& c,
                                       uint32_t& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
}

template <int kTmRPT>
__global__ void __launch_bounds__(kRbThreads, 1) rb_tmem_kernel(RbParams P) {
  constexpr int kTmR = kRbThreads * kTmRPT;         // rows per CTA
  constexpr int kTmCols = 4 * 8 * kTmRPT;           // TMEM columns: 4 warps per lane quarter
  constexpr int BC = 8, G = 4, EB = 16, NI = G * 256 / kRbThreads;
  extern __shared__ __align__(128) uint8_t smem[];
  __half* xs0 = reinterpret_cast<__half*>(smem + kRbTableBytes);                // [2][96]
  float* cs = reinterpret_cast<float*>(smem + kRbCsOff);   // [8]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(cs + 8);
  uint32_t* s2h = reinterpret_cast<uint32_t*>(smem + kRbS2Off);  // half2 (s[c], s[c])

  const int tid = threadIdx.x, warp = tid >> 5;
  if (tid < 16) {
    const __half2 h2 = __float2half2_rn(P.s[tid]);
    s2h[tid] = *reinterpret_cast<const uint32_t*>(&h2);
  }
  // row blocks of P.rpb <= kTmR rows (balanced over the row blocks, whole
  // warps): warps past the block take part in the builds and barriers only
  const int64_t row0 = (int64_t)blockIdx.x * P.rpb;
  const int slice = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.z * BC;
  const int r_begin = slice * P.rounds_per_slice;
  const int r_end = min(P.nrounds, r_begin + P.rounds_per_slice);
  const int nr = r_end - r_begin;
  const bool warp_on = warp * 32 * kTmRPT < P.rpb;
  const int64_t my_row = row0 + (int64_t)tid * kTmRPT;
  const int64_t left = warp_on ? P.m - my_row : 0;
  const int nvalid = left <= 0 ? 0 : (left < kTmRPT ? (int)left : kTmRPT);
  const bool has_words = warp_on && my_row < P.mp;
  const uint32_t tab = smem_u32(smem);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
        smem_u32(tmem_slot)), "n"(kTmCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }

  auto load_x = [&](int t) -> __half {
    __half v = __ushort_as_half((unsigned short)0);
    if (tid < kRbXN && t < nr) {
      const int gl = tid / (3 * BC), rem = tid % (3 * BC), r = rem / BC, c = rem % BC;
      const int64_t j = (int64_t)(r_begin + t) * G + gl;
      if (j < P.nb && c0 + c < P.b) v = P.x[(j * 3 + r) * P.b + c0 + c];
    }
    return v;
  };

  // this thread's words of one round: RPT lo words, RPT hi halves, RPT rotations
  const int64_t rstride = P.mp / kTmRPT;               // rotation words per quad
  const uint32_t* plo = P.lo + (int64_t)r_begin * P.mp + my_row;
  const uint16_t* phi = P.hi + (int64_t)r_begin * P.mp + my_row;
  const uint32_t* prot = P.rot + (int64_t)r_begin * rstride + my_row / kTmRPT;
  uint32_t wlo[kTmRPT], whi[kTmRPT / 2], wrot = 0;
  auto load_words = [&](int t) {
    if (has_words && t < nr) {
      const uint32_t* l = plo + (int64_t)t * P.mp;
#pragma unroll
      for (int v = 0; v < kTmRPT / 4; ++v)
        ldg_v4(l + 4 * v, wlo[4 * v], wlo[4 * v + 1], wlo[4 * v + 2], wlo[4 * v + 3]);
      const uint16_t* h = phi + (int64_t)t * P.mp;
#pragma unroll
      for (int v = 0; v < kTmRPT / 8; ++v)
        ldg_v4(h + 8 * v, whi[4 * v], whi[4 * v + 1], whi[4 * v + 2], whi[4 * v + 3]);
      wrot = ldg_u32(prot + (int64_t)t * rstride);
    } else {
#pragma unroll
      for (int v = 0; v < kTmRPT; ++v) wlo[v] = 0;
#pragma unroll
      for (int v = 0; v < kTmRPT / 2; ++v) whi[v] = 0;
      wrot = 0;
    }
  };
  if (P.early) load_words(0);
  griddep_wait();
  griddep_launch_dependents();
  if (!P.early) load_words(0);
  if (tid < kRbXN) xs0[tid] = load_x(0);
  __half xnext = load_x(1);

  tm_fence_before();
  MSG_JITTER();
  __syncthreads();
  tm_fence_after();
  const uint32_t tbase = *tmem_slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(warp >> 2) * (8 * kTmRPT);
  if (warp_on) {  // zero accumulators
    float z[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) z[i] = 0.f;
#pragma unroll
    for (int p = 0; p < kTmRPT / 2; ++p) tm_st16(tbase + 16 * p, z);
  }
  const int tt = tid % G;
  uint8_t* const bdst = smem + (uint32_t)(tid / G) * 64 + (uint32_t)tt * EB;

  for (int t = 0; t < nr; ++t) {
    const __half* xs = xs0 + (t & 1) * kRbXN;
    MSG_JITTER();
    __syncthreads();  // the gathers of round t-1 are done with the tables; xs[t&1] written
    if (t + 1 < nr && tid < kRbXN) xs0[((t + 1) & 1) * kRbXN + tid] = xnext;
    xnext = load_x(t + 2);
    {  // ---- build (as rb_lut_kernel)
      const __half2* xg = reinterpret_cast<const __half2*>(xs + tt * 3 * BC);
      __half2 x0[BC / 2], x1[BC / 2], t2[BC / 2];
#pragma unroll
      for (int c = 0; c < BC / 2; ++c) { x0[c] = xg[c]; x1[c] = xg[BC / 2 + c]; t2[c] = xg[BC + c]; }
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int lw = tid / G + i * (kRbThreads / G);
        const __half2 sa = *reinterpret_cast<const __half2*>(&s2h[lw & 15]);
        const __half2 sb = *reinterpret_cast<const __half2*>(&s2h[lw >> 4]);
        __half2 b2[BC / 2];
#pragma unroll
        for (int c = 0; c < BC / 2; ++c) b2[c] = __hfma2(sb, x1[c], __hmul2(sa, x0[c]));
        uint8_t* dst = bdst + i * (kRbThreads / G) * 64;
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const __half2 s2 = *reinterpret_cast<const __half2*>(&s2h[h]);
          uint32_t wv[BC / 2];
#pragma unroll
          for (int c = 0; c < BC / 2; ++c) {
            const __half2 e2 = __hfma2(s2, t2[c], b2[c]);
            wv[c] = *reinterpret_cast<const uint32_t*>(&e2);
          }
          MSG_DASSERT(dst + h * 256 * 64 + 16 <= smem + kRbTableBytes);
          *reinterpret_cast<uint4*>(dst + h * 256 * 64) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        }
      }
    }
    MSG_JITTER();
    __syncthreads();
    if (!warp_on) continue;  // (warp-uniform) no rows of this block: next round's barrier
    // ---- gather: row pairs through registers; the next round's words are
    // loaded into the same registers right after their last use
    const bool more = t + 1 < nr;
    const uint32_t* nlo = plo + (int64_t)(t + 1) * P.mp;
    const uint16_t* nhi = phi + (int64_t)(t + 1) * P.mp;
    const uint32_t rot_a = wrot << 4, rot_b = wrot >> 12;  // rows 0-7 / 8-15 at bits 4+2r'
    if (more && has_words) wrot = ldg_u32(prot + (int64_t)(t + 1) * rstride);
    tm_wait_st();  // the previous round's accumulator stores are complete
    float va[16], vb[16];
    tm_ld16(tbase, va);
    tm_wait_ld();
#pragma unroll
    for (int p = 0; p < kTmRPT / 2; ++p) {
      float (&cur)[16] = (p & 1) ? vb : va;
      float (&nxt)[16] = (p & 1) ? va : vb;
      if (p + 1 < kTmRPT / 2) tm_ld16(tbase + 16 * (p + 1), nxt);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = 2 * p + h;
        const uint32_t hw = whi[r >> 1];
        const uint32_t t0 = ((r < 8 ? rot_a : rot_b) >> (2 * (r & 7))) & 0x30u;
        quad_lookups_rot<BC>(wlo[r], h ? (hw >> 16) : hw, t0, tab, cur + 8 * h);
      }
      if (more && has_words) {
        if ((p & 1) == 1) {  // rows 2p-2 .. 2p+1 done: their lo words
          const int r = 2 * p - 2;
          ldg_v4(nlo + r, wlo[r], wlo[r + 1], wlo[r + 2], wlo[r + 3]);
        }
        if (p == 3) ldg_v4(nhi, whi[0], whi[1], whi[2], whi[3]);
        if constexpr (kTmRPT == 16) {
          if (p == 7) ldg_v4(nhi + 8, whi[4], whi[5], whi[6], whi[7]);
        }
      }
      tm_st16(tbase + 16 * p, cur);
      tm_wait_ld();
    }
  }
  // ---- partials: accumulators + this slice's symmetry correction
  tm_wait_st();
  MSG_JITTER();
  __syncthreads();  // the tables are free: scratch for the correction sum
  slice_correction<BC, G>(P, r_begin, r_end, c0, reinterpret_cast<float*>(smem), cs);
  float cv[BC];
#pragma unroll
  for (int c = 0; c < BC; ++c) cv[c] = cs[c];
#pragma unroll
  for (int p = 0; p < kTmRPT / 2; ++p) {
    if (!warp_on) break;
    float v[16];
    tm_ld16(tbase + 16 * p, v);
    tm_wait_ld();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = 2 * p + h;
      if (r >= nvalid) continue;
      float* dst = P.partial + ((int64_t)slice * P.m + my_row + r) * P.b + c0;
      float vr[BC];
#pragma unroll
      for (int c = 0; c < BC; ++c) vr[c] = v[8 * h + c] + cv[c];
      store_partial_row<BC>(dst, vr, P.b, c0);
    }
  }
  tm_fence_before();
  MSG_JITTER();
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmem_slot), "n"(kTmCols));
}

// ============================================================================
// host side
// ============================================================================
// tables per round from the batch: 8-column tiles (rounds of 4 groups) from
// b = 5 -- one padded tile beats 4 + (b - 4) columns in two tiles (b = 6 at
// cfg4: 48 + 15 -> ~39 + 8 us) -- 4-column tiles for b = 2..4 (measured b = 2
// on 4-column tiles slower than on the 2-column kernel, so that stays)
int rb_group_count(int64_t b) { return b >= 5 ? 4 : (b >= 4 ? 8 : 16); }

bool rb_eligible(int width, int x_dtype, int64_t b, int d, int scale_mode, bool sym,
                 bool f32_entries, bool s_exact16) {
  return width == 4 && d == 3 && x_dtype == MSG_F16 && b >= 2 && sym && !f32_entries &&
         s_exact16 && scale_mode != MSG_SCALE_PER_GROUP;
}

int64_t rb_layout_bytes(int64_t m, int64_t k, int G, int rpt) { return rb_layout(m, k, G, rpt).total; }

int rb_repack(const uint8_t* packed, int64_t m, int64_t k, int G, int rpt, uint8_t* out,
              cudaStream_t s) {
  RbLayout L = rb_layout(m, k, G, rpt);
  if (L.nb == 0 || m == 0) return fail(MSG_ERR_UNSUPPORTED, "row-block layout needs a full group");
  const int rb = row_bytes(k, 4);
  const int64_t tiles = ((m + kRpTileRows - 1) / kRpTileRows) *
                        ((L.nqp + kRpTileQuads - 1) / kRpTileQuads);
  const int grid = (int)std::min<int64_t>(tiles, (int64_t)sm_count() * 16);
  if (G == 4) {
    const int64_t t4 = ceil_div(L.mp, kRb4Rows) * ceil_div(L.nqp, kRb4Quads);
    const int g4 = (int)std::min<int64_t>(t4, (int64_t)sm_count() * 16);
    if (rpt == 8) repack_rb4_kernel<8><<<g4, 128, 0, s>>>(packed, m, k, rb, L, out);
    else repack_rb4_kernel<16><<<g4, 128, 0, s>>>(packed, m, k, rb, L, out);
  } else {
    repack_rb_kernel<<<grid, 256, 0, s>>>(packed, m, k, rb, L, out);
  }
  MSG_LAUNCH_CHECK();
  // rows m .. mp-1 of every plane are zero (they are never read)
  if (L.tail) {
    repack_rb_tail_kernel<<<(int)std::min<int64_t>(ceil_div(m, 256), sm_count() * 4), 256, 0, s>>>(
        packed, m, k, rb, L, out);
    MSG_LAUNCH_CHECK();
  }
  return MSG_OK;
}

struct RbPlan {
  int G, bc, S, rps, nrounds, nrow_blocks, ncol_tiles, rpt, rpb;
  int64_t partial_bytes, smem;
};

RbPlan rb_plan(int64_t m, int64_t k, int64_t b, int rpt) {
  RbPlan p{};
  p.G = rb_group_count(b);
  p.bc = 32 / p.G;
  p.rpt = p.G == 4 ? rpt : rb_rows_per_thread(p.G);
  RbLayout L = rb_layout(m, k, p.G, p.G == 4 ? rpt : 16);
  p.nrounds = (int)(L.nqp / (p.G / 4));
  // rounds of 4: as many row blocks as full-size CTAs need, of equal height in
  // whole warps (11008 rows at 4096 per CTA: 3 x 3840 instead of 4096 + 4096 +
  // 2816 -- every CTA gathers for the tallest block)
  p.rpb = kRbThreads * p.rpt;
  if (p.G == 4 && m > 0) {
    const int64_t nrb = ceil_div(m, (int64_t)kRbThreads * p.rpt), wrows = 32 * p.rpt;
    p.rpb = (int)(ceil_div(ceil_div(m, nrb), wrows) * wrows);
  }
  p.nrow_blocks = (int)ceil_div(m, (int64_t)p.rpb);
  p.ncol_tiles = (int)ceil_div(b, p.bc);
  const int64_t base = (int64_t)p.nrow_blocks * p.ncol_tiles;
  int64_t S = std::max<int64_t>(1, sm_count() / std::max<int64_t>(1, base));
  S = std::min<int64_t>(S, p.nrounds);
  p.rps = (int)ceil_div(p.nrounds, S);
  p.S = (int)ceil_div(p.nrounds, p.rps);
  p.partial_bytes = al256((int64_t)p.S * m * b * 4);
  p.smem = kRbS2Off + 64;  // tables, staged x, corrections, TMEM slot, s offsets
  return p;
}

int64_t rb_workspace_bytes(int64_t m, int64_t k, int64_t b, int rpt) {
  return rb_plan(m, k, b, rpt).partial_bytes;
}

// Rows per thread of the rounds-of-4 kernel (b >= 8): 16 (8192-row CTAs)
// unless an 8192-row block would be mostly empty or the row count is small
// enough that the k-slice partials (~S x 8192 x b x 4 bytes, a fixed ~39 MB
// at b = 8) rival the weight stream -- then 8 (4096-row CTAs, half the
// partials, twice the table builds per lookup).  flags can force either.
int rb_choose_rpt(int64_t m, int64_t b, int flags) {
  if (rb_group_count(b) != 4) return 16;
  if (flags & MSG_FLAG_RB_ROWS8) return 8;
  if (flags & MSG_FLAG_RB_ROWS16) return 16;
  // measured (one B200): 4096-row CTAs win at m <= 16384 with one or two
  // 8-column tiles (cfg3 11008 x 4096 b = 16: 69.9 -> 55.4 us; 8192-row
  // shards of cfg5: 46.5 -> 40.3 us), lose at m = 65536 (210.6 -> 219.4 us)
  // and at b = 64 (209.6 -> 220.1 us), tie at m = 32768
  return (m <= 16384 && b <= 16) ? 8 : 16;
}

template <int BC>
static int launch_rb_t(const RbPlan& pl, RbParams& P, cudaStream_t s) {
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    MSG_CUDA_CHECK(cudaFuncSetAttribute(rb_lut_kernel<BC>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    configured_dev = dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.nrow_blocks, pl.S, pl.ncol_tiles);
  cfg.blockDim = dim3(kRbThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MSG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, rb_lut_kernel<BC>, P));
  return MSG_OK;
}

template <int RPT>
static int launch_rb_tmem(const RbPlan& pl, RbParams& P, cudaStream_t s) {
  static int configured_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (configured_dev != dev) {
    MSG_CUDA_CHECK(cudaFuncSetAttribute(rb_tmem_kernel<RPT>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    configured_dev = dev;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.nrow_blocks, pl.S, pl.ncol_tiles);
  cfg.blockDim = dim3(kRbThreads);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MSG_CUDA_CHECK(cudaLaunchKernelEx(&cfg, rb_tmem_kernel<RPT>, P));
  return MSG_OK;
}

int launch_rb(const uint8_t* wrep, int64_t m, int64_t k, const double* values, double beta,
              const void* x, int64_t b, int scale_mode, const void* q, int q_dtype, void* y,
              int y_dtype, void* ws, int64_t ws_bytes, bool early, bool lut_only,
              const TailVals& tv, int rpt, cudaStream_t s) {
  const RbPlan pl = rb_plan(m, k, b, rpt);
  if (ws_bytes < pl.partial_bytes)
    return fail(MSG_ERR_WORKSPACE, "workspace too small: need %lld bytes",
                (long long)pl.partial_bytes);
  RbLayout L = rb_layout(m, k, pl.G, pl.G == 4 ? pl.rpt : 16);
  RbParams P{};
  P.lo = reinterpret_cast<const uint32_t*>(wrep + L.lo_off);
  P.hi = reinterpret_cast<const uint16_t*>(wrep + L.hi_off);
  P.rot = reinterpret_cast<const uint32_t*>(wrep + L.rot_off);
  P.mp = L.mp;
  P.m = m;
  P.nb = L.nb;
  P.x = reinterpret_cast<const __half*>(x);
  P.b = b;
  for (int c = 0; c < 16; ++c) P.s[c] = (float)(values[c] - beta);
  P.beta = (float)beta;
  P.rounds_per_slice = pl.rps;
  P.nrounds = pl.nrounds;
  P.rpb = pl.rpb;
  P.early = early ? 1 : 0;
  P.partial = reinterpret_cast<float*>(ws);
  int e = MSG_OK;
  switch (pl.bc) {
    case 8: e = pl.rpt == 8 ? launch_rb_tmem<8>(pl, P, s) : launch_rb_tmem<16>(pl, P, s); break;
    case 4: e = launch_rb_t<4>(pl, P, s); break;
    default: e = launch_rb_t<2>(pl, P, s); break;
  }
  if (e || lut_only) return e;
  const uint16_t* tailp = L.tail ? reinterpret_cast<const uint16_t*>(wrep + L.tail_off) : nullptr;
  return launch_finish(P.partial, pl.S, m, b, k, 3, tailp, tv, x, MSG_F16, scale_mode, q, q_dtype,
                       y, y_dtype, s);
}

}  // namespace msg
