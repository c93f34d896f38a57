/*
 * msgemm_b200.h -- C ABI of the B200-native msGeMM hot path.
 *
 * The reference (arXiv 2310.06178, /root/reference/pkg/src/msgemm) is a
 * pure-Python/numpy library with no FFI; its "drop-in boundary" is the Python
 * function surface re-exported at pkg/src/msgemm/__init__.py:10-92.  Every
 * entry point below is the device-side replacement of one of those
 * functions; the Python package paper_2310_06178_b200 binds them with ctypes
 * and keeps the reference's signatures, dtypes and error behaviour
 * (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - All array pointers are DEVICE pointers, caller-owned; the library never
 *     allocates device memory.  Scratch goes in a caller-provided workspace
 *     sized by the matching *_workspace_bytes() query.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *     Every call is stream-ordered and never synchronises the host.
 *   - Codebook values are passed as a HOST array of 2^width doubles (the
 *     reference's Codebook.values, codebook.py:16-47); they travel in the
 *     kernel parameter block.
 *   - Return 0 on success or a negative MSG_ERR_* code; msg_last_error()
 *     returns a thread-local message.  Python maps the codes to the
 *     reference's exception types (ValueError, IndexError, TableBudgetError).
 *   - Arrays are C-contiguous: packed weights (m, row_bytes(k,width)) uint8,
 *     X (k, b), Y (m, b), LUT entries (num_blocks, 2^(width*d)).
 */
#ifndef MSGEMM_B200_H
#define MSGEMM_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define MSG_API __attribute__((visibility("default")))
#else
#define MSG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define MSG_OK               0
#define MSG_ERR_VALUE       -1  /* -> ValueError                        */
#define MSG_ERR_INDEX       -2  /* -> IndexError                        */
#define MSG_ERR_BUDGET      -3  /* -> TableBudgetError (MemoryError)    */
#define MSG_ERR_UNSUPPORTED -4  /* -> NotImplementedError (GPU limits)  */
#define MSG_ERR_CUDA        -5  /* -> RuntimeError                      */
#define MSG_ERR_WORKSPACE   -6  /* -> ValueError (workspace too small)  */

/* element types */
#define MSG_F32  0
#define MSG_F16  1
#define MSG_F64  2
#define MSG_I32  3
#define MSG_I64  4
#define MSG_U8   5
#define MSG_I8   6
#define MSG_I16  7
#define MSG_BF16 8

/* scale modes (packing.py:21-36 ScaleSpec) */
#define MSG_SCALE_NONE      0
#define MSG_SCALE_PER_ROW   1
#define MSG_SCALE_PER_GROUP 2

/* msg_gemm flags */
#define MSG_FLAG_F32_ENTRIES   1  /* fp32 table entries even for fp16 X (exact-int mode)  */
#define MSG_FLAG_NO_SYMMETRY   2  /* full 16^d tables (default: sign-symmetric half tables) */
#define MSG_FLAG_FORCE_GENERIC 4  /* global-memory table path (any d, width, dtype)        */
#define MSG_FLAG_LUT_PHASE_ONLY 8 /* measurement: launch only the fused LUT kernel (Y untouched;
                                     a LANE workspace keeps the sums and must be re-zeroed) */
#define MSG_FLAG_NO_LANE      16  /* do not use the b=1 lane kernel (use the row-block kernel) */
#define MSG_FLAG_NO_ROWBLOCK  32  /* do not use the batched d=3 row-block kernel (use the generic fused kernel) */
#define MSG_FLAG_RB_ROWS8    128  /* tuning: the b >= 8 row-block kernel with 4096-row CTAs (MSG_LAYOUT_RB4S) */
#define MSG_FLAG_RB_ROWS16   256  /* tuning: the b >= 8 row-block kernel with 8192-row CTAs (MSG_LAYOUT_RB4)  */
#define MSG_FLAG_STATIC_WEIGHTS 64 /* the repacked weights were not written by the kernel launched just
                                      before on this stream: the LUT kernel may start streaming them
                                      before that kernel completes (programmatic dependent launch) */

/* weight layouts produced by msg_repack */
#define MSG_LAYOUT_NONE 0  /* reference row-major nibbles only      */
#define MSG_LAYOUT_QUAD 1  /* quad planes for the fused LUT kernel  */
#define MSG_LAYOUT_LANE 2  /* lane-rotated 32-group chunks for the b=1, d=3 GEMV kernel */
/* 3: retired */
#define MSG_LAYOUT_RB4  4  /* row-block planes, rounds of 4 groups (b >= 8: 8-column tiles)  */
#define MSG_LAYOUT_RB8  5  /* row-block planes, rounds of 8 groups (b = 4..7: 4-column tiles) */
#define MSG_LAYOUT_RB16 6  /* row-block planes, rounds of 16 groups (b = 2, 3: 2-column tiles) */
#define MSG_LAYOUT_RB4S 7  /* as RB4 with rotations for 8 rows per thread (4096-row CTAs)     */

MSG_API const char* msg_last_error(void);
MSG_API int msg_version(void);
MSG_API int msg_device_sm_count(void);

/* ---------- host path helpers (no reference counterpart) ---------- */
/* Launch an instantiated CUDA graph (the drop-in host path's captured
 * H2D -> msg_gemm -> D2H sequence) on `stream`; sync != 0 also waits for it. */
MSG_API int msg_graph_run(void* graph_exec, void* stream, int sync);
MSG_API int msg_stream_sync(void* stream);

/* ---------- packing (packing.py) ---------- */

/* codes (m,k) uint8 -> packed (m,row_bytes) ; packing.py:99-114 _pack_code_rows */
MSG_API int msg_pack_codes(const uint8_t* codes, int64_t m, int64_t k, int width,
                   uint8_t* packed, void* stream);

/* packed -> codes (m,k) uint8 ; packing.py:117-128 _unpack_code_rows / :172-174 codes */
MSG_API int msg_unpack_codes(const uint8_t* packed, int64_t m, int64_t k, int width,
                     uint8_t* codes, void* stream);

/* packed -> int64 (m, k/d) group indices ; packing.py:219-228 group_indices */
MSG_API int msg_group_indices(const uint8_t* packed, int64_t m, int64_t k, int width, int d,
                      int64_t* out, void* stream);

/* values (m,k) of dtype -> packed codes by nearest codebook value, after
 * dividing out per-element scale grid (optional, same dtype as values, f64);
 * bad_count receives the number of non-representable weights (device int64)
 * and bad_first the flat index of the first one.  packing.py:146-169 pack */
MSG_API int msg_encode_values(const double* weights, const double* grid, int64_t m, int64_t k,
                      int width, const double* values,
                      uint8_t* packed, int64_t* bad_count_and_first, void* stream);

/* Conditioning of sign-symmetric tables per row (new; no reference
 * counterpart -- the reference keeps full tables, lut.py:59-72).  ratio[i]
 * (device float, m entries) = sqrt(sum_j (sum_{r<d} |v[c_jr]-beta|)^2) /
 * sum_c |v[c_ic]| for width-4 rows: the expected half-table rounding error of
 * row i relative to the reference's tolerance bound sum_c |W_ic||x_c|
 * (suites.py:106-124) at unit activations; +inf for rows without a nonzero
 * weight (they must come out exactly 0) or with fewer than min(8, ceil(k/2))
 * nonzero weights (their bound rests on a few |x_c|).  The Python layer computes rows
 * above a dtype-dependent threshold with full tables instead. */
MSG_API int msg_row_conditioning(const uint8_t* packed, int64_t m, int64_t k, int d,
                                 const double* values, double beta, float* ratio, void* stream);

/* Row gather / scatter of n rows of row_bytes bytes: scatter != 0 ->
 * dst[idx[i]] = src[i]; else dst[i] = src[idx[i]].  idx: device int64 (n,). */
/* Copy `bytes` from src to dst with a kernel (16-byte aligned; src may be
 * pinned host memory, read over PCIe under UVA): unlike a memcpy node, the
 * kernel lets the next kernel of the stream start its prologue (PDL), so the
 * host path's LUT kernel prefetches weights while X arrives. */
MSG_API int msg_stage_copy(const void* src, void* dst, int64_t bytes, void* stream);
MSG_API int msg_copy_rows(const void* src, const int64_t* idx, int64_t n, int64_t row_bytes,
                          void* dst, int scatter, void* stream);

/* ---------- phase 1 (lut.py) ---------- */

/* Full table for one activation vector x (k,) with stride `ldx` elements:
 * entries (k/d, 2^(width*d)) of dtype; built with the reference's rounding
 * order (lut.py:59-72).  lut.py:98-127 build_lut / :88-95 build_lut_block
 * (block_lo/block_hi select a block range). */
MSG_API int msg_lut_build(const void* x, int dtype, int64_t k, int64_t ldx, int d,
                  const double* values, int width, int64_t block_lo, int64_t block_hi,
                  void* entries, void* stream);

/* ---------- K3: weight repack ---------- */
MSG_API int64_t msg_repacked_bytes(int64_t m, int64_t k, int d, int layout);
/* symmetric=1 folds the sign symmetry of an antisymmetric codebook into the
 * stored indices (top index bit -> complement + sign bit). */
MSG_API int msg_repack(const uint8_t* packed, int64_t m, int64_t k, int d, int layout,
               int symmetric, uint8_t* out, void* stream);

/* ---------- K1+K2: msGeMM (gemm.py:89-153) ---------- */

/* Which layout msg_gemm needs for these arguments (MSG_LAYOUT_*), and the
 * workspace it needs; returns <0 on argument error.  For MSG_LAYOUT_LANE the
 * workspace holds the kernel's int64 row sums and tile counters: it must be
 * zero-filled before its first use and dedicated to LANE calls on one stream
 * (every call leaves it zero again). */
MSG_API int msg_gemm_plan(int64_t m, int64_t k, int width, const double* values, int x_dtype,
                  int64_t b, int d, int scale_mode, int64_t group_size, int flags,
                  int* layout_out, int* symmetric_out, int64_t* workspace_bytes_out);

/* Y (m,b) = dequant(W) @ X with the two-phase LUT algorithm.
 * packed: reference layout (always required); wrep: msg_repack output for
 * the layout msg_gemm_plan returned (may be NULL when that layout is NONE).
 * q: scales (PerRow (m,), PerGroup (m, k/group_size)) of q_dtype or NULL. */
MSG_API int msg_gemm(const uint8_t* packed, const uint8_t* wrep, int64_t m, int64_t k, int width,
             const double* values, const void* x, int x_dtype, int64_t b, int d,
             int scale_mode, int64_t group_size, const void* q, int q_dtype,
             void* y, int y_dtype, void* workspace, int64_t workspace_bytes,
             int flags, void* stream);

/* msg_gemm whose finishing kernels store every element of Y also into
 * n_peers (0..7) more buffers at the same element offset: y_peers[i] is the
 * address in another rank's Y that corresponds to y (mapped peer memory, e.g.
 * torch symmetric memory over NVLink; 16-byte aligned like y).  A row-sharded
 * call (sharded.py) thus leaves its slice in every rank's Y -- the all-gather
 * of SURVEY.md 8(e) fused into the epilogue; the ranks still need a barrier
 * before reading.  NOT_SUPPORTED on the generic (global-table) path. */
MSG_API int msg_gemm_fanout(const uint8_t* packed, const uint8_t* wrep, int64_t m, int64_t k,
                            int width, const double* values, const void* x, int x_dtype,
                            int64_t b, int d, int scale_mode, int64_t group_size, const void* q,
                            int q_dtype, void* y, int y_dtype, void* workspace,
                            int64_t workspace_bytes, int flags, void* stream,
                            void* const* y_peers, int n_peers);

/* ---------- K4: dequantise-then-MMA comparison kernel (gemm.py:206-216 naive_gemm) ---------- */
/* bytes of the tensor-core tile layout of W ([m/128][k/64][128][32 B], nibbles
 * permuted for the fp16 magic-number dequantisation) */
MSG_API int64_t msg_mma_layout_bytes(int64_t m, int64_t k);
/* int4 / uint4 codebooks only (NOT_SUPPORTED otherwise) */
MSG_API int msg_repack_mma(const uint8_t* packed, int64_t m, int64_t k, const double* values,
                           uint8_t* out, void* stream);
MSG_API int64_t msg_dequant_mma_workspace_bytes(int64_t m, int64_t k, int64_t b);
/* Y (m,b) = dequant(W) @ X, X fp16 (k,b), 1 <= b <= 256; tcgen05.mma kind::f16
 * with fp32 accumulation in TMEM; Y of y_dtype (fp32 or fp16). */
MSG_API int msg_dequant_mma(const uint8_t* wmma, int64_t m, int64_t k, const double* values,
                            const void* x, int x_dtype, int64_t b, void* y, int y_dtype,
                            void* workspace, int64_t workspace_bytes, void* stream);

/* Dense comparison baseline for small batches: Y (m,b) = dequant(W) @ X from
 * the reference packed layout (no repack), int4/uint4 codebooks, fp16 X,
 * 1 <= b <= 8, rows of a multiple of 16 bytes (k % 32 == 0); CUDA-core
 * dequantise + exact fp16 x fp16 -> fp32 FMAs, HBM-bound at b = 1..2.
 * gemm.py:206-216 naive_gemm(dense(pwm), X) semantics as msg_dequant_mma. */
MSG_API int msg_dequant_gemv(const uint8_t* packed, int64_t m, int64_t k, const double* values,
                             const void* x, int x_dtype, int64_t b, void* y, int y_dtype,
                             void* stream);

/* Dense comparison baseline for 1 <= b <= 16, same inputs and result contract
 * as msg_dequant_gemv: the packed rows are streamed once, dequantised in
 * registers and multiplied with mma.sync m16n8k16 (fp32 accumulation); split
 * k across a thread-block cluster, partial tiles summed through distributed
 * shared memory in rank order (one kernel, no workspace, deterministic). */
MSG_API int msg_dequant_hmma(const uint8_t* packed, int64_t m, int64_t k, const double* values,
                             const void* x, int x_dtype, int64_t b, void* y, int y_dtype,
                             void* stream);

/* ---------- dense reference product (gemm.py:206-216 naive_gemm) ---------- */
/* Y (m,b) = W (m,k) @ X (k,b), operands of any supported dtype, converted
 * in-kernel.  mode 0: both integer -> int64 Y, wrapping int64 arithmetic
 * (numpy's int64 matmul); 1: fp16 Y, fp32 sum of exact products in k order
 * (numpy's half loop, bit-exact); 2: f32 Y, 3: f64 Y, both from a fp64 sum in
 * k order (numpy uses BLAS there: same values within rounding).  The Python
 * layer picks the mode from np.result_type(W, X) like numpy does. */
MSG_API int msg_naive_gemm(const void* w, int w_dtype, const void* x, int x_dtype, int64_t m,
                           int64_t k, int64_t b, int mode, void* y, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MSGEMM_B200_H */
