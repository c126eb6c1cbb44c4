/*
 * lpqt_b200.h — C ABI of liblpqt_b200.so, the sm_100a FP6 (e3m2) W6A16 path.
 *
 * The reference (`lpqt` 0.1.0, /root/reference/pkg/src/lpqt) is a pure-Python
 * package with no FFI; each entry point below replaces one reference function
 * on the hot path (cited as file:line) and is what a ctypes / cffi binding
 * of that function binds to.  The Python package
 * `paper_2312_08583_b200` is the in-repo binding.
 *
 * Conventions
 *  - Plain pointers + sizes; every pointer is DEVICE memory unless noted.
 *  - Every call is asynchronous on the caller's `stream` (a cudaStream_t
 *    passed as void*; NULL = legacy default stream) and allocates nothing:
 *    callers pass workspaces sized by the *_bytes() queries.
 *  - Return value: LPQT_OK or a negative LPQT_E_* code for argument errors
 *    detected on the host.  Data-dependent errors (non-finite weights, a scale
 *    that overflows binary16, a folded scale above 65504) are OR-ed as
 *    LPQT_F_* bits into the caller's device word `dev_flags`, which the
 *    caller zeroes before and reads after the call (the Python binding maps
 *    them to the reference's InvalidInput / ScaleOverflow exceptions,
 *    errors.py:8, :32).
 *  - dtype codes: LPQT_F64, LPQT_F32, LPQT_F16, LPQT_BF16.
 */
#ifndef LPQT_B200_H_
#define LPQT_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (host-detected) — errors.py:4-53 ------------------- */
#define LPQT_OK                 0
#define LPQT_E_INVALID_INPUT   -1   /* InvalidInput      errors.py:8   */
#define LPQT_E_SHAPE           -2   /* ShapeError        errors.py:28  */
#define LPQT_E_SCALE_OVERFLOW  -3   /* ScaleOverflow     errors.py:32  */
#define LPQT_E_PAYLOAD         -4   /* PayloadMismatch   errors.py:24  */
#define LPQT_E_INVALID_CODE    -5   /* InvalidCode       errors.py:20  */
#define LPQT_E_UNSUPPORTED     -6   /* dtype/layout not offered         */
#define LPQT_E_WORKSPACE       -7   /* workspace too small              */
#define LPQT_E_CUDA           -100  /* CUDA launch/driver failure       */

/* ---- device flag bits (data-dependent errors) --------------------------- */
#define LPQT_F_NONFINITE      1u    /* quantizer.py:200-201, codec.py:119-120 -> InvalidInput */
#define LPQT_F_SCALE_INF      2u    /* quantizer.py:150-151                  -> InvalidInput */
#define LPQT_F_FOLD_OVERFLOW  4u    /* dequant.py:66-68                       -> ScaleOverflow */
#define LPQT_F_BAD_SCALE      8u    /* dequant.py:63-64 (scale <= 0 / inf)    -> InvalidInput */
#define LPQT_F_BAD_CODE      16u    /* packing.py:56-60 code >= 64            -> InvalidCode  */

/* ---- dtype / layout codes ------------------------------------------------ */
#define LPQT_F64   0
#define LPQT_F32   1
#define LPQT_F16   2
#define LPQT_BF16  3

#define LPQT_Y_NM  0   /* Y[n, m] (reference layout, gemm.py:65 returns N x M) */
#define LPQT_Y_MN  1   /* Y[m, n] (torch.nn.Linear layout)                     */

const char* lpqt_strerror(int status);
int lpqt_abi_version(void);               /* bumps on any signature change (6: ablation rebuild flags, native FP5 tiles, sub-tile FGQ, encode self-test) */

/* codec.py:116-132 encode_rtn_array: x[n] (dtype) -> codes[n] (u8). */
int lpqt_fp6_encode_rtn(const void* x, int dtype, int64_t n, uint8_t* codes,
                        uint32_t* dev_flags, void* stream);

/* packing.py:63-90 pack: codes[n] -> canonical seg4[seg4_length(n)],
 * seg2[tail_length(n)] (pad bytes written as zero). */
int lpqt_fp6_pack(const uint8_t* codes, int64_t n, uint8_t* seg4, uint8_t* seg2,
                  uint32_t* dev_flags, void* stream);
/* packing.py:93-118 unpack: canonical planes -> codes[n]. */
int lpqt_fp6_unpack(const uint8_t* seg4, const uint8_t* seg2, int64_t n,
                    uint8_t* codes, void* stream);
int64_t lpqt_fp6_seg4_length(int64_t n);  /* packing.py:28-30 */
int64_t lpqt_fp6_tail_length(int64_t n);  /* packing.py:33-36 */

/* dequant.py:61-69 fold_scale_array: f16 scales[n] -> folded[n] = S * 2^12. */
int lpqt_fp6_fold_scales(const uint16_t* scales, int64_t n, uint16_t* folded,
                         uint32_t* dev_flags, void* stream);

/* dequant.py:82-86 dequant_bias_shift_array (elementwise, f16 out) and
 * dequant.py:72-79 dequant_naive_array.  `scale` is per element. */
int lpqt_fp6_dequant_bias_shift(const uint8_t* codes, const uint16_t* folded,
                                int64_t n, uint16_t* out, void* stream);
int lpqt_fp6_dequant_naive(const uint8_t* codes, const uint16_t* scales,
                           int64_t n, uint16_t* out, void* stream);

/* quantizer.py:189-248 quantize_tensor, CGQ x FP6_E3M2 (one scale per row).
 * W[N, K] row-major with row stride ldw (elements), any LPQT_* dtype.
 * Writes scales[N] (f16 bits), folded[N] when bias_shift, and the canonical
 * planes seg4/seg2 of the row-major code stream (flat index r*K + k).
 * `codes_ws` is ignored (ABI v1 argument; pass NULL).  Two launches: row
 * scales, then encode + pack (8 codes per thread). */
int lpqt_fp6_quantize_pack(const void* W, int dtype, int64_t N, int64_t K,
                           int64_t ldw, int bias_shift, uint16_t* scales,
                           uint16_t* folded, uint8_t* seg4, uint8_t* seg2,
                           uint8_t* codes_ws, uint32_t* dev_flags, void* stream);

/* quantizer.py:269-299 dequantize_tensor for CGQ FP6 from canonical planes:
 * out[N, K] = compose[c] * folded[row] (path 1, "bias_shift") or
 * value[c] * scales[row] (path 0, "naive"); out dtype F64 (exact, the
 * reference's return type) or F16 (the bias-shift binary16 rounding). */
int lpqt_fp6_dequantize_tensor(const uint8_t* seg4, const uint8_t* seg2,
                               const uint16_t* row_scale, int path,
                               int64_t N, int64_t K, void* out, int out_dtype,
                               void* stream);

/* ---- B200 weight tile layout (new; no reference counterpart) -------------
 * The GEMM consumes weights in a tile-contiguous layout: 128-row x 128-k
 * tiles of 12288 bytes (6 bits/weight) stored [row_tile][k_tile], N and K
 * zero-padded to multiples of 128.  The canonical planes stay the parity
 * artifact; prepack/unprepack are exact inverses. */
int64_t lpqt_fp6_tiles_bytes(int64_t N, int64_t K);
int lpqt_fp6_prepack(const uint8_t* seg4, const uint8_t* seg2, int64_t N,
                     int64_t K, uint8_t* tiles, void* stream);
/* quantize_tensor (quantizer.py:189-248) straight into the tile layout:
 * scales[N] (+ folded[N] when bias_shift) exactly as lpqt_fp6_quantize_pack,
 * and tiles (lpqt_fp6_tiles_bytes(N, K) bytes) equal to
 * prepack(quantize_pack(W)) byte for byte, without the canonical planes. */
int lpqt_fp6_quantize_tiles(const void* W, int dtype, int64_t N, int64_t K,
                            int64_t ldw, int bias_shift, uint16_t* scales,
                            uint16_t* folded, uint8_t* tiles,
                            uint32_t* dev_flags, void* stream);
int lpqt_fp6_unprepack(const uint8_t* tiles, int64_t N, int64_t K,
                       uint8_t* codes, void* stream);
/* Standalone transform (the GEMM's register dequant): tiles -> out[N, K]
 * f16 = value_f16[c] * S[row] rounded to binary16 (dequant.py:72-79), which
 * equals the bias-shift result compose[c] * (S * 2^12) bit for bit
 * (dequant.py:82-86; the reference's exhaustive test_dequant.py:93-102). */
int lpqt_fp6_tiles_dequant(const uint8_t* tiles, const uint16_t* scales,
                           int64_t N, int64_t K, uint16_t* out, void* stream);

/* Activation staging: X in the reference layout [K, M] (gemm.py:65, any
 * dtype, row stride ldx) -> Xt[M, Kp] f16 row-major (K-major operand),
 * Kp = round_up(K, 8), pad columns zero.  Values round to binary16 (A16). */
int lpqt_stage_activations(const void* X, int dtype, int64_t K, int64_t M,
                           int64_t ldx, uint16_t* Xt, int64_t Kp, void* stream);

/* gemm.py:65-94 gemm_quantized (CGQ FP6): Y = diag(S * 2^12) * (C . X) where
 * C holds the bias-shifted code values (== diag(S) * (V . X), exactly); the
 * fold S * 2^12 (dequant.py:46-69) is formed in an fp32 register, so it is
 * exact and has no binary16 overflow limit.
 * tiles: prepacked weights; scales[N] f16 bits (S); Xt[M, ldx] f16 K-major
 * (ldx >= K, ldx % 8 == 0, 16-B aligned); Y per y_dtype (F32/F16/BF16)
 * and y_layout (LPQT_Y_NM: Y[n*ldy + m]; LPQT_Y_MN: Y[m*ldy + n]).
 * split_k: 0 = auto (plan below), else forced.  The kernel is tcgen05 (A =
 * dequantized weights in TMEM, B = X via TMA, fp32 accumulate in TMEM).
 * Workspace: lpqt_w6a16_workspace_bytes(); it must be zeroed once at
 * allocation (split-K tile counters are self-resetting). */
int64_t lpqt_w6a16_workspace_bytes(int64_t M, int64_t N, int64_t K, int split_k);
int lpqt_w6a16_plan(int64_t M, int64_t N, int64_t K, int split_k,
                    int* block_n, int* splits, int* grid, int* stages);
/* Plan with schedule flags: out[0..5] = block_n, splits, grid, stages,
 * schedule (0 stream-K, 1 cluster split-K, 2 whole tiles round-robin —
 * prefill whose activations outgrow L2), cluster size (n_out <= 6). */
int lpqt_w6a16_plan_ex(int64_t M, int64_t N, int64_t K, int split_k, int flags,
                       int* out, int n_out);
int lpqt_w6a16_linear(const uint8_t* tiles, const uint16_t* scales,
                      const uint16_t* Xt, int64_t ldx, int64_t M, int64_t N,
                      int64_t K, void* Y, int y_dtype, int y_layout,
                      int64_t ldy, int split_k, void* workspace,
                      int64_t workspace_bytes, void* stream);

/* Same, with launch flags.  LPQT_LAUNCH_PDL launches the kernel with
 * programmatic dependent launch: it may start while the preceding kernel on
 * the stream is still running; it streams and dequantizes weight tiles at
 * once and waits for the preceding grid only before reading Xt and writing
 * Y / the workspace.  The caller guarantees the tiles and scales are not
 * written by any kernel still in flight on the stream (true for weights
 * quantized ahead of time).  Back-to-back layers then overlap one kernel's
 * tail with the next one's weight prefetch. */
#define LPQT_LAUNCH_PDL 1
/* Schedule overrides (default: automatic).  LPQT_SCHED_STREAMK forces the
 * stream-K schedule (split_k > 0: about split_k CTAs per tile);
 * LPQT_SCHED_CLUSTER forces cluster split-K with a cluster of split_k CTAs
 * (k-split factor, 1..8) for decode batches (M <= 32). */
#define LPQT_SCHED_STREAMK 2
#define LPQT_SCHED_CLUSTER 4
/* Prefill (CGQ, even number of 128-row weight tiles): the CTA-pair kernel
 * (tcgen05 cta_group::2, M = 256 x N = 256 MMAs, prefill2sm.cu) is picked by
 * a time model; LPQT_SCHED_PAIR forces it where the shape allows,
 * LPQT_SCHED_SINGLE forbids it (A/B hooks). */
#define LPQT_SCHED_SINGLE 8
#define LPQT_SCHED_PAIR 16
/* The paper's Bias-Shift ablation ("the same FP6 kernel
 * without Bias-Shift"), decode batches M <= 16, CGQ FP6 only (else
 * LPQT_E_UNSUPPORTED).  The product kernel rebuilds weights with the
 * hardware e3m2 converter and applies S in fp32 after the contraction
 * (gemm.py:84-88); these flags swap in the paper's software rebuilds, each
 * followed by the per-weight binary16 scale multiply of the reference's
 * dequant paths:
 *   LPQT_REBUILD_BIAS_SHIFT  compose (sign << 15 | eeemm << 8, dequant.py:37-41)
 *                            x folded scale S * 2^12 (dequant.py:82-86);
 *   LPQT_REBUILD_NAIVE       exponent + 12, subnormals x 2^12, then x S
 *                            (dequant_naive_array, dequant.py:72-79).
 * Both give the binary16 dequantized weight bit for bit (so identical Y).
 * Folded scales above 65504 (S > 15.99) overflow under BIAS_SHIFT, as in
 * the reference (ScaleOverflow). */
#define LPQT_REBUILD_BIAS_SHIFT 32
#define LPQT_REBUILD_NAIVE 64
/* `tiles` are native FP5 tiles (lpqt_fp5n_prepack), CGQ; single-SM kernels
 * (decode and prefill), no pair kernel, no LPQT_REBUILD_* */
#define LPQT_WEIGHTS_FP5 128

/* Self-test of the quantizer's division-free RTN quotient (not a reference
 * interface): every positive finite binary16 scale against every positive
 * finite binary16 (dtype LPQT_F16) / bfloat16 (LPQT_BF16) weight with
 * |w| <= 29 S, e3m2 codes and f32 quotients against the __fdiv_rn path.
 * out3[0] = code mismatches, out3[1] = quotient mismatches, out3[2] = pairs.
 * Synchronous. */
int lpqt_selftest_fp6_encode(int dtype, unsigned long long* out3);
int lpqt_w6a16_linear_ex(const uint8_t* tiles, const uint16_t* scales,
                         const uint16_t* Xt, int64_t ldx, int64_t M, int64_t N,
                         int64_t K, void* Y, int y_dtype, int y_layout,
                         int64_t ldy, int split_k, void* workspace,
                         int64_t workspace_bytes, int flags, void* stream);

/* The linear that will run next on the same stream (decode chains: QKV ->
 * O -> gate_up -> down -> next block's QKV).  With it, each CTA of this
 * launch, once it has requested its last weight tile, issues bulk L2
 * prefetches (cp.async.bulk.prefetch.L2) of the first `bytes_per_cta`
 * bytes that the matching CTA of the next launch will stream (derived from
 * that launch's plan; 0 = 64 KiB).  Weights are static, so this only moves
 * HBM reads earlier: HBM keeps streaming through this launch's drain and
 * the next one's start-up.  Ignored when the next launch has more than one
 * batch tile (prefill).  Not a reference interface (no counterpart). */
typedef struct lpqt_next_linear {
  const uint8_t* tiles;   /* next weight, tile layout */
  int64_t M, N, K;        /* next problem (plan inputs) */
  int split_k, flags;     /* next launch's split_k / schedule flags */
  int64_t bytes_per_cta;  /* prefetch depth per next-launch CTA */
} lpqt_next_linear;

/* Fused GEMM + all-gather over peer memory (column-parallel TP).
 * Every rank runs its row shard's GEMM and its epilogue stores each output
 * element straight into every peer's (NVLink P2P / symmetric) copy of the
 * full Y: y[p] is peer p's Y buffer already offset to this rank's block (NM
 * layout: + row0 * ldy, MN layout: + row0), same dtype / layout / ldy on all
 * peers.  Completion is part of the same kernel: each CTA fences its stores
 * at system scope and counts itself in `done` (a zeroed int the caller owns,
 * reset by the kernel); the last CTA writes `epoch` into slot `rank` of every
 * peer's flag array (flags[p], LPQT_MAX_PEERS u32, zeroed once) and waits
 * until its own array holds >= epoch from every peer.  When the kernel
 * completes, Y is whole on this GPU.  epoch: strictly increasing per call
 * (wrapping compare); the caller must not reuse a Y buffer a slower peer
 * may still be reading (the Python wrapper alternates two).  npeers = 1
 * (y[0] = own buffer) is a plain launch plus the counter. */
#define LPQT_MAX_PEERS 8
typedef struct lpqt_peer_out {
  void* y[LPQT_MAX_PEERS];
  uint32_t* flags[LPQT_MAX_PEERS];
  int npeers, rank;
  uint32_t epoch;
  int* done;
} lpqt_peer_out;

int lpqt_w6a16_linear_gather(const uint8_t* tiles, const uint16_t* scales,
                             int64_t block, const uint16_t* Xt, int64_t ldx,
                             int64_t M, int64_t N, int64_t K, int y_dtype,
                             int y_layout, int64_t ldy, int split_k,
                             void* workspace, int64_t workspace_bytes,
                             int flags, const lpqt_peer_out* peers,
                             void* stream);

int lpqt_w6a16_linear_pf(const uint8_t* tiles, const uint16_t* scales,
                         const uint16_t* Xt, int64_t ldx, int64_t M, int64_t N,
                         int64_t K, void* Y, int y_dtype, int y_layout,
                         int64_t ldy, int split_k, void* workspace,
                         int64_t workspace_bytes, int flags,
                         const lpqt_next_linear* next, void* stream);

/* ---- FGQ x FP6 (quantizer.py FGQ blocks :91-115, gemm.py:96-110) ---------
 * One binary16 scale per (row, block of `block` columns), stored row-major
 * (index r * ceil(K / block) + j); block <= 0 or >= K is CGQ (one per row),
 * identical to the entries above.  Quantize / dequantize accept any block
 * size; the GEMM takes blocks of whole 128-k tiles (block % 128 == 0, else
 * LPQT_E_UNSUPPORTED) and applies each block's scale to the rebuilt binary16
 * weights before the MMA (the binary16 dequant of dequant.py:72-79).
 * lpqt_w6a16_linear_blocks with 0 < block < K reads `scales` as the
 * STAGE-ORDERED block scales (lpqt_fgq_stage_params, below), not the
 * row-major array; with block <= 0 or >= K they are the per-row scales. */
int lpqt_fp6_quantize_pack_blocks(const void* W, int dtype, int64_t N,
                                  int64_t K, int64_t ldw, int64_t block,
                                  int bias_shift, uint16_t* scales,
                                  uint16_t* folded, uint8_t* seg4,
                                  uint8_t* seg2, uint32_t* dev_flags,
                                  void* stream);
int lpqt_fp6_quantize_tiles_blocks(const void* W, int dtype, int64_t N,
                                   int64_t K, int64_t ldw, int64_t block,
                                   int bias_shift, uint16_t* scales,
                                   uint16_t* folded, uint8_t* tiles,
                                   uint32_t* dev_flags, void* stream);
int lpqt_fp6_dequantize_tensor_blocks(const uint8_t* seg4, const uint8_t* seg2,
                                      const uint16_t* block_scale, int path,
                                      int64_t N, int64_t K, int64_t block,
                                      void* out, int out_dtype, void* stream);
int lpqt_fp6_tiles_dequant_blocks(const uint8_t* tiles, const uint16_t* scales,
                                  int64_t N, int64_t K, int64_t block,
                                  uint16_t* out, void* stream);
int lpqt_w6a16_linear_blocks(const uint8_t* tiles, const uint16_t* scales,
                             int64_t block, const uint16_t* Xt, int64_t ldx,
                             int64_t M, int64_t N, int64_t K, void* Y,
                             int y_dtype, int y_layout, int64_t ldy,
                             int split_k, void* workspace,
                             int64_t workspace_bytes, int flags,
                             const lpqt_next_linear* next, void* stream);

/* ---- FP5 e3m1 (codec.py FP5_E3M1, packing.py 4 + 1 split) ----------------
 * Same contracts as the FP6 entries with seg4 = c >> 1 (align4(ceil(n/2)) B)
 * and a one-bit tail (lpqt_fp5_tail_length(n) = align4(ceil(n/8)) B, little-
 * endian bit order).  Scales are peak / 24 (max_value).  FP5 weights run the
 * GEMM through the FP6 tile layout (lpqt_fp5_prepack: every e3m1 value is an
 * e3m2 value), i.e. at FP6's 0.75 B per weight. */
int64_t lpqt_fp5_tail_length(int64_t n);
int lpqt_fp5_encode_rtn(const void* x, int dtype, int64_t n, uint8_t* codes,
                        uint32_t* dev_flags, void* stream);
int lpqt_fp5_pack(const uint8_t* codes, int64_t n, uint8_t* seg4,
                  uint8_t* seg1, uint32_t* dev_flags, void* stream);
int lpqt_fp5_unpack(const uint8_t* seg4, const uint8_t* seg1, int64_t n,
                    uint8_t* codes, void* stream);
int lpqt_fp5_quantize_pack_blocks(const void* W, int dtype, int64_t N,
                                  int64_t K, int64_t ldw, int64_t block,
                                  int bias_shift, uint16_t* scales,
                                  uint16_t* folded, uint8_t* seg4,
                                  uint8_t* seg1, uint32_t* dev_flags,
                                  void* stream);
int lpqt_fp5_dequantize_tensor_blocks(const uint8_t* seg4, const uint8_t* seg1,
                                      const uint16_t* block_scale, int path,
                                      int64_t N, int64_t K, int64_t block,
                                      void* out, int out_dtype, void* stream);
int lpqt_fp5_dequant_bias_shift(const uint8_t* codes, const uint16_t* folded,
                                int64_t n, uint16_t* out, void* stream);
int lpqt_fp5_dequant_naive(const uint8_t* codes, const uint16_t* scales,
                           int64_t n, uint16_t* out, void* stream);
int lpqt_fp5_prepack(const uint8_t* seg4, const uint8_t* seg1, int64_t N,
                     int64_t K, uint8_t* tiles, void* stream);

/* FP5 e3m1 in its own 4+1 tile layout (0.625 B per weight, vs the FP6 tiles'
 * 0.75 of lpqt_fp5_prepack): 128 x 128 tiles of 10240 B — a s|eee nibble
 * plane and a mantissa bit plane per 32-weight group, arranged so the GEMM's
 * rebuild is two shifts + two logic ops per four weights ahead of the
 * hardware e3m2 converter (common.cuh).  Planes as packing.py:84-85
 * (seg4 = c >> 1, seg1 = c & 1).  For lpqt_w6a16_linear_blocks with
 * LPQT_WEIGHTS_FP5 (CGQ only).  Not a reference interface (a layout change
 * like lpqt_fp6_prepack). */
int64_t lpqt_fp5n_tiles_bytes(int64_t N, int64_t K);
int lpqt_fp5n_prepack(const uint8_t* seg4, const uint8_t* seg1, int64_t N,
                      int64_t K, uint8_t* tiles, void* stream);
/* inverse -> row-major e3m1 codes[N, K] (uint8) */
int lpqt_fp5n_unprepack(const uint8_t* tiles, int64_t N, int64_t K,
                        uint8_t* codes, void* stream);
/* tiles -> out[N, K] binary16 = value_f16[c] * S[n] through the GEMM's
 * rebuild (dequant_naive_array, dequant.py:72-79) */
int lpqt_fp5n_tiles_dequant(const uint8_t* tiles, const uint16_t* scales,
                            int64_t N, int64_t K, uint16_t* out, void* stream);

/* ---- INT4 asymmetric, CGQ / FGQ (quantizer.py:232-244, packing.py:121-141)
 * The paper's comparator format: per block zero point RN_f16(min) and scale
 * RN_f16((max - min) / 15), levels clip(rint((w - Z) / S), 0, 15), two per
 * byte (ceil(n / 2) bytes, even index low nibble); dequantize = Z + S * level
 * in f64.  The comparator GEMM dequantizes and calls a library GEMM. */
int lpqt_int4_quantize_blocks(const void* W, int dtype, int64_t N, int64_t K,
                              int64_t ldw, int64_t block, uint16_t* scales,
                              uint16_t* zeros, uint8_t* nibbles,
                              uint32_t* dev_flags, void* stream);
int lpqt_int4_pack(const uint8_t* levels, int64_t n, uint8_t* nibbles,
                   uint32_t* dev_flags, void* stream);
int lpqt_int4_unpack(const uint8_t* nibbles, int64_t n, uint8_t* levels,
                     void* stream);
int lpqt_int4_dequantize_blocks(const uint8_t* nibbles, const uint16_t* scales,
                                const uint16_t* zeros, int64_t N, int64_t K,
                                int64_t block, double* out, void* stream);

/* FGQ / INT4 block parameters in GEMM stage order: for weight tile (row tile
 * rt, k tile kt) the 128 rows' f16 scale (with_zeros / INT4: scale | zero
 * << 16, u32) of the block holding kt.  Built once per weight from the
 * row-major per-block arrays (block <= 0 or >= K: one per row, else a
 * multiple of 128); the GEMM's weight producer copies them next to the
 * weight bytes of each stage.  Without zeros (FP6 / FP5) each row's scales
 * are normalised by a power of two 2^e_r (max in [2^10, 2^11)) and the f32
 * row factors 2^e_r follow the stage-ordered scales (the GEMM applies them in
 * fp32).  lpqt_fgq_stage_bytes(N, K, with_zeros) bytes. */
int64_t lpqt_fgq_stage_bytes(int64_t N, int64_t K, int with_zeros);
int lpqt_fgq_stage_params(const uint16_t* scales, const uint16_t* zeros,
                          int64_t N, int64_t K, int64_t block, void* out,
                          void* stream);

/* W4A16 comparator GEMM: INT4 tiles (lpqt_int4_tiles_bytes(N, K) bytes,
 * lpqt_int4_prepack of the nibble payload) and the stage-ordered scale |
 * zero words (lpqt_fgq_stage_params with zeros); the binary16 weight
 * Z + S * level is rebuilt in registers and runs the same tcgen05 pipeline
 * as the FP6 GEMM (flags: LPQT_LAUNCH_PDL, LPQT_SCHED_STREAMK,
 * LPQT_SCHED_CLUSTER; LPQT_SCHED_SINGLE is a no-op — there is no CTA-pair
 * W4A16 kernel, LPQT_SCHED_PAIR is refused with LPQT_E_INVALID_INPUT).
 * block: the parameters' block size (validated). */
int64_t lpqt_int4_tiles_bytes(int64_t N, int64_t K);
int lpqt_int4_prepack(const uint8_t* nibbles, int64_t N, int64_t K,
                      uint8_t* tiles, void* stream);
int lpqt_w4a16_linear_blocks(const uint8_t* tiles, const uint32_t* params,
                             int64_t block, const uint16_t* Xt, int64_t ldx,
                             int64_t M, int64_t N, int64_t K, void* Y,
                             int y_dtype, int y_layout, int64_t ldy,
                             int split_k, void* workspace,
                             int64_t workspace_bytes, int flags,
                             void* stream);

/* Reference-order GEMMs (exact.cu): the reference's loops replayed one
 * thread per output element, k ascending, every product and sum rounded
 * separately — bit-identical to the reference on the same inputs.  They run
 * the reference-API calls the A16 tcgen05 kernel cannot reproduce within the
 * reference's tolerance: float32 / float64 activations, FGQ blocks of any
 * width, INT4 (S * sum(level x) + Z * sum(x)).
 *   lpqt_gemm_exact_quantized — gemm.py:65-110 gemm_quantized: codes [N, K]
 *     uint8 row-major (fmt 0 FP6 e3m2 codes, 1 FP5 e3m1 codes, 2 INT4
 *     levels), f16 scales (and INT4 zero points) one per row (block <= 0 or
 *     >= K) or per block of `block` columns row-major, X [K, M] float32,
 *     Y [N, M] float32.
 *   lpqt_gemm_exact_dense — gemm.py:41-51 gemm_dense (dtype LPQT_F32) and
 *     gemm.py:28-38 gemm_reference (LPQT_F64): W [N, K], X [K, M], Y [N, M]
 *     in that dtype. */
int lpqt_gemm_exact_quantized(const uint8_t* codes, int fmt,
                              const uint16_t* scales, const uint16_t* zeros,
                              int64_t N, int64_t K, int64_t block,
                              const float* X, int64_t M, float* Y,
                              void* stream);
int lpqt_gemm_exact_dense(const void* W, const void* X, int dtype, int64_t N,
                          int64_t K, int64_t M, void* Y, void* stream);

/* Number of kernel launches performed by this library since load (for the
 * bench's gpu_launches claim). */
int64_t lpqt_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* LPQT_B200_H_ */
