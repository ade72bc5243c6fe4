/*
 * entquant.h — C ABI of the B200-native EntQuant hot path (libentquant.so).
 *
 * Paper: "Float8@2bits: Entropy Coding Enables Data-Free Model Compression",
 * arXiv 2601.22787.  P:<n> = line n of PAPER.md, S:<n> = line n of SPEC.md; the
 * readings of ambiguous passages are listed in DESIGN.md §3 and numbered R1..R15.
 *
 * Conventions (all entry points):
 *  - Tensor / array pointers are CUDA DEVICE pointers unless the parameter name ends in
 *    `_host`.  The caller allocates and owns every buffer (PyTorch does, in the binding).
 *    The library is stateless, holds no persistent allocation, is reentrant, and orders
 *    all device work on the given stream.  Structs are read on the host at call time.
 *  - bf16 values are passed as their 16-bit patterns (uint16_t); row-major storage.
 *  - Synchronous errors (bad arguments, shapes, undersized buffers, CUDA launch failures)
 *    are returned before any kernel is queued.  Data-dependent errors found on the device
 *    (corrupt / truncated streams, empty histograms) are OR-ed as EQ_EF_* bits into a
 *    caller-provided device word `d_err` (zero it first); eq_check() maps it to a status.
 *  - Only the entry points documented "synchronous" block the host.
 *  - Errors never write outside the caller's buffers.
 */
#ifndef ENTQUANT_H
#define ENTQUANT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* eq_stream_t;   /* a cudaStream_t; NULL = legacy default */

typedef enum {
    EQ_OK = 0,
    EQ_ERR_ARG = 1,                 /* null pointer, bad enum / parameter value           */
    EQ_ERR_SHAPE = 2,               /* rows/cols invalid or mismatched              */
    EQ_ERR_EMPTY = 3,               /* empty stream / histogram                    */
    EQ_ERR_BUFFER = 4,              /* arena, payload or scratch too small         */
    EQ_ERR_CORRUPT = 5,             /* rANS end-state / length check failed        */
    EQ_ERR_TRUNCATED = 6,           /* chunk offsets outside the payload           */
    EQ_ERR_UNKNOWN_SYMBOL = 7,      /* symbol with zero table frequency            */
    EQ_ERR_UNREACHABLE_TARGET = 8,  /* λ calibration cannot reach the target rate  */
    EQ_ERR_CUDA = 9                 /* a CUDA runtime error                                */
} eq_status;

/* device error-word bits (d_err) */
#define EQ_EF_CORRUPT        0x1u
#define EQ_EF_TRUNCATED      0x2u
#define EQ_EF_EMPTY          0x4u
#define EQ_EF_UNKNOWN_SYMBOL 0x8u
#define EQ_EF_BUFFER         0x10u

#define EQ_FMT_E4M3   0u            /* Float8 E4M3 (torch float8_e4m3fn)            */
#define EQ_FMT_INT8   1u            /* symmetric Int8, codes −127..127        */
#define EQ_OUT_FP8    0u            /* decode to the raw 8-bit codes (E4M3 or Int8; scale  */
                                    /* left to the GEMM epilogue)                          */
#define EQ_OUT_BF16   1u            /* decode + fused per-row dequant to bf16      */

/* rANS renormalisation (the "ANS" of P:155/P:213/P:229; nvCOMP's own is undocumented).
 * Both: 32-bit state, M = 2^12, cum in code order, chunk = 4-byte LE final state followed by
 * the renormalisation units in decode order (R9, R14). */
#define EQ_CODEC_BYTE 0u            /* L = 2^23, byte units (≤ 2 per symbol)    */
#define EQ_CODEC_WORD 1u            /* R14: L = 2^16, 16-bit little-endian word units       */
                                    /* (≤ 1 per symbol: the GPU decoder's fast path)         */
#define EQ_CODEC_PAIR 2u            /* R15: the word codec over PAIRS of the block's top-15   */
                                    /* codes, escape to singles; eq_block.freq then holds   */
                                    /* 512 u16: [0,256) single table, [256,481) pair table  */
                                    /* by ra*15+rb, [481] escape, [482] K, [484,492) rank   */
                                    /* codes as bytes                                        */
#define EQ_CODEC_PAIR_G 3u          /* R18: EQ_CODEC_PAIR's tables and symbols, reordered:   */
                                    /* per 16-symbol group of a chunk, the group's pair     */
                                    /* steps (kept pair or escape), then the two codes of   */
                                    /* each escaped pair in position order, then an odd     */
                                    /* last symbol; same table buffer as EQ_CODEC_PAIR      */

/* Chunking of a block's symbol stream (R10). */
#define EQ_CHUNK_LAYER 0u           /* chunks of chunk_symbols restart at every layer start */
#define EQ_CHUNK_ROW   1u           /* ... and at every row start: a row of K columns is    */
                                    /* ceil(K/cs) chunks (4096+4096+4096+2048 for K=14336),  */
                                    /* independent K slices for eq_qmatmul (§8(f) row 1);    */
                                    /* identical bytes to EQ_CHUNK_LAYER when K % cs == 0    */
#define EQ_CHUNK_INTERLEAVED 2u     /* R17: layer chunking over super-chunks of 32*cs        */
                                    /* symbols whose 16-symbol groups are dealt to their 32  */
                                    /* chunks in turn (chunk j: groups j, j+32, ...); the    */
                                    /* rest of the layer is plain chunks.  A decoder warp's  */
                                    /* stores are then contiguous.  Pair codecs only; needs  */
                                    /* chunk_symbols % 32 == 0 and cols % 16 == 0 (else      */
                                    /* EQ_ERR_ARG / EQ_ERR_SHAPE); not for eq_qmatmul        */

#define EQ_SCALES_SEARCH 0u         /* exhaustive per-row Eq. 4 minimisation (R5)          */
#define EQ_SCALES_ABSMAX 1u         /* AbsMax scales, Eq. 1 (the λ = 0 lossless-FP8 rate)  */
#define EQ_SCALES_GIVEN  2u         /* caller supplies eq_block.scales                     */

#define EQ_MAX_LAYERS 8             /* layers per block (a Llama block has 7)              */
#define EQ_DEFAULT_CHUNK 4096u      /* symbols per chunk (R9)               */
#define EQ_PROB_BITS 12u            /* table precision M = 2^12                    */
#define EQ_PAYLOAD_SLACK 256u       /* bytes of readable slack required after a payload    */
#define EQ_ARENA_ALIGN 256u         /* each decoded layer starts at a multiple of this     */

/* One weight matrix W [rows, cols], bf16 row-major, row = output channel. */
typedef struct {
    const void* w;                  /* device, rows*cols bf16                              */
    int64_t rows, cols;
} eq_tensor;

typedef struct {
    uint32_t format;                /* EQ_FMT_E4M3 | EQ_FMT_INT8                           */
    uint32_t chunk_symbols;         /* 1 .. 262144; default EQ_DEFAULT_CHUNK       */
    uint32_t prob_bits;             /* must be 12                                          */
    uint32_t scale_mode;            /* EQ_SCALES_*                                         */
    double   lambda;                /* Eq. 4 λ ≥ 0, SPEC normalisation (R4)                */
    int32_t  oct_lo, oct_hi;        /* search bracket, octaves around AbsMax (R5): -1, 20  */
    uint32_t exclude_mask;          /* bit l: layer l keeps AbsMax scales (λ = 0) — the    */
                                    /* super-weight exclusion of P:393-396          */
    uint32_t codec;                 /* EQ_CODEC_BYTE (0, default) | _WORD | _PAIR          */
    uint32_t chunk_mode;            /* EQ_CHUNK_LAYER (0, default) | _ROW | _INTERLEAVED     */
} eq_params;

/* One compressed transformer block: all its layers in one bitstream with one table
 * (App. A.1).  Device arrays are caller-allocated; sizes from
 * eq_encode_bounds().  Host fields describe the layers in block order. */
typedef struct {
    uint8_t*  payload;              /* device: chunk streams back to back                 */
    uint64_t  payload_cap;          /* bytes allocated (must include EQ_PAYLOAD_SLACK)    */
    uint64_t  payload_bytes;        /* bytes used (set by eq_quantize_encode)             */
    uint32_t* chunk_off;            /* device: n_chunks+1 byte offsets into payload       */
    uint32_t  n_chunks;
    uint32_t  chunk_symbols;        /* chunk length used when encoding                     */
    uint16_t* freq;                 /* device: 256 normalised frequencies, Σ = 4096       */
                                    /* (512 u16 for EQ_CODEC_PAIR, see above)             */
    uint16_t* scales;               /* device: bf16 per-row scales, layers concatenated   */
    uint32_t  n_layers;
    uint32_t  format;               /* EQ_FMT_* of the symbols (set by eq_quantize_encode) */
    int64_t   layer_rows[EQ_MAX_LAYERS];
    int64_t   layer_cols[EQ_MAX_LAYERS];
    uint32_t  codec;                /* EQ_CODEC_* of the streams (set by eq_quantize_encode) */
    uint32_t  chunk_mode;           /* EQ_CHUNK_* of the streams (set by eq_quantize_encode) */
} eq_block;

/* ---------------------------------------------------------------- library info */
const char* eq_status_string(eq_status s);
const char* eq_version(void);

/* ---------------------------------------------------------------- sizing (host only)
 * Sizes for encoding `n_layers` tensors as one block: payload capacity (worst case 4 bytes
 * per chunk + 2 bytes per symbol for EQ_CODEC_BYTE / _WORD, 3 bytes per symbol for
 * EQ_CODEC_PAIR — an escaped pair is three words — plus slack), chunk count, and the scratch bytes
 * eq_quantize_encode needs (codes stream + tables + chunk sizes).  EQ_ERR_SHAPE for
 * rows/cols < 1 or > 2^31, EQ_ERR_ARG for n_layers outside 1..EQ_MAX_LAYERS. */
eq_status eq_encode_bounds(const eq_tensor* layers, uint32_t n_layers, const eq_params* p,
                           uint64_t* payload_cap, uint32_t* n_chunks, uint64_t* scratch_bytes);

/* Byte offset of each decoded layer inside an arena holding `n_blocks` blocks, in block
 * then layer order, each start aligned to EQ_ARENA_ALIGN; elements are 1 (FP8) or 2
 * (bf16) bytes.  layer_offsets[b*EQ_MAX_LAYERS + l]; *total_bytes = arena size needed. */
eq_status eq_arena_layout(const eq_block* blocks, uint32_t n_blocks, uint32_t out_dtype,
                          uint64_t* layer_offsets, uint64_t* total_bytes);

/* ---------------------------------------------------------------- encode-side steps
 * §8(a) rows a1-a6; each is also used by eq_quantize_encode.  Asynchronous. */

/* a1, Eq. (1), Alg. 1 l.1: s0_i = bf16_rne(max_j |W_ij| / Q_max), Q_max = 448
 * (E4M3) or 127 (Int8); all-zero row -> 1.  s0: device [rows] bf16. */
eq_status eq_absmax(const eq_tensor* w, uint32_t format, uint16_t* s0, eq_stream_t stream);

/* Scratch bytes eq_search_scales needs for `w`. */
uint64_t eq_search_scratch_bytes(const eq_tensor* w);

/* a2, Eq. (4) P:175-188 with R4/R5: for each row i (all rows, or the `n_rows` row indices
 * in device array `rows`) and each of the `n_lambda` host values lambdas_host[k], the bf16
 * scale minimising f_i(s) = Σ_j|W_ij − s·v_ij| / ‖W‖₁ + λ_k·Σ_j|v_ij| / (rows·cols) over the
 * contiguous bf16 patterns in [bf16(s0·2^oct_lo), bf16(s0·2^oct_hi)], smallest s on ties;
 * all-zero rows keep s = 1.  Outputs (device): scales[k*rows + i] and, if obj != NULL,
 * obj[k*rows + i] = f_i(s*).  Terms |W − s·v| are exact f32, sums f64 (deterministic
 * order).  n_lambda ≤ 32. */
eq_status eq_search_scales(const eq_tensor* w, uint32_t format, const double* lambdas_host, uint32_t n_lambda,
                           int32_t oct_lo, int32_t oct_hi, const uint32_t* rows, uint32_t n_rows,
                           uint16_t* scales, double* obj, void* scratch, uint64_t scratch_bytes,
                           eq_stream_t stream);

/* a3 + a4, Alg. 1 l.3: codes = RNE_γ(clamp(W/s, ±Q_max)) — E4M3
 * with −0 → +0, or Int8 (half to even, two's-complement byte) — for all rows (rows == NULL)
 * or the listed rows, written row-major into `codes` (device, rows*cols bytes; may be NULL
 * to only count), and the 256-bin histogram ACCUMULATED into hist (device uint64[256]). */
eq_status eq_quantize_hist(const eq_tensor* w, uint32_t format, const uint16_t* scales, const uint32_t* rows,
                           uint32_t n_rows, uint8_t* codes, uint64_t* hist, eq_stream_t stream);

/* a5 (R8): normalise hist (device uint64[256]) to freq (device uint16[256],
 * Σ = 4096, every present symbol ≥ 1) by the integer largest-remainder rule.  An empty
 * histogram sets EQ_EF_EMPTY in d_err. */
eq_status eq_build_table(const uint64_t* hist, uint16_t* freq, uint32_t* d_err, eq_stream_t stream);

/* a5 for EQ_CODEC_PAIR (reading R15; one table per block): from the
 * block histogram hist (device uint64[256]) write the pair half of the table buffer,
 * table[256..512) (device uint16, the layout of EQ_CODEC_PAIR above): ranks = the 15 most
 * frequent present codes (ties: lower code); pair (ra, rb) kept iff 32·M·c_a·c_b ≥ T²; the R8
 * rule over [kept pairs in (ra, rb) order, escape = T² − Σ kept] to M = 4096; unused entries 0.
 * table[0..256) (the single table, eq_build_table) is not touched.  Block counts must stay
 * below 2^50 (always true within eq_encode_bounds' limits).  An empty histogram sets
 * EQ_EF_EMPTY in d_err.  Asynchronous; one CTA. */
eq_status eq_build_pair_table(const uint64_t* hist, uint16_t* table, uint32_t* d_err, eq_stream_t stream);

/* a6 (Alg. 1 l.4-5, R9/R10/R14): rANS-encode the concatenated symbol stream
 * `codes` of the block's layers (sizes rows*cols in block order, from `blk`), chunks of
 * blk->chunk_symbols restarting at each layer, into blk->payload / blk->chunk_off with
 * table blk->freq and renormalisation blk->codec (EQ_CODEC_*; else EQ_ERR_ARG).  chunk_sizes: device scratch uint32[n_chunks].  *payload_bytes_dev
 * (device uint64) receives the total.  A zero-frequency symbol sets EQ_EF_UNKNOWN_SYMBOL. */
eq_status eq_rans_encode(const uint8_t* codes, const eq_block* blk, uint32_t* chunk_sizes,
                         uint64_t* payload_bytes_dev, uint32_t* d_err, eq_stream_t stream);

/* ---------------------------------------------------------------- north-star calls */

/* Alg. 1 for one block: scales (per p->scale_mode; layers in p->exclude_mask
 * keep AbsMax scales), 8-bit quantisation in p->format, one
 * histogram + table over the concatenated stream, chunked rANS.  Fills out->payload,
 * chunk_off, n_chunks, chunk_symbols, freq, scales (device, caller-allocated per
 * eq_encode_bounds) and out->payload_bytes.  SYNCHRONOUS: waits for the stream to read
 * payload_bytes and the device error word.  scratch: device, ≥ *scratch_bytes of
 * eq_encode_bounds.  EQ_ERR_BUFFER if a capacity is too small. */
eq_status eq_quantize_encode(const eq_tensor* layers, uint32_t n_layers, const eq_params* p,
                             eq_block* out, void* scratch, uint64_t scratch_bytes,
                             eq_stream_t stream);

/* Alg. 2 l.1-2 + App. A.1 arena: decode every chunk of `n_blocks`
 * blocks in ONE launch (chunk-parallel, lane per chunk) and write each layer, row-major,
 * into `arena` at the offsets of eq_arena_layout (views, no copies).  EQ_OUT_BF16 fuses
 * the dequantiser out = RNE_bf16(s_row · value(code)) for the block's format (E4M3 or Int8);
 * EQ_OUT_FP8 writes the codes.  All blocks of one call must share one codec (EQ_ERR_ARG
 * otherwise).
 * Per-chunk integrity (final state == L of the codec, every byte consumed) and offset
 * bounds are checked on the device and reported in d_err (EQ_EF_CORRUPT / EQ_EF_TRUNCATED).
 * Asynchronous; EQ_ERR_BUFFER if arena_bytes is below the layout's total. */
eq_status eq_decode_dequant(const eq_block* blocks, uint32_t n_blocks, uint32_t out_dtype,
                            void* arena, uint64_t arena_bytes, uint32_t* d_err,
                            eq_stream_t stream);

/* Chunks the decoder of `codec` (EQ_CODEC_*) / `out_dtype` keeps in flight at once on CUDA
 * device `device` (SMs × resident CTAs per SM × chunks per CTA; one chunk per lane).  A
 * launch with n chunks runs ceil(n / lanes) rounds of one chunk-length serial chain each, so
 * callers choose chunk_symbols to keep n / lanes near a whole number of rounds.
 * Host only; EQ_ERR_ARG for bad enums. */
eq_status eq_decode_lanes(uint32_t codec, uint32_t out_dtype, int device, uint64_t* lanes);

/* End-to-end variant with HOST buffers: blocks_host[b].payload / chunk_off / freq / scales
 * are host pointers (pinned for full speed; arena_host too).  Copies them into `workspace`
 * (device, ≥ eq_decode_host_workspace_bytes), decodes, and copies the decoded arena to
 * arena_host, pipelined over ≤ 8 groups of blocks: the host→device copy of the next group
 * and the device→host copy of the previous one overlap the decode of the current one (two
 * copy streams created and destroyed inside the call, ordered after prior work on `stream`).
 * SYNCHRONOUS (returns after the last device→host copy, with eq_check). */
uint64_t eq_decode_host_workspace_bytes(const eq_block* blocks_host, uint32_t n_blocks,
                                        uint32_t out_dtype);
eq_status eq_decode_dequant_host(const eq_block* blocks_host, uint32_t n_blocks, uint32_t out_dtype,
                                 void* arena_host, uint64_t arena_bytes, void* workspace,
                                 uint64_t workspace_bytes, eq_stream_t stream);

/* Alg. 2 l.3 fused with l.1-2 (§8(f) NEXT row 1, config 4; all four codecs — the word
 * and pair codecs (R15, R18) run the warp-specialised kernel): Y_q = X_q · Ŵ_qᵀ for
 * n_jobs layers `layers[q]` of block `blk` in ONE launch, Ŵ = the layer's decoded +
 * dequantised bf16 weights (never written to memory): each chunk is decoded straight into
 * tcgen05 shared-memory tiles and multiplied on the 5th-gen tensor cores (bf16 × bf16 →
 * fp32 accumulate in TMEM); a row split over several chunks yields per-chunk partial sums
 * that a second kernel adds in chunk order (deterministic).
 * layers: HOST array [n_jobs] (1 ≤ n_jobs ≤ EQ_MAX_LAYERS) of layer indices;
 * x: HOST array of n_jobs DEVICE pointers, bf16 [batch, cols_q] row-major, 16-byte aligned;
 * y: HOST array of n_jobs DEVICE pointers, fp32 [batch, rows_q], 16-byte aligned, disjoint.
 * workspace: device, ≥ eq_qmatmul_workspace_bytes (0 when every row is one chunk), 16-byte
 * aligned; caller-owned, reused freely after the stream passes the call.
 * Requires row-independent chunks — EQ_CHUNK_ROW (R16: any cols that are a multiple of 64; a
 * ragged last chunk per row is fine) or EQ_CHUNK_LAYER with cols % chunk_symbols == 0 —
 * rows % 128 == 0, chunk_symbols % 64 == 0, 1 ≤ batch ≤ 256 (else EQ_ERR_SHAPE);
 * EQ_ERR_BUFFER for a short workspace.  Stream integrity checks as eq_decode_dequant (d_err).
 * Asynchronous. */
uint64_t eq_qmatmul_workspace_bytes(const eq_block* blk, uint32_t n_jobs, const uint32_t* layers,
                                    uint32_t batch);
eq_status eq_qmatmul_group(const eq_block* blk, uint32_t n_jobs, const uint32_t* layers,
                           const void* const* x, float* const* y, uint32_t batch, void* workspace,
                           uint64_t workspace_bytes, uint32_t* d_err, eq_stream_t stream);
/* Single-layer form of eq_qmatmul_group (x, y device pointers). */
eq_status eq_qmatmul(const eq_block* blk, uint32_t layer, const void* x, uint32_t batch, float* y,
                     void* workspace, uint64_t workspace_bytes, uint32_t* d_err, eq_stream_t stream);

/* §8(f) NEXT row 3 — the paper's solver for Eq. 4: per layer, L-BFGS over
 * the per-channel scales with straight-through gradients through Q_γ, from AbsMax.
 * Reading R13: variables u = log2 s, evaluated scales RNE_bf16(2^u), Armijo
 * backtracking on the true discrete objective (R4), two-loop recursion.
 * lr ≤ 0 selects the paper's rule (0.25 for λ > 30, else 1.0); a steepest-descent step moves
 * the largest log2-scale by lr, a quasi-Newton step starts at lr. */
typedef struct {
    uint32_t max_iters;       /* accepted steps per layer (default 100)                    */
    uint32_t history;         /* curvature pairs kept, 1..32 (default 10)                  */
    uint32_t trials;          /* backtracking step lengths evaluated per pass, 1..8 (4)    */
    uint32_t max_backtracks;  /* Armijo trials per iteration before failing (32)          */
    double lr;                /* initial step length; ≤ 0: P:507 rule                     */
    double c1;                /* Armijo constant (1e-4)                                    */
    double grad_tol;          /* stop when max |∂F/∂u| ≤ grad_tol (1e-7)                   */
    double change_tol;        /* stop when |ΔF| or max |Δu| < change_tol (1e-9)            */
} eq_lbfgs_params;

void eq_lbfgs_default_params(eq_lbfgs_params* p);
uint64_t eq_lbfgs_scratch_bytes(const eq_tensor* layers, uint32_t n_layers, const eq_lbfgs_params* p);
/* Optimise the scales of n_layers (≤ EQ_MAX_LAYERS) layers, each independently with its own
 * ‖W‖₁ and M·N (Eq. 4 per layer, "optimize each layer separately").  params may be
 * NULL (defaults).  Outputs (device, caller-owned): scales bf16 bits [Σ rows] in layer
 * order; trace (nullable) f64 [n_layers][max_iters+1] = objective after each accepted step
 * (entry 0 = AbsMax objective; unused entries NaN); info (nullable) u32 [n_layers][4] =
 * {accepted steps, converged, evaluation passes, done}.  Deterministic.  SYNCHRONOUS (polls
 * completion).  EQ_ERR_BUFFER if scratch_bytes < eq_lbfgs_scratch_bytes. */
eq_status eq_lbfgs_scales(const eq_tensor* layers, uint32_t n_layers, uint32_t format, double lambda,
                          const eq_lbfgs_params* params, uint16_t* scales, double* trace,
                          uint32_t* info, void* scratch, uint64_t scratch_bytes, eq_stream_t stream);
/* Eq. 4 of one layer at given bf16 scales (device [rows]) and its straight-through gradient
 * w.r.t. u = log2 s (SPEC ste_gradient): f_out (device, 1 double) = objective,
 * g_out (device, rows doubles).  Scratch as eq_lbfgs_scratch_bytes(layer, 1, NULL).
 * Asynchronous. */
eq_status eq_rd_eval(const eq_tensor* layer, uint32_t format, double lambda, const uint16_t* scales,
                     double* f_out, double* g_out, void* scratch, uint64_t scratch_bytes,
                     eq_stream_t stream);

/* SYNCHRONOUS: waits for `stream`, reads the device error word and maps its first set
 * bit to a status (EQ_OK when zero). */
eq_status eq_check(const uint32_t* d_err, eq_stream_t stream);

/* λ for a target rate (one global λ per target entropy; R11).  Estimates
 * the rate on every `row_stride`-th row of the given layers (all treated as one layer
 * set) as histogram entropy + per-parameter side information, over a log-spaced λ grid
 * refined twice.  SYNCHRONOUS.  scratch ≥ eq_calibrate_scratch_bytes.  Returns
 * EQ_ERR_UNREACHABLE_TARGET if the target lies outside the rates of λ ∈ [0, 1e6]. */
uint64_t eq_calibrate_scratch_bytes(const eq_tensor* layers, uint32_t n_layers, uint32_t row_stride);
eq_status eq_calibrate_lambda(const eq_tensor* layers, uint32_t n_layers, const eq_params* p,
                              double target_bits, uint32_t row_stride, double* lambda_out,
                              double* est_bits_out, void* scratch, uint64_t scratch_bytes,
                              eq_stream_t stream);

/* Optional CRC verify mode (CRC-32 over the uncompressed block
 * stream — the codes vec(W_q) of a block's layers in order).  CRC-32/IEEE: reflected polynomial
 * 0xEDB88320, initial value and final XOR 0xFFFFFFFF ("123456789" → 0xCBF43926).
 * data: device, n bytes (any alignment); crc: device, one uint32 (written, not read);
 * scratch: device, ≥ eq_crc32_scratch_bytes(n) (4 bytes per 4 KB piece), caller-owned.
 * Two launches (per-piece CRCs, then one CTA folds them with GF(2) zero-byte operators).
 * EQ_ERR_ARG for NULL pointers, EQ_ERR_BUFFER for short scratch.  Asynchronous.
 * After eq_quantize_encode returns, its scratch begins with the block's codes in layer order
 * (Σ rows·cols bytes): the stream whose CRC a container records at encode time; after a
 * decode to EQ_OUT_FP8 the same CRC over the decoded layers verifies the round trip. */
uint64_t eq_crc32_scratch_bytes(uint64_t n);
eq_status eq_crc32(const void* data, uint64_t n, uint32_t* crc, void* scratch, uint64_t scratch_bytes,
                   eq_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* ENTQUANT_H */
