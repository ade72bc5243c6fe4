// qmatmul.cu — §8(f) NEXT row 1 / config 4: QMatMul of Alg. 2 l.3 fused with the
// entropy decode and dequantisation of l.1-2: Y = X · Ŵᵀ for one layer of a compressed block,
// where Ŵ = RNE_bf16(s_row · value(code)) is never written to HBM.  The paper runs a Marlin
// FP8 GEMM (W8A16) on the buffer nvCOMP decoded into; here the decoded rows go
// straight into tcgen05 shared-memory operand tiles.
//
// One launch covers a GROUP of GEMMs of one block (e.g. all 7 linears, or q/k/v).  Chunks
// must be row-aligned (K % chunk_symbols == 0), so the chunks of a row are independent K
// slices: CTA = (GEMM, 128-row tile, chunk column j), 128 threads, lane r decodes chunk j of
// row r.  Every CTA does identical work (one chunk per lane) and a Llama-3-8B block at
// chunk 2048 gives 832 CTAs, one wave at 5-6 CTAs/SM.  Per 64-column K step:
//   1. each lane decodes + dequantises its next 64 symbols into registers (overlapping the
//      tensor cores' reads of the previous step), waits on the MMA mbarrier, and stores them
//      into the A tile (bf16, K-major, SWIZZLE_128B canonical UMMA layout: 8-row × 128 B
//      atoms, 16-byte chunk j of row r at chunk j ^ (r & 7));
//   2. the 128 threads stage X[:, k0:k0+64] (bf16, K-major, same layout) as the B tile;
//   3. fence.proxy.async, barrier; one thread issues 4 × tcgen05.mma.cta_group::1.kind::f16
//      (M=128, N=batch padded to 8, K=16 each) accumulating fp32 in TMEM, then
//      tcgen05.commit → mbarrier.
// Epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes 32w..32w+31 = rows) → fp32 partial
// [j][b][row] (or Y directly when a row is one chunk); k_qmm_reduce sums the partials in a
// fixed order (deterministic split-K).
#include "common.cuh"
// (EQ_WRING = 128, five segments in flight per decoder lane, measured: same time at batch 1, and
// at batch 64 the extra 8 KB per CTA leaves 2 CTAs/SM, 0.29 -> 0.45 ms; profiles/r2/s1qmm)
#include "decode_core.cuh"
#include "pair_core.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <type_traits>

#ifndef EQ_QMM_MIN_CTAS
#define EQ_QMM_MIN_CTAS 3
#endif

namespace eq {

constexpr int kTileRows = 128;                // MMA M = TMEM lanes
constexpr int kTiles = 2;                     // row tiles per CTA (share the LUT and the B tile)
constexpr int kQThreads = kTileRows * kTiles;
#ifndef EQ_QMM_K
#define EQ_QMM_K 64
#endif
constexpr int kQK = EQ_QMM_K;                 // K columns per step: 64 (SWIZZLE_128B rows) or 32 (SWIZZLE_64B)
constexpr int kRowB = kQK * 2;                // bytes per tile row = swizzle span
constexpr int kAtom = 8 * kRowB;              // 8-row swizzle atom (1024 or 512 bytes)
constexpr int kChunks = kRowB / 16;           // 16-byte chunks per row
constexpr int kATile = kTileRows * kRowB;     // 16 KB (or 8 KB) per row tile
static_assert(kQK == 64 || kQK == 32, "K step");
// 16-byte chunk c of row r of a K-major swizzled tile: 128B mode XORs c with r & 7, 64B mode
// with (r >> 1) & 3 (address bits [4,6) ^= bits [7,9))
__device__ __forceinline__ uint32_t swz(uint32_t r, uint32_t c) {
    return kQK == 64 ? (c ^ (r & 7)) : (c ^ ((r >> 1) & 3));
}

// one GEMM of the group: layer `layer` of the block, X [n_real][K] bf16, output fp32
struct QmmJob {
    const uint16_t* x;
    float* out;               // cpr == 1: Y [n_real][rows]; else partials [cpr][n_real][rows]
    const uint16_t* scales;   // the layer's first row
    uint32_t chunk0, rows, K, cpr, tile_begin;
};

struct QmmParams {
    QmmJob job[EQ_MAX_LAYERS];
    uint32_t n_jobs;
    const uint8_t* payload;
    const uint32_t* off;
    const uint16_t* freq;
    uint64_t payload_bytes;
    uint32_t* err;
    uint32_t format, cs, n_pad, n_real, idesc, tmem_cols, acc_cols;
    uint32_t k2p20, k2p12, kneg2p14, k4;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: start >> 4, LBO = 1 (unused for
// swizzled K-major), SBO = 1024 B (stride between 8-row atoms), version 1, layout type 2
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) |
           ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}
// K-major SWIZZLE_64B: SBO = 512 B between 8-row atoms, layout type 4
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(512u >> 4) << 32) |
           ((uint64_t)1u << 46) | ((uint64_t)4u << 61);
}
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    return kQK == 64 ? umma_desc_sw128(saddr) : umma_desc_sw64(saddr);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{ .reg .pred p; WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra WAIT_%=; }" ::"r"(bar),
        "r"(parity)
        : "memory");
}

template <class C>
__device__ __forceinline__ uint4 dequant8(const C& c, uint32_t q0, uint32_t q1) {
    if (c.i8)
        return make_uint4(dequant2_i8(q0, c.s), dequant2_i8(q0 >> 16, c.s), dequant2_i8(q1, c.s),
                          dequant2_i8(q1 >> 16, c.s));
    if (c.s16)
        return make_uint4(dequant2_h(q0, c.s16), dequant2_h(q0 >> 16, c.s16), dequant2_h(q1, c.s16),
                          dequant2_h(q1 >> 16, c.s16));
    return make_uint4(dequant2(q0, c.s), dequant2(q0 >> 16, c.s), dequant2(q1, c.s), dequant2(q1 >> 16, c.s));
}

// one lane's next 64 decoded + dequantised symbols, held in registers (8 × 16 bytes) so the
// decode of step t+1 overlaps the tensor-core reads of step t's tile
__device__ __forceinline__ void decode_step(Chain& c, const DecTable& T, const uint8_t* payload, uint4 v[kQK / 8]) {
    #pragma unroll
    for (int g = 0; g < kQK / 16; ++g) {                // kQK / 16 × 16 symbols
        const uint32_t q0 = decode4(c, T);
        const uint32_t q1 = decode4(c, T);
        stage_wait_all(); ring_issue(c.br, payload); stage_commit();
        const uint32_t q2 = decode4(c, T);
        const uint32_t q3 = decode4(c, T);
        stage_wait_all(); ring_issue(c.br, payload); stage_commit();
        v[2 * g] = dequant8(c, q0, q1);
        v[2 * g + 1] = dequant8(c, q2, q3);
    }
    c.i += kQK;
}

// EQ_CODEC_WORD: the same 64 symbols with word renormalisation (decode_one_w)
__device__ __forceinline__ void decode_step(ChainW& c, const DecTable& T, const uint8_t* payload, uint4 v[kQK / 8]) {
    #pragma unroll
    for (int g = 0; g < kQK / 16; ++g) {                // kQK / 16 × 16 symbols
        const uint32_t q0 = decode4_w(c, T);
        const uint32_t q1 = decode4_w(c, T);
        ring_step_w(c.r, payload);
        const uint32_t q2 = decode4_w(c, T);
        const uint32_t q3 = decode4_w(c, T);
        ring_step_w(c.r, payload);
        v[2 * g] = dequant8(c, q0, q1);
        v[2 * g + 1] = dequant8(c, q2, q3);
    }
    c.i += kQK;
}

__device__ __forceinline__ bool chunk_begin(ChainW& c, const QmmParams& P, uint32_t chunk, uint32_t ring, uint32_t len) {
    c.i = 0;
    c.n = len;
    c.runaway = false;
    const uint32_t a = __ldg(P.off + chunk), e = __ldg(P.off + chunk + 1);
    if (e < a || (uint64_t)e > P.payload_bytes || e - a < 4) {
        atomicOr(P.err, EQ_EF_TRUNCATED);
        c.active = false;
        return false;
    }
    c.active = true;
    c.a = a;
    c.e = e;
    c.r.ring = ring;
    const uint32_t g0 = a & ~15u;
    #pragma unroll
    for (uint32_t q = 0; q < kWRing / 16; ++q) stage_segment_w(ring, P.payload, g0 + 16 * q);
    c.r.gn = g0 + kWRing;
    stage_commit();
    stage_wait_all();
    const uint32_t m = kWRing - 1, A = a + kWBias;
    c.x = lds_u16(ring | (A & m)) | (lds_u16(ring | ((A + 2) & m)) << 16);
    c.r.w = lds_u16(ring | ((A + 4) & m));
    c.r.Q = A + 6;
    return true;
}

__device__ __forceinline__ void chunk_end(const ChainW& c, uint32_t* err) {
    if (c.active && (c.runaway || c.x != kLw || c.r.Q - (2u + kWBias) != c.e)) atomicOr(err, EQ_EF_CORRUPT);
}

// A corrupt stream can consume words past its chunk; checked before every 64-symbol step so
// the ring never stages beyond the payload's readable slack (≤ 128 bytes per step + 48 ahead)
__device__ __forceinline__ bool runaway_q(const ChainW& c) { return c.r.Q > c.e + (2u + kWBias); }
__device__ __forceinline__ bool runaway_q(const Chain& c) { return c.br.wi4 > c.wlimit4; }

// start decoding chunk `chunk` (payload bytes, ring staging, first state) for this lane
__device__ __forceinline__ bool chunk_begin(Chain& c, const QmmParams& P, uint32_t chunk, uint32_t ring, uint32_t len) {
    c.i = 0;
    c.n = len;
    c.runaway = false;
    const uint32_t a = __ldg(P.off + chunk), e = __ldg(P.off + chunk + 1);
    if (e < a || (uint64_t)e > P.payload_bytes || e - a < 4) {
        atomicOr(P.err, EQ_EF_TRUNCATED);
        c.active = false;
        return false;
    }
    c.active = true;
    c.a = a;
    c.e = e;
    c.wlimit4 = ((e >> 2) + 16) * 4u;
    c.br.ring = ring;
    const uint32_t s0 = a >> 4;
    #pragma unroll
    for (int q = 0; q < 4; ++q) stage_segment(ring, P.payload, s0 + q);
    c.br.gs = s0 + 4;
    stage_commit();
    stage_wait_all();
    const uint32_t wa = a >> 2;
    const uint32_t h = bswap32(lds_u32(ring | ((wa * 4u) & 0x3Cu)));
    const uint32_t m = bswap32(lds_u32(ring | (((wa + 1) * 4u) & 0x3Cu)));
    const uint32_t sh = (a & 3) * 8;
    c.x = bswap32(__funnelshift_lc(m, h, sh));
    c.br.hi = m << sh;
    c.br.lo = 0;
    c.br.nb = 32 - (int)sh;
    c.br.wi4 = (wa + 2) * 4u;
    c.br.refill();
    return true;
}

__device__ __forceinline__ void chunk_end(const Chain& c, uint32_t* err) {
    if (!c.active) return;
    const int64_t inserted = 8ll * (int64_t)(c.br.wi4 - (c.a >> 2) * 4u) - 8ll * (int64_t)(c.a & 3);
    const int64_t consumed = inserted - c.br.nb;
    if (c.runaway || c.br.wi4 > c.wlimit4 || c.x != kL || consumed != 8ll * (int64_t)(c.e - c.a))
        atomicOr(err, EQ_EF_CORRUPT);
}

// CTA = (job, pair of 128-row tiles, chunk column j): lane r of half h decodes the j-th
// chunk of row 128·(2p+h)+r — cs columns [j·cs, (j+1)·cs) — and each half accumulates that
// K-slice of its 128 × batch output in its own TMEM columns.  Every CTA does the same work
// (one chunk per lane), so one grouped launch over all GEMMs of a block fills the GPU evenly.
static_assert(EQ_WENTRY == 1 && EQ_ZFAST == 0, "k_qmatmul builds the LUT in the (f−1)-on-top entry layout");
template <bool WORD>
__global__ void __launch_bounds__(kQThreads, EQ_QMM_MIN_CTAS) k_qmatmul(const __grid_constant__ QmmParams P) {
    extern __shared__ __align__(1024) uint8_t dsm_raw[];
    // SWIZZLE_128B atoms are addressed by absolute shared-address bits: align the carve-out
    uint8_t* dsm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
    // layout: [A tiles 2 × 16 KB | B tile | LUT 16 KB | rings | wsum | bar | tmem slot]; the
    // symbol prefix sums used while building the LUT live in the (not yet used) A tiles
    uint8_t* a_tiles = dsm;
    uint8_t* b_tile = dsm + kTiles * kATile;
    const uint32_t b_tile_bytes = (P.n_pad * (uint32_t)kRowB + 1023u) & ~1023u;
    uint32_t* lut = reinterpret_cast<uint32_t*>(b_tile + b_tile_bytes);
    uint32_t* rings = lut + kM;                                      // 256 × 64 B
    uint32_t* wsum = rings + kQThreads * kRingWords;                 // 8
    uint64_t* bars = reinterpret_cast<uint64_t*>(wsum + 8);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 1);
    uint32_t* cum = reinterpret_cast<uint32_t*>(a_tiles);            // 257 words

    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const uint32_t h = (uint32_t)t / kTileRows, r = (uint32_t)t % kTileRows;

    // ---- which GEMM, row tiles and chunk column
    uint32_t jb = 0;
    for (uint32_t q = 1; q < P.n_jobs; ++q)
        if (blockIdx.x >= P.job[q].tile_begin) jb = q;
    const QmmJob& J = P.job[jb];
    const uint32_t local = blockIdx.x - J.tile_begin;
    const uint32_t pair = local / J.cpr, jcol = local - pair * J.cpr;
    const uint32_t n_tiles = J.rows / kTileRows;
    const bool my_on = kTiles * pair + h < n_tiles;                 // this half's tile exists

    // ---- TMEM accumulators (warp 0), mbarrier (thread 0)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(P.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        mbar_init(smem_u32(&bars[0]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // ---- block LUT (as in k_decode)
    {
        uint32_t v = P.freq[t];                      // 256 threads = 256 symbols
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
            if (lane >= d) v += o;
        }
        if (lane == 31) wsum[warp] = v;
        __syncthreads();
        uint32_t add = 0;
        for (int q = 0; q < warp; ++q) add += wsum[q];
        cum[t + 1] = v + add;
        if (t == 0) cum[0] = 0;
    }
    __syncthreads();
    const bool table_ok = cum[256] == kM;
    if (table_ok) {
        for (int slot = t; slot < (int)kM; slot += kQThreads) {
            int lo = 0, hi = 255;
            while (lo < hi) {
                int mid = (lo + hi + 1) >> 1;
                if (cum[mid] <= (uint32_t)slot) lo = mid; else hi = mid - 1;
            }
            uint32_t fs = cum[lo + 1] - cum[lo];
            // decode_one_w and decode_one both read the (f−1)-on-top layout
            lut[slot] = (uint32_t)lo | (((uint32_t)slot - cum[lo]) << 8) | ((fs - 1) << 20);
        }
    } else if (t == 0) {
        atomicOr(P.err, EQ_EF_CORRUPT);
    }
    __syncthreads();
    const uint32_t tmem = *tmem_slot;
    DecTable T;
    T.k2p20 = P.k2p20;
    T.k2p12 = P.k2p12;
    T.kneg2p14 = P.kneg2p14;
    T.k4 = P.k4;
    T.lut_s = smem_u32(lut);
    T.f0 = cum[1];
    T.ez = (T.f0 - 1) << 8;
    __syncthreads();                                 // cum (in the A tiles) read by everyone

    // ---- this lane's row and chunk
    const uint32_t kbase = jcol * P.cs;
    const uint32_t clen = min(P.cs, J.K - kbase);    // the last chunk of a row may be shorter (EQ_CHUNK_ROW)
    const uint32_t steps = clen / kQK;
    const uint32_t grow = (kTiles * pair + h) * kTileRows + r;
    const uint32_t ring = smem_u32(rings + t * kRingWords);
    typename std::conditional<WORD, ChainW, Chain>::type c;
    c.sc = J.scales;
    c.i8 = P.format == EQ_FMT_INT8;
    c.active = false;
    c.runaway = false;
    c.s = 0.f;
    c.s16 = 0;
    if (my_on) {
        c.s = bf16_bits_to_float(J.scales[grow]);
        c.s16 = c.i8 ? 0 : scale_f16(c.s);
        if (table_ok) chunk_begin(c, P, J.chunk0 + grow * J.cpr + jcol, ring, clen);
    }
    uint8_t* a_tile = a_tiles + h * kATile;
    uint8_t* arow = a_tile + (r >> 3) * kAtom + (r & 7) * kRowB;
    const uint32_t bar = smem_u32(&bars[0]);

    for (uint32_t st = 0; st < steps; ++st) {
        uint4 v[kQK / 8];
        if (c.active && !runaway_q(c)) {
            decode_step(c, T, P.payload, v);
        } else {
            c.runaway = c.runaway || c.active;           // stop reading a stream that overran its chunk
            #pragma unroll
            for (int q = 0; q < kQK / 8; ++q) v[q] = make_uint4(0, 0, 0, 0);
        }
        if (st > 0) mbar_wait(bar, (st - 1) & 1);     // tensor cores done reading step st-1
        #pragma unroll
        for (int q = 0; q < kQK / 8; ++q) *reinterpret_cast<uint4*>(arow + (swz(r, q) << 4)) = v[q];
        // activations X[:, k0:k0+kQK] -> B tile (rows = batch, zero-padded)
        const uint32_t k0 = kbase + st * kQK;
        for (uint32_t piece = t; piece < P.n_pad * kChunks; piece += kQThreads) {
            const uint32_t b = piece / kChunks, j = piece % kChunks;
            uint4 xv = make_uint4(0, 0, 0, 0);
            if (b < P.n_real) xv = __ldg(reinterpret_cast<const uint4*>(J.x + (uint64_t)b * J.K + k0) + j);
            *reinterpret_cast<uint4*>(b_tile + (b >> 3) * kAtom + (b & 7) * kRowB + (swz(b, j) << 4)) = xv;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (t == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t db = umma_desc(smem_u32(b_tile));
            #pragma unroll
            for (int hh = 0; hh < kTiles; ++hh) {
                if (kTiles * pair + hh >= n_tiles) continue;
                const uint64_t da = umma_desc(smem_u32(a_tiles + hh * kATile));
                #pragma unroll
                for (int kk = 0; kk < kQK / 16; ++kk) {
                    const uint32_t acc = (st > 0 || kk > 0) ? 1u : 0u;
                    // +32 bytes per K=16 slice inside the swizzle atom (start address in 16 B units)
                    asm volatile(
                        "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(
                            tmem + hh * P.acc_cols),
                        "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(P.idesc), "r"(acc));
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                         : "memory");
        }
    }
    chunk_end(c, P.err);
    stage_wait_all();
    // ---- wait for the last MMAs, read the accumulators
    mbar_wait(bar, (steps - 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    float* out = J.out + (uint64_t)jcol * P.n_real * J.rows;
    for (uint32_t col = 0; col < P.n_pad; col += 8) {
        uint32_t v[8];
        // warp w reads TMEM lanes 32·(w % 4) .. +31 (= rows r of its half) of half h's columns
        const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + h * P.acc_cols + col;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (my_on) {
            #pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t b = col + q;
                if (b < P.n_real) out[(uint64_t)b * J.rows + grow] = __uint_as_float(v[q]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols));
}

// ================================================================ warp-specialised kernel
// k_qmm_ws — EQ_CODEC_WORD / EQ_CODEC_PAIR blocks (the bench's codec), row-chunked streams.
// CTA = (GEMM, NTILE 128-row tiles, chunk column j), 32·(4·NTILE + 1) threads (NTILE = 2: 288):
//   warps 0 .. 4·NTILE−1  decoders (4 per tile, one copy of the tables for all): lane r decodes
//              chunk j of its row (its rANS chain), dequantises with the row scale and writes 32
//              columns per K step (64 B, bf16) into its tile's sub-tile of A stage s of a
//              kWsStages-deep ring (K-major, SWIZZLE_64B canonical UMMA layout), then
//              fence.proxy.async + one mbarrier arrive per warp on full[s];
//   warp 4·NTILE  producer + MMA issuer (one elected lane): TMA-loads X[:, k0 : k0 + 32] as the B
//              stage (the tensor map's SWIZZLE_64B box lands in the UMMA layout; rows past the
//              batch are zero-filled), waits full[s], issues per tile 2 × tcgen05.mma (M = 128,
//              N = batch rounded up to 16, K = 16) into that tile's TMEM accumulator (columns
//              h·N) and commits to empty[s], which frees both stages for step + kWsStages.
// The decoders never wait for the tensor cores unless they run kWsStages steps ahead; no
// CTA-wide barrier inside the K loop.  Epilogue: decoder warp w reads TMEM lanes 32·(w % 4) of
// accumulator w / 4 (tcgen05.ld 32x32b) and writes Y (one chunk column) or the split-K partial.
#ifndef EQ_QMM_NTILE
#define EQ_QMM_NTILE 2                         // 128-row tiles (4 decoder warps each) per CTA
#endif
#ifndef EQ_QMM_WS_STAGES
#define EQ_QMM_WS_STAGES (EQ_QMM_NTILE > 1 ? 2 : 3)   // (2 vs 3 stages measured equal; 2 keeps 3 CTAs/SM at NTILE 2)
#endif
#ifndef EQ_QMM_WS_MIN_CTAS
#define EQ_QMM_WS_MIN_CTAS 3
#endif
#ifndef EQ_QMM_VALS
#define EQ_QMM_VALS 1                          // R18: decode into bf16x2 values (one HFMA2 per pair)
#endif
#ifndef EQ_QMM_HALF
#define EQ_QMM_HALF 1                          // decoder K step as a loop over two 16-symbol halves
#endif
#ifndef EQ_QMM_NARROW
#define EQ_QMM_NARROW 1                        // pair codec: 2·id LUT entries when every kept pair has f ≤ 2048
#endif
constexpr int kQmmNTile = EQ_QMM_NTILE;
constexpr int kWsStages = EQ_QMM_WS_STAGES;   // the default; a launch that would lose its one-wave
                                              // fit at kWsStages CTAs/SM may take 1 stage (below)
constexpr int kWsK = 32;                       // K columns per step (one SWIZZLE_64B row = 64 B)
constexpr int kWsRowB = kWsK * 2;
constexpr int kWsATile = kTileRows * kWsRowB;  // 8 KB per A stage
constexpr int kWsDec = 128;                   // decoder lanes (rows) per 128-row tile

struct QmmWsParams {
    CUtensorMap tmap[EQ_MAX_LAYERS];           // X of each job: [batch, K] bf16, box {32, n_pad}, SWIZZLE_64B
    QmmJob job[EQ_MAX_LAYERS];
    uint32_t n_jobs;
    const uint8_t* payload;
    const uint32_t* off;
    const uint16_t* freq;
    uint64_t payload_bytes;
    uint32_t* err;
    uint32_t format, cs, n_pad, n_real, idesc, tmem_cols, b_stage_bytes;
    uint32_t k2p20, k2p12, kneg2p14, k4;
};

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.release.cta.shared::cta.b64 st, [%0]; }" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("{ .reg .b64 st; mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1; }" ::"r"(bar),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

// the 8 codes -> 8 bf16 (16 bytes) of one lane, with the lane's row scale
template <class C>
__device__ __forceinline__ uint4 ws_dequant8(const C& c, uint32_t q0, uint32_t q1) {
    return dequant8(c, q0, q1);
}

// NTILE = 128-row tiles per CTA: 4·NTILE decoder warps (one row per lane) share one copy of the
// tables and one X stage; NTILE A sub-tiles per stage feed NTILE TMEM accumulators (columns
// h·n_pad).  NTILE = 2 holds twice the chains per CTA for the same table memory.
template <int CODEC, int NTILE, int STAGES>
__global__ void __launch_bounds__(32 * (4 * NTILE + 1), EQ_QMM_WS_MIN_CTAS) k_qmm_ws(const __grid_constant__ QmmWsParams P) {
    constexpr int kDec = kWsDec * NTILE;           // decoder lanes
    constexpr uint32_t kAStage = NTILE * kWsATile;
    extern __shared__ __align__(1024) uint8_t ws_raw[];
    uint8_t* dsm = ws_raw + ((1024u - (smem_u32(ws_raw) & 1023u)) & 1023u);
    // layout: [A stages (NTILE sub-tiles each) | B stages | tables | rings | barriers | tmem slot]
    uint8_t* a_st = dsm;
    uint8_t* b_st = dsm + STAGES * kAStage;
    uint8_t* tabs = b_st + STAGES * P.b_stage_bytes;
    constexpr bool kPairC = is_pair_codec(CODEC);
    constexpr bool kVals = CODEC == EQ_CODEC_PAIR_G && EQ_QMM_VALS;    // R18: bf16x2 value table
    constexpr uint32_t kTabBytes = kPairC ? kPairSmemBytes + (kVals ? 4u * kPairValWords : 0u) : (kM + 260) * 4u;
    uint32_t* rings = reinterpret_cast<uint32_t*>(tabs + ((kTabBytes + 127u) & ~127u));
    uint64_t* bars = reinterpret_cast<uint64_t*>(rings + kDec * (kWRing / 4));     // full[S], empty[S]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES);

    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    uint32_t jb = 0;
    for (uint32_t q = 1; q < P.n_jobs; ++q)
        if (blockIdx.x >= P.job[q].tile_begin) jb = q;
    const QmmJob& J = P.job[jb];
    const uint32_t local = blockIdx.x - J.tile_begin;
    const uint32_t tile = local / J.cpr, jcol = local - tile * J.cpr;
    const uint32_t kbase = jcol * P.cs;
    const uint32_t clen = min(P.cs, J.K - kbase);
    const uint32_t steps = clen / kWsK;
    const uint32_t grow = tile * (NTILE * kTileRows) + (uint32_t)t;  // decoder lanes only

    // ---- the decoder lanes start staging their chunk while the tables are built
    ChainW c;
    c.active = false;
    c.runaway = false;
    c.i8 = P.format == EQ_FMT_INT8;
    c.s = 0.f;
    c.s16 = 0;
    const uint32_t ring = smem_u32(rings + t * (kWRing / 4));
    uint32_t s2row = 0;
    if (t < kDec && grow < J.rows) {
        s2row = (uint32_t)J.scales[grow] * 0x10001u;
        c.s = bf16_bits_to_float(J.scales[grow]);
        c.s16 = c.i8 ? 0 : scale_f16(c.s);
        const uint32_t chunk = J.chunk0 + grow * J.cpr + jcol;
        const uint32_t a = __ldg(P.off + chunk), e = __ldg(P.off + chunk + 1);
        if (e < a || (uint64_t)e > P.payload_bytes || e - a < 4) {
            atomicOr(P.err, EQ_EF_TRUNCATED);
        } else {
            c.active = true;
            c.a = a;
            c.e = e;
            c.i = 0;
            c.n = clen;
            c.r.ring = ring;
            const uint32_t g0 = a & ~15u;
            #pragma unroll
            for (uint32_t q = 0; q < kWRing / 16; ++q) stage_segment_w(ring, P.payload, g0 + 16 * q);
            c.r.gn = g0 + kWRing;
        }
    }
    stage_commit();
    // ---- tables (all 160 threads reach the barriers; the 128 decoder threads work)
    PairTab PT{};
    DecTable WT{};
    bool ok;
    uint32_t mode = 1;                             // pair codec: 2 = narrow LUT entries (2·id)
    if constexpr (kPairC) {
        uint32_t* lut = reinterpret_cast<uint32_t*>(tabs);
        uint8_t* lut1 = tabs + kPairLutWords * 4;
        uint16_t* cum = reinterpret_cast<uint16_t*>(lut1 + kM);
        uint32_t cesc = 0;
        mode = pair_tables_build<kDec, false, EQ_QMM_NARROW, kVals, kVals>(P.freq, lut, lut1, cum, cesc, P.err,
                                                                          P.format == EQ_FMT_INT8);
        ok = mode != 0;
        __syncthreads();                           // table stores visible to every decoder lane
        if (ok) PT = pair_tab(P.freq, lut, lut1, cum, cesc, P.k2p20, P.k2p12);
    } else {
        uint32_t* lut = reinterpret_cast<uint32_t*>(tabs);
        uint32_t* cum = lut + kM;
        if (t < 32) {                              // exclusive prefix of the 256 frequencies
            uint32_t v[8], sum = 0;
            #pragma unroll
            for (int j = 0; j < 8; ++j) { v[j] = P.freq[t * 8 + j]; sum += v[j]; }
            uint32_t inc = sum;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                if (t >= d) inc += o;
            }
            uint32_t run = inc - sum;
            #pragma unroll
            for (int j = 0; j < 8; ++j) { cum[t * 8 + j] = run; run += v[j]; }
            if (t == 31) cum[256] = inc;
        }
        __syncthreads();
        ok = cum[256] == kM;
        if (ok && t < kDec) {
            lut_walk<256, kDec>(lut, cum, [&](uint32_t slot, int sym) -> uint32_t {
                const uint32_t fs = cum[sym + 1] - cum[sym];
                return (uint32_t)sym | ((slot - cum[sym]) << 8) | ((fs - 1) << 20);   // (f−1)-on-top layout
            });
        } else if (!ok && t == 0) {
            atomicOr(P.err, EQ_EF_CORRUPT);
        }
        __syncthreads();
        WT.k2p20 = P.k2p20;
        WT.k2p12 = P.k2p12;
        WT.kneg2p14 = P.kneg2p14;
        WT.k4 = P.k4;
        WT.lut_s = smem_u32(lut);
    }
    if (!ok) {                                     // nothing decodable: the whole CTA leaves together
        stage_wait_all();
        return;
    }
    // ---- barriers (first thread of the MMA warp), TMEM accumulators (the MMA warp)
    constexpr int kMmaWarp = 4 * NTILE;
    if (t == kDec) {
        for (int q = 0; q < STAGES; ++q) {
            mbar_init(smem_u32(&bars[q]), 4 * NTILE + 1);         // the decoder warps + the TMA arrive
            mbar_init(smem_u32(&bars[STAGES + q]), 1);         // tcgen05.commit
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(P.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == kMmaWarp) {
        // ===== producer (TMA of X) + MMA issuer: one lane
        if (lane == 0) {
            const CUtensorMap* map = &P.tmap[jb];
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
            const uint32_t pre = steps < (uint32_t)STAGES ? steps : (uint32_t)STAGES;
            for (uint32_t q = 0; q < pre; ++q) {
                const uint32_t fb = smem_u32(&bars[q]);
                mbar_arrive_tx(fb, P.b_stage_bytes);
                tma_load_2d(smem_u32(b_st + q * P.b_stage_bytes), map, (int32_t)(kbase + q * kWsK), 0, fb);
            }
            for (uint32_t st = 0; st < steps; ++st) {
                const uint32_t sidx = st % STAGES, use = st / STAGES;
                mbar_wait(smem_u32(&bars[sidx]), use & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint64_t db = umma_desc_sw64(smem_u32(b_st + sidx * P.b_stage_bytes));
                #pragma unroll
                for (int h = 0; h < NTILE; ++h) {
                    const uint64_t da = umma_desc_sw64(smem_u32(a_st + sidx * kAStage + h * kWsATile));
                    #pragma unroll
                    for (int kk = 0; kk < kWsK / 16; ++kk) {
                        const uint32_t acc = (st > 0 || kk > 0) ? 1u : 0u;
                        asm volatile(
                            "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(
                                tmem + (uint32_t)h * P.n_pad),
                            "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(P.idesc), "r"(acc));
                    }
                }
                const uint32_t eb = smem_u32(&bars[STAGES + sidx]);
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(eb)
                             : "memory");
                if (st + STAGES < steps) {      // refill the B stage once the MMAs that read it are done
                    mbar_wait(eb, use & 1);
                    const uint32_t fb = smem_u32(&bars[sidx]);
                    mbar_arrive_tx(fb, P.b_stage_bytes);
                    tma_load_2d(smem_u32(b_st + sidx * P.b_stage_bytes), map,
                                (int32_t)(kbase + (st + STAGES) * kWsK), 0, fb);
                }
            }
        }
        __syncwarp();
    } else {
        // ===== decoders: lane r = row r of the tile
        stage_wait_all();
        if (c.active) {
            const uint32_t m = kWRing - 1, A = c.a + kWBias;
            c.x = lds_u16(ring | (A & m)) | (lds_u16(ring | ((A + 2) & m)) << 16);
            c.r.w = lds_u16(ring | ((A + 4) & m));
            c.r.Q = A + 6;
        }
        const uint32_t r = (uint32_t)t & (kTileRows - 1);          // row within the lane's 128-row sub-tile
        const uint32_t row_off = (r >> 3) * 512u + (r & 7) * (uint32_t)kWsRowB;
        const uint32_t sw = (r >> 1) & 3;                         // SWIZZLE_64B: 16-byte chunk q at q ^ sw
        const uint32_t qlim = c.e + (2u + kWBias);
        const uint32_t a0 = smem_u32(a_st) + ((uint32_t)t / kTileRows) * kWsATile + row_off;
        // one K step = 32 symbols of the lane's chain into 4 × 16 bytes of its A row; branches
        // once per step (live chain, scale mode), stage index / phase by counters
        auto run = [&](auto narrow_c) {
            constexpr bool NARROW = decltype(narrow_c)::value;
            static_assert(kPairC || !NARROW, "narrow entries are a pair-codec layout");
            const uint32_t s16 = c.i8 ? 0u : (uint32_t)c.s16;
            [[maybe_unused]] const uint32_t s2 = kVals ? s2row : 0u;   // the row's bf16 scale, twice (R18 values)
            uint32_t sidx = 0, use = 0;
            for (uint32_t st = 0; st < steps; ++st) {
                if (st >= (uint32_t)STAGES) mbar_wait(smem_u32(&bars[STAGES + sidx]), (use & 1) ^ 1);
                const uint32_t arow = a0 + sidx * kAStage;
#if EQ_QMM_HALF
                // the step as a (not unrolled) loop over two halves of 16 symbols: half the code
                // of the fully unrolled step (the decoder loop then fits the instruction cache)
                if (c.active && !c.runaway) {
                    [[maybe_unused]] const uint16_t h16 = (uint16_t)s16;
                    #pragma unroll 1
                    for (uint32_t hs = 0; hs < 2; ++hs) {
                        [[maybe_unused]] uint32_t q[4];
                        if constexpr (kVals) {
                            // R18 with values: the half's 8 pairs as bf16x2 words, one HFMA2 each
                            uint32_t v[8];
                            bool esc = false;
                            #pragma unroll
                            for (int u = 0; u < 8; ++u) v[u] = decode_pair_g<NARROW, true, NARROW>(c.x, c.r, PT, esc);
                            ring_step_w(c.r, P.payload);
                            if (esc) patch_escapes_vals(v, c.x, c.r, PT, P.payload, c.i8);
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(arow + (((2 * hs) ^ sw) << 4)),
                                         "r"(mul_bf16x2(v[0], s2)), "r"(mul_bf16x2(v[1], s2)), "r"(mul_bf16x2(v[2], s2)),
                                         "r"(mul_bf16x2(v[3], s2)) : "memory");
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(arow + (((2 * hs + 1) ^ sw) << 4)),
                                         "r"(mul_bf16x2(v[4], s2)), "r"(mul_bf16x2(v[5], s2)), "r"(mul_bf16x2(v[6], s2)),
                                         "r"(mul_bf16x2(v[7], s2)) : "memory");
                        } else if constexpr (CODEC == EQ_CODEC_PAIR_G) {
                            // R18: the half is one 16-symbol group — 8 pair steps without an
                            // escape branch, then its escaped pairs' codes
                            bool esc = false;
                            #pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const uint32_t p0 = decode_pair_g<NARROW>(c.x, c.r, PT, esc);
                                const uint32_t p1 = decode_pair_g<NARROW>(c.x, c.r, PT, esc);
                                q[u] = __byte_perm(p0, p1, 0x5410);
                            }
                            ring_step_w(c.r, P.payload);
                            if (esc) patch_escapes(q, 8, c.x, c.r, PT, P.payload);
                        } else if constexpr (CODEC == EQ_CODEC_PAIR) {
                            #pragma unroll
                            for (int u = 0; u < 2; ++u) {
                                const uint32_t p0 = decode_pair<NARROW>(c.x, c.r, PT, P.payload);
                                const uint32_t p1 = decode_pair<NARROW>(c.x, c.r, PT, P.payload);
                                const uint32_t p2 = decode_pair<NARROW>(c.x, c.r, PT, P.payload);
                                const uint32_t p3 = decode_pair<NARROW>(c.x, c.r, PT, P.payload);
                                q[2 * u] = __byte_perm(p0, p1, 0x5410);
                                q[2 * u + 1] = __byte_perm(p2, p3, 0x5410);
                            }
                            ring_step_w(c.r, P.payload);              // one stage per 8 pair steps
                        } else {
                            q[0] = decode4_w(c, WT);
                            q[1] = decode4_w(c, WT);
                            ring_step_w(c.r, P.payload);
                            q[2] = decode4_w(c, WT);
                            q[3] = decode4_w(c, WT);
                            ring_step_w(c.r, P.payload);
                        }
                        if constexpr (!kVals) {
                        uint4 v0, v1;
                        if (s16) {
                            v0 = make_uint4(dequant2_h(q[0], h16), dequant2_h(q[0] >> 16, h16), dequant2_h(q[1], h16),
                                            dequant2_h(q[1] >> 16, h16));
                            v1 = make_uint4(dequant2_h(q[2], h16), dequant2_h(q[2] >> 16, h16), dequant2_h(q[3], h16),
                                            dequant2_h(q[3] >> 16, h16));
                        } else {
                            v0 = dequant8(c, q[0], q[1]);
                            v1 = dequant8(c, q[2], q[3]);
                        }
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(arow + (((2 * hs) ^ sw) << 4)),
                                     "r"(v0.x), "r"(v0.y), "r"(v0.z), "r"(v0.w) : "memory");
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(arow + (((2 * hs + 1) ^ sw) << 4)),
                                     "r"(v1.x), "r"(v1.y), "r"(v1.z), "r"(v1.w) : "memory");
                        }
                    }
                    c.i += kWsK;
                    if (c.r.Q > qlim) c.runaway = true;           // overran its chunk: stop reading
                } else {
                    #pragma unroll
                    for (uint32_t g = 0; g < kWsK / 8; ++g)
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(arow + ((g ^ sw) << 4)), "r"(0u),
                                     "r"(0u), "r"(0u), "r"(0u) : "memory");
                }
#else
                static_assert(CODEC != EQ_CODEC_PAIR_G, "R18 groups are the K step's 16-symbol halves (EQ_QMM_HALF)");
                uint4 v[kWsK / 8];
                if (c.active && !c.runaway) {
                    uint32_t q[kWsK / 4];
                    #pragma unroll
                    for (uint32_t g = 0; g < kWsK / 8; ++g) {
                        if constexpr (CODEC == EQ_CODEC_PAIR) {
                            const uint32_t p0 = decode_pair<NARROW>(c.x, c.r, PT, P.payload);
                            const uint32_t p1 = decode_pair<NARROW>(c.x, c.r, PT, P.payload);
                            const uint32_t p2 = decode_pair<NARROW>(c.x, c.r, PT, P.payload);
                            const uint32_t p3 = decode_pair<NARROW>(c.x, c.r, PT, P.payload);
                            q[2 * g] = __byte_perm(p0, p1, 0x5410);
                            q[2 * g + 1] = __byte_perm(p2, p3, 0x5410);
                            if (g & 1) ring_step_w(c.r, P.payload);   // one stage per 8 pair steps
                        } else {
                            q[2 * g] = decode4_w(c, WT);
                            q[2 * g + 1] = decode4_w(c, WT);
                            ring_step_w(c.r, P.payload);              // one stage per 8 steps
                        }
                    }
                    if (s16) {
                        const uint16_t h = (uint16_t)s16;
                        #pragma unroll
                        for (uint32_t g = 0; g < kWsK / 8; ++g)
                            v[g] = make_uint4(dequant2_h(q[2 * g], h), dequant2_h(q[2 * g] >> 16, h),
                                              dequant2_h(q[2 * g + 1], h), dequant2_h(q[2 * g + 1] >> 16, h));
                    } else {
                        #pragma unroll
                        for (uint32_t g = 0; g < kWsK / 8; ++g) v[g] = dequant8(c, q[2 * g], q[2 * g + 1]);
                    }
                    c.i += kWsK;
                    if (c.r.Q > qlim) c.runaway = true;           // overran its chunk: stop reading
                } else {
                    #pragma unroll
                    for (uint32_t g = 0; g < kWsK / 8; ++g) v[g] = make_uint4(0, 0, 0, 0);
                }
                #pragma unroll
                for (uint32_t g = 0; g < kWsK / 8; ++g)
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(arow + ((g ^ sw) << 4)), "r"(v[g].x),
                                 "r"(v[g].y), "r"(v[g].z), "r"(v[g].w)
                                 : "memory");
#endif
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&bars[sidx]));
                if (++sidx == (uint32_t)STAGES) { sidx = 0; ++use; }
            }
        };
        if constexpr (kPairC && EQ_QMM_NARROW) {
            if (mode == 2) run(std::true_type{});                 // CTA-uniform
            else run(std::false_type{});
        } else {
            run(std::false_type{});
        }
        stage_wait_all();
        if (c.active && (c.runaway || c.x != kLw || c.r.Q - (2u + kWBias) != c.e)) atomicOr(P.err, EQ_EF_CORRUPT);
        // ---- epilogue: the last commit covers every MMA of this CTA
        const uint32_t last = steps - 1;
        mbar_wait(smem_u32(&bars[STAGES + last % STAGES]), (last / STAGES) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        float* out = J.out + (uint64_t)jcol * P.n_real * J.rows;
        for (uint32_t col = 0; col < P.n_pad; col += 8) {
            uint32_t v[8];
            const uint32_t taddr = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(warp >> 2) * P.n_pad + col;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                         : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            #pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t b = col + q;
                if (b < P.n_real && grow < J.rows) out[(uint64_t)b * J.rows + grow] = __uint_as_float(v[q]);
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == kMmaWarp) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols));
}

// Y = Σ_j partial_j in a fixed order (j = 0, 1, …): deterministic split-K reduction
struct RedJob {
    const float* part;
    float* y;
    uint32_t n, cpr;          // n = batch · rows (multiple of 4)
};
struct RedParams {
    RedJob job[EQ_MAX_LAYERS];
};

__global__ void __launch_bounds__(256) k_qmm_reduce(const __grid_constant__ RedParams R) {
    const RedJob& J = R.job[blockIdx.y];
    const uint32_t n4 = J.n >> 2;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
        float4 a = __ldcs(reinterpret_cast<const float4*>(J.part) + i);
        for (uint32_t j = 1; j < J.cpr; ++j) {
            const float4 b = __ldcs(reinterpret_cast<const float4*>(J.part + (uint64_t)j * J.n) + i);
            a.x += b.x;
            a.y += b.y;
            a.z += b.z;
            a.w += b.w;
        }
        reinterpret_cast<float4*>(J.y)[i] = a;
    }
}

struct QmmPlan {
    uint32_t chunk0[EQ_MAX_LAYERS];
    uint64_t srow[EQ_MAX_LAYERS];
};

static eq_status qmm_validate(const eq_block* blk, uint32_t n_jobs, const uint32_t* layers, uint32_t batch,
                              QmmPlan* plan) {
    if (!blk || !layers || n_jobs < 1 || n_jobs > EQ_MAX_LAYERS) return EQ_ERR_ARG;
    if (!blk->payload || !blk->chunk_off || !blk->freq || !blk->scales || blk->format > EQ_FMT_INT8) return EQ_ERR_ARG;
    if (blk->codec > EQ_CODEC_PAIR_G) return EQ_ERR_ARG;
    if (blk->n_layers < 1 || blk->n_layers > EQ_MAX_LAYERS) return EQ_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(blk->payload) & 15) != 0) return EQ_ERR_ARG;
    if (blk->payload_cap < blk->payload_bytes + EQ_PAYLOAD_SLACK) return EQ_ERR_BUFFER;
    const uint32_t cs = blk->chunk_symbols;
    if (blk->chunk_mode > EQ_CHUNK_ROW) return EQ_ERR_ARG;
    if (batch < 1 || batch > 256 || cs == 0 || cs % kQK != 0) return EQ_ERR_SHAPE;
    uint32_t chunk0 = 0;
    uint64_t srow = 0;
    for (uint32_t l = 0; l < blk->n_layers; ++l) {
        plan->chunk0[l] = chunk0;
        plan->srow[l] = srow;
        chunk0 += (uint32_t)layer_chunks(blk->chunk_mode, blk->layer_rows[l], blk->layer_cols[l], cs);
        srow += (uint64_t)blk->layer_rows[l];
    }
    for (uint32_t q = 0; q < n_jobs; ++q) {
        const uint32_t l = layers[q];
        if (l >= blk->n_layers) return EQ_ERR_ARG;
        const uint64_t rows = blk->layer_rows[l], K = blk->layer_cols[l];
        // a row's chunks must be independent K slices: row chunking (any K, multiple of the K
        // step), or layer chunking with rows made of whole chunks
        const bool row_aligned = blk->chunk_mode == EQ_CHUNK_ROW ? K % kQK == 0 : K % cs == 0;
        if (rows == 0 || rows % kTileRows != 0 || K == 0 || !row_aligned) return EQ_ERR_SHAPE;
    }
    return EQ_OK;
}

static uint64_t qmm_part_bytes(uint64_t cpr, uint64_t batch, uint64_t rows) {
    return cpr > 1 ? (cpr * batch * rows * 4 + EQ_ARENA_ALIGN - 1) / EQ_ARENA_ALIGN * EQ_ARENA_ALIGN : 0;
}

// cuTensorMapEncodeTiled from the driver, resolved once through the runtime (no libcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// Launch of k_qmm_ws (word / pair codecs): one CTA per (GEMM, 128-row tile, chunk column);
// the split-K partials go to the same workspace offsets as the byte-codec kernel's (the caller
// runs k_qmm_reduce afterwards).
static eq_status qmm_ws_launch(const eq_block* blk, uint32_t n_jobs, const uint32_t* layers, const QmmPlan& plan,
                               const void* const* x, float* const* y, uint32_t batch, void* workspace, uint32_t* d_err,
                               cudaStream_t st) {
    auto encode = tensor_map_encoder();
    if (!encode) return EQ_ERR_CUDA;
    QmmWsParams W;
    memset(&W, 0, sizeof(W));
    const uint32_t cs = blk->chunk_symbols;
    const uint32_t n_pad = (batch + 15) & ~15u;    // UMMA N: a multiple of 16 for M = 128
    uint64_t ws_off = 0;
    uint32_t tiles = 0;
    for (uint32_t q = 0; q < n_jobs; ++q) {
        const uint32_t l = layers[q];
        QmmJob& J = W.job[q];
        J.x = static_cast<const uint16_t*>(x[q]);
        J.scales = blk->scales + plan.srow[l];
        J.chunk0 = plan.chunk0[l];
        J.rows = blk->layer_rows[l];
        J.K = blk->layer_cols[l];
        J.cpr = (J.K + cs - 1) / cs;
        J.tile_begin = tiles;
        tiles += (J.rows + kQmmNTile * kTileRows - 1) / (kQmmNTile * kTileRows) * J.cpr;
        if (J.cpr == 1) {
            J.out = y[q];
        } else {
            J.out = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + ws_off);
            ws_off += qmm_part_bytes(J.cpr, batch, J.rows);
        }
        // X [batch, K] bf16 row-major: dims {K, batch}, row stride 2K bytes, box {32, n_pad}
        const cuuint64_t dims[2] = {J.K, batch};
        const cuuint64_t strides[1] = {(cuuint64_t)J.K * 2};
        const cuuint32_t box[2] = {(cuuint32_t)kWsK, n_pad};
        const cuuint32_t estr[2] = {1, 1};
        if (encode(&W.tmap[q], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x[q]), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return EQ_ERR_ARG;
    }
    W.n_jobs = n_jobs;
    W.payload = blk->payload;
    W.off = blk->chunk_off;
    W.freq = blk->freq;
    W.payload_bytes = blk->payload_bytes;
    W.err = d_err;
    W.format = blk->format;
    W.cs = cs;
    W.n_pad = n_pad;
    W.n_real = batch;
    W.tmem_cols = 32;
    while (W.tmem_cols < kQmmNTile * n_pad) W.tmem_cols <<= 1;
    W.b_stage_bytes = (n_pad * (uint32_t)kWsRowB + 1023u) & ~1023u;
    // instruction descriptor, kind::f16: D f32, A = B = bf16, both K-major, N = n_pad, M = 128
    W.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((n_pad >> 3) << 17) | ((128u >> 4) << 24);
    W.k2p20 = 1u << 20;
    W.k2p12 = 1u << 12;
    W.kneg2p14 = 0u - (1u << 14);
    W.k4 = 4u;
    const size_t tab = is_pair_codec(blk->codec)
                           ? kPairSmemBytes + (blk->codec == EQ_CODEC_PAIR_G && EQ_QMM_VALS ? 4 * kPairValWords : 0)
                           : (kM + 260) * 4;
    auto smem_for = [&](int stages) {
        return (size_t)1024 + stages * kQmmNTile * kWsATile + stages * W.b_stage_bytes + ((tab + 127) & ~(size_t)127) +
               kQmmNTile * kWsDec * kWRing + 2 * stages * 8 + 16;
    };
    const uint32_t codec = blk->codec;
    const void* fS = codec == EQ_CODEC_PAIR_G ? (const void*)k_qmm_ws<EQ_CODEC_PAIR_G, kQmmNTile, kWsStages>
                   : codec == EQ_CODEC_PAIR   ? (const void*)k_qmm_ws<EQ_CODEC_PAIR, kQmmNTile, kWsStages>
                                              : (const void*)k_qmm_ws<EQ_CODEC_WORD, kQmmNTile, kWsStages>;
    const void* f1 = codec == EQ_CODEC_PAIR_G ? (const void*)k_qmm_ws<EQ_CODEC_PAIR_G, kQmmNTile, 1>
                   : codec == EQ_CODEC_PAIR   ? (const void*)k_qmm_ws<EQ_CODEC_PAIR, kQmmNTile, 1>
                                              : (const void*)k_qmm_ws<EQ_CODEC_WORD, kQmmNTile, 1>;
    const int threads = 32 * (4 * kQmmNTile + 1);
    // resident CTAs per SM with kWsStages stages and with 1: one stage (the decoders then wait for
    // each step's MMAs: ~6 % slower per CTA) only when it turns two waves into one — e.g. a
    // Llama-3-8B block at chunk 2048 and batch 64, where the 4 KB X stages cost the third CTA/SM
    int dev = 0, sms = 0, cS = 0, c1 = 0;
    EQ_CUDA_TRY(cudaGetDevice(&dev));
    EQ_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    EQ_CUDA_TRY(cudaFuncSetAttribute(fS, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_for(kWsStages)));
    EQ_CUDA_TRY(cudaFuncSetAttribute(f1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_for(1)));
    // resident CTAs from the kernels' own resource use (cudaOccupancyMaxActiveBlocksPerMultiprocessor
    // reports 1 for these tcgen05 kernels, while 3 run per SM: ncu launch__occupancy_limit_*)
    int smem_sm = 0, reserved = 0;
    EQ_CUDA_TRY(cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    EQ_CUDA_TRY(cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev));
    auto ctas_per_sm = [&](const void* f, size_t dyn, int* out) -> cudaError_t {
        cudaFuncAttributes a;
        cudaError_t e = cudaFuncGetAttributes(&a, f);
        if (e != cudaSuccess) return e;
        const size_t per = a.sharedSizeBytes + dyn + (size_t)reserved;
        const int by_smem = (int)((size_t)smem_sm / per);
        const int regs = ((a.numRegs * 32 + 255) / 256) * 256 * (threads / 32);   // per-warp allocation granularity
        const int by_regs = regs > 0 ? 65536 / regs : 32;
        *out = std::min(std::min(by_smem, by_regs), 2048 / threads);
        return cudaSuccess;
    };
    EQ_CUDA_TRY(ctas_per_sm(fS, smem_for(kWsStages), &cS));
    EQ_CUDA_TRY(ctas_per_sm(f1, smem_for(1), &c1));
    const bool one = (uint64_t)tiles > (uint64_t)cS * sms && (uint64_t)tiles <= (uint64_t)c1 * sms;
    const size_t smem = smem_for(one ? 1 : kWsStages);
    if (codec == EQ_CODEC_PAIR_G) {
        if (one) k_qmm_ws<EQ_CODEC_PAIR_G, kQmmNTile, 1><<<tiles, threads, smem, st>>>(W);
        else k_qmm_ws<EQ_CODEC_PAIR_G, kQmmNTile, kWsStages><<<tiles, threads, smem, st>>>(W);
    } else if (codec == EQ_CODEC_PAIR) {
        if (one) k_qmm_ws<EQ_CODEC_PAIR, kQmmNTile, 1><<<tiles, threads, smem, st>>>(W);
        else k_qmm_ws<EQ_CODEC_PAIR, kQmmNTile, kWsStages><<<tiles, threads, smem, st>>>(W);
    } else {
        if (one) k_qmm_ws<EQ_CODEC_WORD, kQmmNTile, 1><<<tiles, threads, smem, st>>>(W);
        else k_qmm_ws<EQ_CODEC_WORD, kQmmNTile, kWsStages><<<tiles, threads, smem, st>>>(W);
    }
    EQ_CUDA_TRY(cudaGetLastError());
    return EQ_OK;
}

}  // namespace eq

using namespace eq;

extern "C" uint64_t eq_qmatmul_workspace_bytes(const eq_block* blk, uint32_t n_jobs, const uint32_t* layers,
                                               uint32_t batch) {
    QmmPlan plan;
    if (qmm_validate(blk, n_jobs, layers, batch, &plan) != EQ_OK) return 0;
    uint64_t total = 0;
    for (uint32_t q = 0; q < n_jobs; ++q) {
        const uint32_t l = layers[q];
        total += qmm_part_bytes((blk->layer_cols[l] + blk->chunk_symbols - 1) / blk->chunk_symbols, batch, blk->layer_rows[l]);
    }
    return total;
}

extern "C" eq_status eq_qmatmul_group(const eq_block* blk, uint32_t n_jobs, const uint32_t* layers,
                                      const void* const* x, float* const* y, uint32_t batch, void* workspace,
                                      uint64_t workspace_bytes, uint32_t* d_err, eq_stream_t stream) {
    QmmPlan plan;
    const eq_status vs = qmm_validate(blk, n_jobs, layers, batch, &plan);
    if (vs != EQ_OK) return vs;
    if (!x || !y || !d_err) return EQ_ERR_ARG;
    const uint64_t need = eq_qmatmul_workspace_bytes(blk, n_jobs, layers, batch);
    if (need > 0 && (!workspace || workspace_bytes < need)) return EQ_ERR_BUFFER;
    if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return EQ_ERR_ARG;
    QmmParams P;
    memset(&P, 0, sizeof(P));
    RedParams R;
    memset(&R, 0, sizeof(R));
    uint32_t n_red = 0;
    uint32_t max_red = 0;
    uint64_t ws_off = 0;
    uint32_t tiles = 0;
    const uint32_t cs = blk->chunk_symbols;
    for (uint32_t q = 0; q < n_jobs; ++q) {
        const uint32_t l = layers[q];
        if (!x[q] || !y[q] || (reinterpret_cast<uintptr_t>(x[q]) & 15) != 0 || (reinterpret_cast<uintptr_t>(y[q]) & 15) != 0)
            return EQ_ERR_ARG;
        QmmJob& J = P.job[q];
        J.x = static_cast<const uint16_t*>(x[q]);
        J.scales = blk->scales + plan.srow[l];
        J.chunk0 = plan.chunk0[l];
        J.rows = blk->layer_rows[l];
        J.K = blk->layer_cols[l];
        J.cpr = (J.K + cs - 1) / cs;
        J.tile_begin = tiles;
        tiles += (J.rows / kTileRows + kTiles - 1) / kTiles * J.cpr;
        if (J.cpr == 1) {
            J.out = y[q];
        } else {
            J.out = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + ws_off);
            ws_off += qmm_part_bytes(J.cpr, batch, J.rows);
            R.job[n_red].part = J.out;
            R.job[n_red].y = y[q];
            R.job[n_red].n = batch * J.rows;
            R.job[n_red].cpr = J.cpr;
            max_red = std::max(max_red, R.job[n_red].n);
            ++n_red;
        }
    }
    if (blk->codec != EQ_CODEC_BYTE) {            // warp-specialised kernel (word and pair codecs)
        const eq_status ws = qmm_ws_launch(blk, n_jobs, layers, plan, x, y, batch, workspace, d_err,
                                           (cudaStream_t)stream);
        if (ws != EQ_OK) return ws;
        if (n_red) {
            const uint32_t gx = std::min<uint32_t>((max_red / 4 + 255) / 256, 148u * 8u);
            k_qmm_reduce<<<dim3(gx, n_red), 256, 0, (cudaStream_t)stream>>>(R);
            EQ_CUDA_TRY(cudaGetLastError());
        }
        return EQ_OK;
    }
    P.n_jobs = n_jobs;
    P.payload = blk->payload;
    P.off = blk->chunk_off;
    P.freq = blk->freq;
    P.payload_bytes = blk->payload_bytes;
    P.err = d_err;
    P.format = blk->format;
    P.cs = cs;
    P.n_pad = (batch + 15) & ~15u;             // UMMA N for M = 128: a multiple of 16 (PTX ISA)
    P.n_real = batch;
    P.acc_cols = P.n_pad;                      // half h accumulates in columns [h·n_pad, (h+1)·n_pad)
    P.tmem_cols = 32;
    while (P.tmem_cols < kTiles * P.n_pad) P.tmem_cols <<= 1;
    // instruction descriptor, kind::f16: D f32, A = B = bf16, both K-major, N, M = 128
    P.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((P.n_pad >> 3) << 17) | ((128u >> 4) << 24);
    P.k2p20 = 1u << 20;
    P.k2p12 = 1u << 12;
    P.kneg2p14 = 0u - (1u << 14);
    P.k4 = 4u;
    const uint32_t b_tile = ((P.n_pad * (uint32_t)kRowB + 1023u) & ~1023u);
    const size_t smem = kTiles * kATile + b_tile + kM * 4 + kQThreads * kRingWords * 4 + 32 + 8 + 8 + 1024;
    if (blk->codec == EQ_CODEC_WORD) {
        EQ_CUDA_TRY(cudaFuncSetAttribute(k_qmatmul<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_qmatmul<true><<<tiles, kQThreads, smem, (cudaStream_t)stream>>>(P);
    } else {
        EQ_CUDA_TRY(cudaFuncSetAttribute(k_qmatmul<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_qmatmul<false><<<tiles, kQThreads, smem, (cudaStream_t)stream>>>(P);
    }
    EQ_CUDA_TRY(cudaGetLastError());
    if (n_red) {
        const uint32_t gx = std::min<uint32_t>((max_red / 4 + 255) / 256, 148u * 8u);
        k_qmm_reduce<<<dim3(gx, n_red), 256, 0, (cudaStream_t)stream>>>(R);
        EQ_CUDA_TRY(cudaGetLastError());
    }
    return EQ_OK;
}

extern "C" eq_status eq_qmatmul(const eq_block* blk, uint32_t layer, const void* x, uint32_t batch, float* y,
                                void* workspace, uint64_t workspace_bytes, uint32_t* d_err, eq_stream_t stream) {
    const void* xs[1] = {x};
    float* ys[1] = {y};
    return eq_qmatmul_group(blk, 1, &layer, xs, ys, batch, workspace, workspace_bytes, d_err, stream);
}
