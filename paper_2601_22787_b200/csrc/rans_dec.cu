// rans_dec.cu — §8(a) rows a7 + a8: chunk-parallel byte-wise rANS decode of E4M3 symbol
// streams (Alg. 2 l.1) with the dequantiser Q† fused into the store, into
// a per-device arena with one view per layer (App. A.1).
//
// Design:
//  - one launch covers all chunks of up to kMaxDecBlocks blocks (enough independent
//    chains to hide the serial per-chunk dependency: Little's law);
//  - a CTA owns kDecThreads consecutive chunks of ONE block; lane = chunk, the rANS state
//    and a 64-bit bit-buffer of upcoming payload bytes live in registers;
//  - the block's decode LUT (4096 × u32: sym | (f−1)<<8 | (slot−c)<<20) is built in shared
//    memory by each CTA from the 256-entry frequency table (no global LUT, no extra pass);
//  - output in 16-symbol groups: 16 B (FP8) or 32 B (bf16) vector stores; one row scale
//    per group when cols % 16 == 0 (generic per-symbol path otherwise).
#include "common.cuh"

#include <algorithm>
#include <cstring>
#include <memory>

namespace eq {

#ifndef EQ_DEC_CHAINS
#define EQ_DEC_CHAINS 1
#endif
#ifndef EQ_K_FLO
#define EQ_K_FLO 1
#endif
constexpr int kChunksPerCta = 256;
constexpr int kChains = EQ_DEC_CHAINS;            // independent chunks per thread (ILP)
constexpr int kDecThreads = kChunksPerCta / kChains;
constexpr int kMaxDecBlocks = 48;
constexpr int kRingWords = 16;

struct DecLayer {
    uint64_t out_off;      // byte offset of the layer in the arena
    uint64_t size;         // rows * cols symbols
    uint32_t chunk0;       // first chunk index of the layer within its block
    uint32_t cols;
    uint32_t scale_off;    // first row's index into the block's scale array
    uint32_t pad;
};

struct DecBlock {
    const uint8_t* payload;
    const uint32_t* off;
    const uint16_t* freq;
    const uint16_t* scales;
    uint64_t payload_bytes;
    uint32_t format;       // EQ_FMT_E4M3 | EQ_FMT_INT8 (bf16 dequant of the codes)
    uint32_t pad0;
    uint32_t n_chunks;
    uint32_t cs;           // chunk symbols
    uint32_t n_layers;
    uint32_t cta0;         // first CTA of this block in the grid
    DecLayer layer[EQ_MAX_LAYERS];
};

struct DecParams {
    uint8_t* arena;
    uint32_t* err;
    uint32_t n_blocks;
    uint32_t pad;
    // multipliers passed at run time so ptxas keeps IMAD / IMAD.HI (FMA pipe) instead of
    // strength-reducing them to LEA / SHF on the (binding) integer ALU pipe
    uint32_t k2p20, k2p12, kneg2p14, k4;
    DecBlock b[kMaxDecBlocks];
};

// ---------------------------------------------------------------- per-chunk bit reader
// Upcoming payload bits, most significant first, in a 64-bit window (hi:lo) holding nb
// valid bits.  A symbol consumes k ∈ {0,8,16} bits with funnel shifts (branch-free);
// refill() runs after every PAIR of symbols and restores nb ≥ 32.
// The chunk's compressed bytes are staged in a 64-byte shared-memory ring by cp.async
// (16-byte segments issued thread-uniformly every 8 symbols, ≥ 8 symbols before use), so
// no register ever waits on a global load (the warp-level scoreboard would otherwise
// serialise the lanes' independent refills).
struct BitReader {
    uint32_t hi, lo;
    int nb;
    uint32_t wi4;          // 4 × (absolute index of the next payload word to insert)
    uint32_t gs;           // next 16-byte payload segment to stage
    uint32_t ring;         // shared address of this chunk's ring (64-byte aligned)

    __device__ __forceinline__ void refill() {
        if (nb < 32) {                              // predicated, not a divergent branch
            uint32_t w;
            asm("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(ring | (wi4 & 0x3Cu)));
            w = bswap32(w);
            hi += w >> nb;                          // = |: the low 32−nb bits of hi are 0
            lo = __funnelshift_r(0u, w, nb);        // = w << (32 − nb)
            nb += 32;
            wi4 += 4;
        }
    }
};

#ifndef EQ_L2HINT
#define EQ_L2HINT 0
#endif
// L2 policies: the compressed input is re-read segment by segment while ~14 GB of output
// streams through L2, so input lines are kept (evict_last) and output lines go first
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void stage_segment(uint32_t ring, const uint8_t* payload, uint32_t seg) {
#if EQ_L2HINT
    asm volatile("cp.async.cg.shared.global.L2::cache_hint.L2::128B [%0], [%1], 16, %2;" ::"r"(ring | ((seg & 3u) << 4)),
                 "l"(payload + (uint64_t)seg * 16), "l"(policy_evict_last()));
#else
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(ring | ((seg & 3u) << 4)),
                 "l"(payload + (uint64_t)seg * 16));
#endif
}
__device__ __forceinline__ void stage_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void stage_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Every 8 symbols (after stage_wait_all): stage one more segment if fewer than 13 words
// lie ahead of the reader.  ≤ 4 words are consumed per 8 symbols, so the words needed
// before the next boundary have always landed and the ring never overwrites an unread word.
__device__ __forceinline__ void ring_issue(BitReader& br, const uint8_t* payload) {
    if (br.gs * 16u <= br.wi4 + 48u) {
        stage_segment(br.ring, payload, br.gs);
        ++br.gs;
    }
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// LUT address: one LOP3 + one IMAD (slot·4 + base) — written in PTX so ptxas keeps the
// mad instead of re-deriving it as shl / and / add
__device__ __forceinline__ uint32_t lut_addr(uint32_t x, uint32_t lut_s) {
    uint32_t a;
    asm("{ .reg .u32 t; and.b32 t, %1, 4095; mad.lo.u32 %0, t, 4, %2; }" : "=r"(a) : "r"(x), "r"(lut_s));
    return a;
}

// bytes to read after a step, ×8: 0 if x ≥ 2^23, 8 if x ≥ 2^15, else 16 (x ≥ 2^11)
__device__ __forceinline__ uint32_t renorm_bits(uint32_t x) {
#if EQ_K_FLO
    // clz(2x) = clz(x) − 1: one IMAD (FMA pipe), FLO.SH (XU pipe), LOP3
    uint32_t z;
    asm("bfind.shiftamt.u32 %0, %1;" : "=r"(z) : "r"(x + x));
    return z & 0x18u;
#else
    return (x < (1u << 23) ? 8u : 0u) + (x < (1u << 15) ? 8u : 0u);
#endif
}

#ifndef EQ_ZFAST
#define EQ_ZFAST 0
#endif
// Per-block constants of the decode step.  ez = the LUT entry of code 0x00 with slot 0:
// code 0x00 is first in code order, so its slots are [0, f0) and its entry for slot s is
// ez | s << 20 — computed in registers instead of loaded, which removes the most frequent
// symbol's lanes from the shared-memory LUT access (fewer bank conflicts).
struct DecTable {
    uint32_t k2p20, k2p12, kneg2p14, k4;   // 2^20, 2^12, −2^14, 4 (see DecParams)
    uint32_t lut_s;        // shared address of the LUT
    uint32_t f0;           // frequency of code 0x00
    uint32_t ez;           // (f0 − 1) << 8
};

// One rANS decode step (Alg. 2 l.1): slot lookup, state update, byte renormalisation.
// LUT entry e: sym | (f−1) << 8 | (slot − c_sym) << 20; returns e (sym in the low byte).
// Field extraction and x>>12 use IMAD.HI (FMA pipe) to balance the integer ALU pipe.
__device__ __forceinline__ uint32_t mad_hi(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// One rANS decode step (Alg. 2 l.1): slot lookup, state update, byte renormalisation.
// LUT entry e: sym | (f−1) << 8 | (slot − c_sym) << 20; returns e (sym in the low byte).
// Everything that has an exact integer-multiply form runs as IMAD / IMAD.HI on the FMA
// pipe, leaving the (binding) ALU pipe the funnel shifts, masks and byte permutes:
//   xs = x >> 12 = hi(x · 2^20);  slot·4 + base = 4x − 2^14·xs + base
//   xs + (slot − c) = hi(e · 2^12) + xs;  f − 1 = hi((e << 12) · 2^12)
__device__ __forceinline__ uint32_t decode_one(uint32_t& x, BitReader& br, const DecTable& T) {
#if EQ_ZFAST
    const uint32_t slot = x & (kM - 1);
    uint32_t e = T.ez | (slot << 20);
    if (slot >= T.f0) e = lds_u32(T.lut_s + slot * 4u);
    const uint32_t xs = mad_hi(x, 1u << 20, 0u);
#else
    const uint32_t xs = mad_hi(x, T.k2p20, 0u);                         // x >> 12
    const uint32_t e = lds_u32(mad_lo(x, T.k4, mad_lo(xs, T.kneg2p14, T.lut_s)));
#endif
    const uint32_t fm1 = mad_hi(mad_lo(e, T.k2p12, 0u), T.k2p12, 0u);   // (e >> 8) & 0xFFF
    x = mad_lo(fm1, xs, xs + (e >> 20));                                // f·⌊x/M⌋ + slot − c
    const uint32_t k = renorm_bits(x);
    x = __funnelshift_lc(br.hi, x, k);
    br.hi = __funnelshift_lc(br.lo, br.hi, k);
    br.lo = br.lo << k;
    br.nb -= (int)k;
    return e;
}

// Q† on two codes: exact e4m3 -> f32, one exact f32 product each, one RNE to bf16 each
__device__ __forceinline__ uint32_t dequant2(uint32_t pair, float s) {
    const float2 v = e4m3x2_to_float2(pair);
    __nv_bfloat162 b = __floats2bfloat162_rn(__fmul_rn(s, v.x), __fmul_rn(s, v.y));
    return *reinterpret_cast<uint32_t*>(&b);
}

// Same result when the row scale is exactly representable in f16 (bf16's 8-bit mantissa
// fits f16's 11 bits; only the range is checked): the e4m3 pair unpacks to f16x2 and the
// mixed-precision FHFMA multiplies each f16 half by the f16 scale straight into f32 —
// the product of a 4- and an 8-bit significand is exact in f32 — then one RNE to bf16.
__device__ __forceinline__ uint32_t dequant2_h(uint32_t pair, uint16_t s16) {
    __half2_raw h = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(pair & 0xFFFFu), __NV_E4M3);
    const uint32_t hv = *reinterpret_cast<uint32_t*>(&h);
    float a, b;
    asm("{ .reg .b16 l, u; mov.b32 {l, u}, %2; fma.rn.f32.f16 %0, l, %3, 0f00000000; fma.rn.f32.f16 %1, u, %3, 0f00000000; }"
        : "=f"(a), "=f"(b) : "r"(hv), "h"(s16));
    __nv_bfloat162 r = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&r);
}

// Int8 base format: s · c is exact in f32 (8 + 8 significant bits), one RNE to bf16
__device__ __forceinline__ uint32_t dequant2_i8(uint32_t pair, float s) {
    const float a = (float)(int8_t)(pair & 0xFFu), b = (float)(int8_t)((pair >> 8) & 0xFFu);
    __nv_bfloat162 r = __floats2bfloat162_rn(__fmul_rn(s, a), __fmul_rn(s, b));
    return *reinterpret_cast<uint32_t*>(&r);
}

// f16 bits of a bf16 scale if exactly representable (normal f16 range), else 0
__device__ __forceinline__ uint16_t scale_f16(float s) {
    const float a = fabsf(s);
    if (!(a >= 6.103515625e-05f && a <= 65504.f)) return 0;
    __half h = __float2half_rn(s);
    return *reinterpret_cast<uint16_t*>(&h);
}

// decoded output is written once and never re-read by this kernel: evict-first in L2
__device__ __forceinline__ void st_out(uint4* p, uint4 v) { __stcs(p, v); }

#ifndef EQ_ST256
#define EQ_ST256 1
#endif
// 32 bytes per lane in one STG.256 (sm_100): half the store instructions and L1 wavefronts
// of two STG.128 to the same per-lane line
__device__ __forceinline__ void st_out32(void* p, uint4 a, uint4 b) {
#if EQ_ST256 && EQ_L2HINT
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z),
                 "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                 : "memory");
#elif EQ_ST256
    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y),
                 "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                 : "memory");
#else
    st_out(reinterpret_cast<uint4*>(p), a);
    st_out(reinterpret_cast<uint4*>(p) + 1, b);
#endif
}

template <bool BF16>
__device__ __forceinline__ void store_one(uint8_t* out, uint64_t i, uint32_t sym, float s, bool i8) {
    if (BF16) {
        float v;
        if (i8) {
            v = (float)(int8_t)sym;
        } else {
            __half_raw h = __nv_cvt_fp8_to_halfraw((__nv_fp8_storage_t)sym, __NV_E4M3);
            v = __half2float(*reinterpret_cast<__half*>(&h));
        }
        reinterpret_cast<uint16_t*>(out)[i] = float_to_bf16_bits(__fmul_rn(s, v));
    } else {
        out[i] = (uint8_t)sym;
    }
}

// ---------------------------------------------------------------- one chunk's decode state
struct Chain {
    uint32_t x;
    BitReader br;
    uint8_t* out;
    const uint16_t* sc;
    uint32_t row, col, cols;
    float s;
    uint16_t s16;          // f16 bits of s when exact, else 0 (FMUL path)
    bool i8;               // Int8 base format
    uint32_t n, i;
    uint32_t a;            // chunk payload byte range [a, e)
    uint32_t e;
    uint32_t wlimit4;      // runaway guard: 64 bytes past the chunk end
    bool active, runaway, fast;
};

// 4 symbols -> one word of codes (first symbol in the low byte), two pair refills
__device__ __forceinline__ uint32_t decode4(Chain& c, const DecTable& T) {
    const uint32_t a = decode_one(c.x, c.br, T);
    const uint32_t b = decode_one(c.x, c.br, T);
    c.br.refill();
    const uint32_t d = decode_one(c.x, c.br, T);
    const uint32_t f = decode_one(c.x, c.br, T);
    c.br.refill();
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(d, f, 0x0040), 0x5410);
}

#ifndef EQ_UNROLL2
#define EQ_UNROLL2 0
#endif
__device__ __forceinline__ void store16_bf16_at(Chain& c, const uint32_t q[4], uint8_t* dst);

// 16 symbols -> bf16 with one row scale (cols % 16 == 0), 32-byte store
__device__ __forceinline__ void store16_bf16(Chain& c, const uint32_t q[4]) {
    store16_bf16_at(c, q, c.out + (uint64_t)c.i * 2);
}

__device__ __forceinline__ void store16_bf16_at(Chain& c, const uint32_t q[4], uint8_t* dst) {
    uint4 lo, hi;
    if (c.i8) {
        lo = make_uint4(dequant2_i8(q[0], c.s), dequant2_i8(q[0] >> 16, c.s), dequant2_i8(q[1], c.s),
                        dequant2_i8(q[1] >> 16, c.s));
        hi = make_uint4(dequant2_i8(q[2], c.s), dequant2_i8(q[2] >> 16, c.s), dequant2_i8(q[3], c.s),
                        dequant2_i8(q[3] >> 16, c.s));
    } else if (c.s16) {
        lo = make_uint4(dequant2_h(q[0], c.s16), dequant2_h(q[0] >> 16, c.s16), dequant2_h(q[1], c.s16),
                        dequant2_h(q[1] >> 16, c.s16));
        hi = make_uint4(dequant2_h(q[2], c.s16), dequant2_h(q[2] >> 16, c.s16), dequant2_h(q[3], c.s16),
                        dequant2_h(q[3] >> 16, c.s16));
    } else {
        lo = make_uint4(dequant2(q[0], c.s), dequant2(q[0] >> 16, c.s), dequant2(q[1], c.s), dequant2(q[1] >> 16, c.s));
        hi = make_uint4(dequant2(q[2], c.s), dequant2(q[2] >> 16, c.s), dequant2(q[3], c.s), dequant2(q[3] >> 16, c.s));
    }
    st_out32(dst, lo, hi);
    c.col += 16;
    if (c.col >= c.cols) {
        c.col -= c.cols;
        ++c.row;
        if (c.i + 16 < c.n) {
            c.s = bf16_bits_to_float(c.sc[c.row]);
            c.s16 = c.i8 ? 0 : scale_f16(c.s);
        }
    }
}

template <bool BF16>
__device__ __forceinline__ void chain_setup(Chain& c, const DecBlock& B, uint32_t chunk, uint32_t ring,
                                            uint8_t* arena, uint32_t* err) {
    c.active = chunk < B.n_chunks;
    c.runaway = false;
    c.i = 0;
    c.n = 0;
    if (!c.active) return;
    uint32_t l = 0;
    while (l + 1 < B.n_layers && chunk >= B.layer[l + 1].chunk0) ++l;
    const DecLayer& Ly = B.layer[l];
    const uint64_t sym0 = (uint64_t)(chunk - Ly.chunk0) * B.cs;
    c.n = (uint32_t)min((uint64_t)B.cs, Ly.size - sym0);
    const uint32_t a = __ldg(B.off + chunk), e = __ldg(B.off + chunk + 1);
    if (e < a || (uint64_t)e > B.payload_bytes || e - a < 4) {
        atomicOr(err, EQ_EF_TRUNCATED);
        c.active = false;
        return;
    }
    c.a = a;
    c.e = e;
    c.wlimit4 = ((e >> 2) + 16) * 4u;
    c.br.ring = ring;
    const uint32_t s0 = a >> 4;
    #pragma unroll
    for (int q = 0; q < 4; ++q) stage_segment(ring, B.payload, s0 + q);
    c.br.gs = s0 + 4;
    c.out = arena + Ly.out_off + sym0 * (BF16 ? 2 : 1);
    c.sc = B.scales + Ly.scale_off;
    c.cols = Ly.cols;
    c.row = (uint32_t)(sym0 / Ly.cols);
    c.col = (uint32_t)(sym0 % Ly.cols);
    c.s = BF16 ? bf16_bits_to_float(c.sc[c.row]) : 0.f;
    c.i8 = B.format == EQ_FMT_INT8;
    c.s16 = (BF16 && !c.i8) ? scale_f16(c.s) : 0;
    c.fast = BF16 ? ((Ly.cols & 15) == 0 && (B.cs & 15) == 0) : ((B.cs & 31) == 0);
}

// after the initial segments landed: read the 4-byte state and fill the window
__device__ __forceinline__ void chain_start(Chain& c) {
    if (!c.active) return;
    const uint32_t wa = c.a >> 2;
    uint32_t h = bswap32(lds_u32(c.br.ring | ((wa * 4u) & 0x3Cu)));
    uint32_t m = bswap32(lds_u32(c.br.ring | (((wa + 1) * 4u) & 0x3Cu)));
    const uint32_t sh = (c.a & 3) * 8;
    c.x = bswap32(__funnelshift_lc(m, h, sh));  // 4-byte little-endian initial state
    c.br.hi = m << sh;                           // remaining bytes of word 1
    c.br.lo = 0;
    c.br.nb = 32 - (int)sh;
    c.br.wi4 = (wa + 2) * 4u;
    c.br.refill();                               // nb ≥ 32 from here on, at pair starts
}

// one chunk alone from its current position to its end (16/32-symbol groups while the
// layout allows, then one symbol at a time)
template <bool BF16>
__device__ __forceinline__ void chain_finish(Chain& c, const uint8_t* payload, const DecTable& T) {
    if (!c.active || c.runaway) return;
    if (c.fast) {
        const uint32_t G = BF16 ? 16 : 32;
#if EQ_UNROLL2
        if (BF16) {
            // two 16-symbol groups per iteration with a running output pointer (fewer
            // loop-control and address instructions per symbol)
            uint8_t* o = c.out + (uint64_t)c.i * 2;
            while (c.i + 32 <= c.n) {
                #pragma unroll
                for (int g = 0; g < 2; ++g) {
                    uint32_t q[4];
                    q[0] = decode4(c, T);
                    q[1] = decode4(c, T);
                    stage_wait_all(); ring_issue(c.br, payload); stage_commit();
                    q[2] = decode4(c, T);
                    q[3] = decode4(c, T);
                    stage_wait_all(); ring_issue(c.br, payload); stage_commit();
                    store16_bf16_at(c, q, o + 32 * g);
                    c.i += 16;
                }
                o += 64;
                if (c.br.wi4 > c.wlimit4) { c.runaway = true; return; }
            }
        }
#endif
        while (c.i + G <= c.n) {
            if (BF16) {
                uint32_t q[4];
                q[0] = decode4(c, T);
                q[1] = decode4(c, T);
                stage_wait_all(); ring_issue(c.br, payload); stage_commit();
                q[2] = decode4(c, T);
                q[3] = decode4(c, T);
                stage_wait_all(); ring_issue(c.br, payload); stage_commit();
                store16_bf16(c, q);
            } else {
                uint32_t q[8];
                #pragma unroll
                for (int k = 0; k < 8; ++k) {
                    q[k] = decode4(c, T);
                    if (k & 1) { stage_wait_all(); ring_issue(c.br, payload); stage_commit(); }
                }
                st_out32(c.out + c.i, make_uint4(q[0], q[1], q[2], q[3]), make_uint4(q[4], q[5], q[6], q[7]));
            }
            c.i += G;
            if (c.br.wi4 > c.wlimit4) { c.runaway = true; return; }
        }
    }
    for (; c.i < c.n; ++c.i) {                  // generic / ragged tail: one symbol at a time
        const uint32_t sym = decode_one(c.x, c.br, T) & 0xFFu;
        c.br.refill();
        if ((c.i & 7) == 7) { stage_wait_all(); ring_issue(c.br, payload); stage_commit(); }
        store_one<BF16>(c.out, c.i, sym, c.s, c.i8);
        if (BF16 && ++c.col == c.cols) {
            c.col = 0;
            ++c.row;
            if (c.i + 1 < c.n) c.s = bf16_bits_to_float(c.sc[c.row]);
        }
        if (c.br.wi4 > c.wlimit4) { c.runaway = true; return; }
    }
}

#ifndef EQ_DEC_MIN_CTAS
#define EQ_DEC_MIN_CTAS 5
#endif

template <bool BF16>
__global__ void __launch_bounds__(kDecThreads, EQ_DEC_MIN_CTAS)
k_decode(const __grid_constant__ DecParams P) {
    __shared__ uint32_t lut[kM];
    __shared__ uint32_t cum[257];
    __shared__ __align__(64) uint32_t rings[kChunksPerCta * kRingWords];

    uint32_t bi = 0;
    while (bi + 1 < P.n_blocks && blockIdx.x >= P.b[bi + 1].cta0) ++bi;
    const DecBlock& B = P.b[bi];
    const int t = threadIdx.x;

    // ---- chunk setup first: the initial cp.async copies overlap the table build
    Chain ch[kChains];
    #pragma unroll
    for (int j = 0; j < kChains; ++j) {
        const uint32_t slot = (uint32_t)(j * kDecThreads + t);
        chain_setup<BF16>(ch[j], B, (blockIdx.x - B.cta0) * kChunksPerCta + slot,
                          (uint32_t)__cvta_generic_to_shared(rings + slot * kRingWords), P.arena, P.err);
    }
    stage_commit();

    // ---- table: exclusive prefix of the 256 frequencies, then the slot LUT
    {
        __shared__ uint32_t wsum[8];
        const int lane = t & 31, w = t >> 5;
        for (int base = 0; base < 256; base += kDecThreads) {
            uint32_t v = B.freq[base + t];
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                uint32_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
                if (lane >= d) v += o;
            }
            if (lane == 31) wsum[(base >> 5) + w] = v;
            cum[base + t + 1] = v;                  // warp-local inclusive prefix for now
        }
        __syncthreads();
        for (int base = 0; base < 256; base += kDecThreads) {
            const int idx = base + t;
            uint32_t add = 0;
            for (int q = 0; q < (idx >> 5); ++q) add += wsum[q];
            cum[idx + 1] += add;
        }
        if (t == 0) cum[0] = 0;
    }
    __syncthreads();
    if (cum[256] != kM) {                     // corrupt table: nothing decodable
        if (t == 0) atomicOr(P.err, EQ_EF_CORRUPT);
        stage_wait_all();
        return;
    }
    for (int slot = t; slot < (int)kM; slot += kDecThreads) {
        int lo = 0, hi = 255;                  // largest s with cum[s] <= slot
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (cum[mid] <= (uint32_t)slot) lo = mid; else hi = mid - 1;
        }
        uint32_t fs = cum[lo + 1] - cum[lo];
        lut[slot] = (uint32_t)lo | ((fs - 1) << 8) | (((uint32_t)slot - cum[lo]) << 20);
    }
    stage_wait_all();
    __syncthreads();
    DecTable T;
    T.k2p20 = P.k2p20;
    T.k2p12 = P.k2p12;
    T.kneg2p14 = P.kneg2p14;
    T.k4 = P.k4;
    T.lut_s = (uint32_t)__cvta_generic_to_shared(lut);
    T.f0 = cum[1];
    T.ez = (T.f0 - 1) << 8;

    #pragma unroll
    for (int j = 0; j < kChains; ++j) chain_start(ch[j]);

    // ---- joint loop: the chains' independent dependency chains interleave (ILP)
    bool joint = true;
    uint32_t ng = 0xFFFFFFFFu;
    #pragma unroll
    for (int j = 0; j < kChains; ++j) {
        joint = joint && ch[j].active && ch[j].fast;
        ng = min(ng, ch[j].n / (BF16 ? 16u : 32u));
    }
    if (joint && kChains > 1) {
        for (uint32_t g = 0; g < ng; ++g) {
            if (BF16) {
                uint32_t q[kChains][4];
                #pragma unroll
                for (int h = 0; h < 2; ++h) {
                    #pragma unroll
                    for (int r = 0; r < 2; ++r) {
                        #pragma unroll
                        for (int j = 0; j < kChains; ++j) q[j][2 * h + r] = decode4(ch[j], T);
                    }
                    stage_wait_all();
                    #pragma unroll
                    for (int j = 0; j < kChains; ++j) ring_issue(ch[j].br, B.payload);
                    stage_commit();
                }
                #pragma unroll
                for (int j = 0; j < kChains; ++j) {
                    store16_bf16(ch[j], q[j]);
                    ch[j].i += 16;
                }
            } else {
                uint32_t q[kChains][8];
                #pragma unroll
                for (int k = 0; k < 8; ++k) {
                    #pragma unroll
                    for (int j = 0; j < kChains; ++j) q[j][k] = decode4(ch[j], T);
                    if (k & 1) {
                        stage_wait_all();
                        #pragma unroll
                        for (int j = 0; j < kChains; ++j) ring_issue(ch[j].br, B.payload);
                        stage_commit();
                    }
                }
                #pragma unroll
                for (int j = 0; j < kChains; ++j) {
                    st_out32(ch[j].out + ch[j].i, make_uint4(q[j][0], q[j][1], q[j][2], q[j][3]),
                             make_uint4(q[j][4], q[j][5], q[j][6], q[j][7]));
                    ch[j].i += 32;
                }
            }
            bool bad = false;
            #pragma unroll
            for (int j = 0; j < kChains; ++j) bad = bad || (ch[j].br.wi4 > ch[j].wlimit4);
            if (bad) break;
        }
    }
    // ---- remainders (ragged tails, unequal lengths, non-fast layouts), one chain at a time
    #pragma unroll
    for (int j = 0; j < kChains; ++j) {
        if (ch[j].active && ch[j].br.wi4 > ch[j].wlimit4) ch[j].runaway = true;
        chain_finish<BF16>(ch[j], B.payload, T);
    }
    stage_wait_all();
    // integrity: final state L and every payload byte of the chunk consumed exactly
    // (bits inserted into the window = 32·(words inserted) − 8·misalignment)
    #pragma unroll
    for (int j = 0; j < kChains; ++j) {
        const Chain& c = ch[j];
        if (!c.active) continue;
        const int64_t inserted = 8ll * (int64_t)(c.br.wi4 - (c.a >> 2) * 4u) - 8ll * (int64_t)(c.a & 3);
        const int64_t consumed = inserted - c.br.nb;            // includes the 32-bit state
        if (c.runaway || c.x != kL || consumed != 8ll * (int64_t)(c.e - c.a)) atomicOr(P.err, EQ_EF_CORRUPT);
    }
}

}  // namespace eq

using namespace eq;

static uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

extern "C" eq_status eq_arena_layout(const eq_block* blocks, uint32_t n_blocks, uint32_t out_dtype,
                                     uint64_t* layer_offsets, uint64_t* total_bytes) {
    if (!blocks || !total_bytes || n_blocks == 0) return EQ_ERR_ARG;
    if (out_dtype != EQ_OUT_FP8 && out_dtype != EQ_OUT_BF16) return EQ_ERR_ARG;
    const uint64_t esz = out_dtype == EQ_OUT_BF16 ? 2 : 1;
    uint64_t pos = 0;
    for (uint32_t b = 0; b < n_blocks; ++b) {
        if (blocks[b].n_layers == 0 || blocks[b].n_layers > EQ_MAX_LAYERS) return EQ_ERR_ARG;
        for (uint32_t l = 0; l < EQ_MAX_LAYERS; ++l) {
            if (l < blocks[b].n_layers) {
                int64_t r = blocks[b].layer_rows[l], c = blocks[b].layer_cols[l];
                if (r < 1 || c < 1) return EQ_ERR_SHAPE;
                pos = align_up(pos, EQ_ARENA_ALIGN);
                if (layer_offsets) layer_offsets[b * EQ_MAX_LAYERS + l] = pos;
                pos += (uint64_t)r * (uint64_t)c * esz;
            } else if (layer_offsets) {
                layer_offsets[b * EQ_MAX_LAYERS + l] = pos;
            }
        }
    }
    *total_bytes = align_up(pos, EQ_ARENA_ALIGN);
    return EQ_OK;
}

// Validates one block's host description and fills its launch descriptor.
static eq_status fill_desc(const eq_block& blk, const uint64_t* offs, DecBlock& d, uint32_t cta0) {
    if (!blk.payload || !blk.chunk_off || !blk.freq || !blk.scales) return EQ_ERR_ARG;
    if (blk.chunk_symbols == 0 || blk.chunk_symbols > 262144u) return EQ_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(blk.payload) & 15) != 0) return EQ_ERR_ARG;   // cp.async 16-byte segments
    if (blk.payload_cap < blk.payload_bytes + EQ_PAYLOAD_SLACK) return EQ_ERR_BUFFER;
    d.payload = blk.payload;
    d.off = blk.chunk_off;
    d.freq = blk.freq;
    d.scales = blk.scales;
    d.payload_bytes = blk.payload_bytes;
    if (blk.format > EQ_FMT_INT8) return EQ_ERR_ARG;
    d.format = blk.format;
    d.cs = blk.chunk_symbols;
    d.n_layers = blk.n_layers;
    d.cta0 = cta0;
    uint32_t chunk = 0, srow = 0;
    for (uint32_t l = 0; l < EQ_MAX_LAYERS; ++l) {
        DecLayer& L = d.layer[l];
        if (l < blk.n_layers) {
            uint64_t size = (uint64_t)blk.layer_rows[l] * (uint64_t)blk.layer_cols[l];
            L.out_off = offs[l];
            L.size = size;
            L.chunk0 = chunk;
            L.cols = (uint32_t)blk.layer_cols[l];
            L.scale_off = srow;
            chunk += (uint32_t)((size + blk.chunk_symbols - 1) / blk.chunk_symbols);
            srow += (uint32_t)blk.layer_rows[l];
        } else {
            L = DecLayer{0, 0, chunk, 1, srow, 0};
        }
    }
    if (chunk != blk.n_chunks) return EQ_ERR_SHAPE;
    d.n_chunks = chunk;
    return EQ_OK;
}

extern "C" eq_status eq_decode_dequant(const eq_block* blocks, uint32_t n_blocks, uint32_t out_dtype,
                                       void* arena, uint64_t arena_bytes, uint32_t* d_err,
                                       eq_stream_t stream) {
    if (!blocks || !arena || !d_err || n_blocks == 0) return EQ_ERR_ARG;
    if (out_dtype != EQ_OUT_FP8 && out_dtype != EQ_OUT_BF16) return EQ_ERR_ARG;
    // whole-arena layout (validates shapes)
    uint64_t total = 0;
    std::unique_ptr<uint64_t[]> all(new uint64_t[(size_t)n_blocks * EQ_MAX_LAYERS]);
    EQ_TRY(eq_arena_layout(blocks, n_blocks, out_dtype, all.get(), &total));
    if (arena_bytes < total) return EQ_ERR_BUFFER;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    for (uint32_t b0 = 0; b0 < n_blocks; b0 += kMaxDecBlocks) {
        const uint32_t nb = std::min<uint32_t>(kMaxDecBlocks, n_blocks - b0);
        DecParams P;
        memset(&P, 0, sizeof(P));
        P.arena = static_cast<uint8_t*>(arena);
        P.err = d_err;
        P.n_blocks = nb;
        P.k2p20 = 1u << 20;
        P.k2p12 = 1u << 12;
        P.kneg2p14 = 0u - (1u << 14);
        P.k4 = 4u;
        uint32_t ctas = 0;
        for (uint32_t k = 0; k < nb; ++k) {
            EQ_TRY(fill_desc(blocks[b0 + k], all.get() + (size_t)(b0 + k) * EQ_MAX_LAYERS, P.b[k], ctas));
            ctas += (P.b[k].n_chunks + kChunksPerCta - 1) / kChunksPerCta;
        }
        // blocks with zero chunks cannot exist (layers are non-empty); ctas > 0
        if (out_dtype == EQ_OUT_BF16)
            k_decode<true><<<ctas, kDecThreads, 0, st>>>(P);
        else
            k_decode<false><<<ctas, kDecThreads, 0, st>>>(P);
        EQ_CUDA_TRY(cudaGetLastError());
    }
    return EQ_OK;
}
