// decode_core.cuh — device-side rANS decode machinery shared by the stand-alone decoder
// (rans_dec.cu, §8(a) rows a7+a8) and the decode-fused tcgen05 GEMM (qmatmul.cu, Alg. 2 l.3).
// See rans_dec.cu for the design notes; all functions are branch-free per lane.
#pragma once
#include "common.cuh"

namespace eq {

#ifndef EQ_K_FLO
#define EQ_K_FLO 1
#endif
constexpr int kRingWords = 16;      // 64-byte per-chunk staging ring (cp.async segments)

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
#define EQ_ZFAST 0       // 1: the old code-0x00 bypass with the (f−1)-in-bits-8-19 LUT layout (slower)
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
    const uint32_t* lutp;  // the LUT (shared array; EQ_WADDR = 1 addressing)
    uint32_t zlim;         // lut_s + 4·f0: LUT addresses below it belong to code 0x00
    uint32_t zk;           // (f0 − 1) << 20 − 64·lut_s: entry of code 0x00 = 64·address + zk
    uint32_t k64;          // 64 (runtime, keeps the IMAD on the FMA pipe)
    uint32_t k2p16;        // 2^16 (runtime, EQ_WMERGE = 1)
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
    const uint32_t fm1 = mad_hi(mad_lo(e, T.k2p12, 0u), T.k2p12, 0u);   // (e >> 8) & 0xFFF
    x = mad_lo(fm1, xs, xs + (e >> 20));                                // f·⌊x/M⌋ + slot − c
#else
    // as decode_one_w: one IMAD.WIDE x·2^20 gives x >> 12 and slot << 20, LEA.HI the LUT
    // address; entry layout sym | (slot − c) << 8 | (f − 1) << 20 (build_lut<1>), so one
    // IMAD.WIDE e·2^12 gives f − 1 and (slot − c) << 20
    uint32_t lo, xs;
    asm("{ .reg .u64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0, %1}, t; }" : "=r"(lo), "=r"(xs) : "r"(x), "r"(T.k2p20));
    const uint32_t e = lds_u32(T.lut_s + (lo >> 18));
    const uint32_t fm1 = mad_hi(e, T.k2p12, 0u);                        // e >> 20
    x = mad_lo(fm1, xs, xs + (mad_lo(e, T.k2p12, 0u) >> 20));           // f·⌊x/M⌋ + slot − c
#endif
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
#ifndef EQ_STPOL
#define EQ_STPOL 2       // output store L2 policy: 0 default, 1 evict_last hint, 2 evict_first hint (default:
                         // decoded lines leave L2 first, the compressed input stays — DRAM reads 4.55 → 2.37 GB)
#endif
__device__ __forceinline__ void st_out32(void* p, uint4 a, uint4 b) {
#if EQ_ST256 && EQ_STPOL == 2
    // evict-first in L2 as an instruction qualifier (STG.E.NA.EFL2): no policy register
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
                 : "memory");
#elif EQ_ST256 && EQ_STPOL
    uint64_t pol;
    if (EQ_STPOL == 1) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    else asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8}, %9;" ::"l"(p),
                 "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w), "l"(pol)
                 : "memory");
#elif EQ_ST256 && EQ_L2HINT
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
template <class C>
__device__ __forceinline__ void store16_bf16_at(C& c, const uint32_t q[4], uint8_t* dst);

// 16 symbols -> bf16 with one row scale (cols % 16 == 0), 32-byte store
template <class C>
__device__ __forceinline__ void store16_bf16(C& c, const uint32_t q[4]) {
    store16_bf16_at(c, q, c.out + (uint64_t)c.i * 2);
}

template <class C>
__device__ __forceinline__ void store16_bf16_at(C& c, const uint32_t q[4], uint8_t* dst) {
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

// ================================================================ EQ_CODEC_WORD (R14)
// 16-bit renormalisation: after a decode step at most ONE word is needed (x ≥ 16 always,
// and (x << 16) ≥ 2^20 ≥ L), so the lane keeps no bit window: it holds the next unconsumed
// word `w` in a register (prefetched from its shared-memory ring as soon as the previous one
// is consumed, off the state's dependency chain) and renormalises with one predicated PRMT.
// Per-chunk staging ring: 64 bytes, filled 16 bytes at a time by cp.async.  Schedule: at
// most one 16-byte segment per 8-step boundary (a lane consumes at most 8 words = 16 bytes
// per 8 steps, so the stage front keeps pace; right after the initial fill it may trail
// its target by one segment, never more).  Every staged segment then starts > q + 16 when
// issued, the next 8 steps read only [q, q + 18), so waiting for all groups at each boundary
// (before issuing) never waits for data issued at that boundary.
// (Measured alternatives: a 128-byte ring with 3 groups in flight — 4 instead of 6 CTAs/SM,
// −4 %; whole 32-byte sectors every 16 steps — the 2-slot ring then has to wait for the
// sector it just issued, −10 %.)
#ifndef EQ_WRING
#define EQ_WRING 64      // bytes per lane (64 for the throughput-bound stand-alone decoders; the fused
                         // GEMM, latency-bound with few resident chains, stages further ahead)
#endif
constexpr uint32_t kWRing = EQ_WRING;
static_assert(kWRing == 64 || kWRing == 128 || kWRing == 256, "ring size");
// Ring addressing: payload byte p lives at ring | ((p + kWBias) & 63), and the reader keeps
// Q = (payload offset of the next word) + kWBias, so a word address is one LOP3 and the test
// "slot of segment gn is free" (all bytes < gn − 48 consumed: gn ≤ q + 48) is gn ≤ Q.
constexpr uint32_t kWBias = kWRing - 16;
// A segment issued at a boundary starts > (read offset) + kWRing − 32 (the stage front keeps pace:
// ≤ 16 bytes consumed and ≤ one segment staged per boundary) and the steps after a boundary
// read < 18 bytes ahead, so it is first needed kWRing/16 − 3 boundaries later: that many newer
// groups may stay in flight (64-byte ring: 1, 128: 5).
constexpr int kWWaitGroups = (int)(kWRing / 16) - 3;

struct WordReader {
    uint32_t Q;            // payload byte offset of the next word to load into w, + kWBias
    uint32_t w;            // the next unconsumed 16-bit word (low half)
    uint32_t gn;           // payload byte offset of the next 16-byte segment to stage
    uint32_t ring;         // shared address of this chunk's ring (64-byte aligned)
};

__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u16 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// initial fill: one 16-byte segment (g multiple of 16) into its slot
__device__ __forceinline__ void stage_segment_w(uint32_t ring, const uint8_t* payload, uint32_t g) {
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(ring | ((g + kWBias) & (kWRing - 1))),
                 "l"(payload + g));
}

// Every 8 steps: wait for all staged segments, then stage segment gn if its slot is free
// (predicated, no branch), one cp.async group per boundary.
#ifndef EQ_RING_ISSUE_FIRST
#define EQ_RING_ISSUE_FIRST 1   // stage, commit, then wait for all but the newest group (same data
                                // guarantee as wait-all-then-stage: the segment issued at this
                                // boundary is never read before the next one); avoids the LDGDEPBAR
                                // of wait_all and the dummy LDS ptxas pads between DEPBAR and LDGSTS
#endif
__device__ __forceinline__ void ring_step_w(WordReader& r, const uint8_t* payload) {
#if EQ_RING_ISSUE_FIRST
    asm volatile("{ .reg .pred p; setp.le.u32 p, %0, %1;\n\t"
                 "@p cp.async.cg.shared.global.L2::128B [%2], [%3], 16;\n\t"
                 "@p add.u32 %0, %0, 16; }\n\t"
                 "cp.async.commit_group;\n\t"
                 "cp.async.wait_group %4;"
                 : "+r"(r.gn) : "r"(r.Q), "r"(r.ring | ((r.gn + kWBias) & (kWRing - 1))), "l"(payload + r.gn),
                   "n"(kWWaitGroups)
                 : "memory");
#else
    asm volatile("cp.async.wait_all;\n\t"
                 "{ .reg .pred p; setp.le.u32 p, %0, %1;\n\t"
                 "@p cp.async.cg.shared.global.L2::128B [%2], [%3], 16;\n\t"
                 "@p add.u32 %0, %0, 16; }\n\t"
                 "cp.async.commit_group;"
                 : "+r"(r.gn) : "r"(r.Q), "r"(r.ring | ((r.gn + kWBias) & (kWRing - 1))), "l"(payload + r.gn)
                 : "memory");
#endif
}

#ifndef EQ_WMERGE
#define EQ_WMERGE 0      // renormalisation merge: 0 = PRMT (ALU pipe), 1 = IMAD (FMA pipe)
#endif
#ifndef EQ_WZERO
#define EQ_WZERO 0       // 1: code 0x00 decoded without the shared-memory LUT (measured slower)
#endif
#ifndef EQ_WADDR
#define EQ_WADDR 2       // LUT address: 0 = 4x − 2^14·xs + base (IMAD.HI + 2 IMADs),
                         // 2 = IMAD.WIDE x·2^20 (xs and slot together) + LEA.HI
#endif
#ifndef EQ_WENTRY
#define EQ_WENTRY 1      // LUT entry layout of build_lut<EQ_WENTRY> (0: f−1 in bits 8-19, 1: in 20-31)
#endif
// One rANS decode step (Alg. 2 l.1) with word renormalisation; returns the LUT entry
// (symbol in the low byte).  State update with IMAD / IMAD.HI / LEA.HI forms; then
// if x < 2^16: x = (x << 16) | w as one PRMT, and the next word is prefetched.
__device__ __forceinline__ uint32_t decode_one_w(uint32_t& x, WordReader& r, const DecTable& T) {
#if EQ_WADDR == 2
    // one IMAD.WIDE: x·2^20 = (x >> 12) : (slot << 20); LUT address = base + (lo >> 18) (LEA.HI)
    uint32_t lo, xs;
    asm("{ .reg .u64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0, %1}, t; }" : "=r"(lo), "=r"(xs) : "r"(x), "r"(T.k2p20));
    const uint32_t la = T.lut_s + (lo >> 18);
#else
    const uint32_t xs = mad_hi(x, T.k2p20, 0u);                         // x >> 12
    const uint32_t la = mad_lo(x, T.k4, mad_lo(xs, T.kneg2p14, T.lut_s));
#endif
#if EQ_WZERO
    // code 0x00 (cum 0, the most frequent symbol) owns slots [0, f0): its entry
    // (f0−1) << 20 | slot << 8 is computed, so only the other lanes access shared memory
    // (fewer random-slot bank conflicts per warp-wide lookup)
    uint32_t e;
    if (la < T.zlim) e = la * 64u + T.zk;
    else e = lds_u32(la);
#else
    const uint32_t e = lds_u32(la);
#endif
#if EQ_WENTRY
    const uint32_t fm1 = mad_hi(e, T.k2p12, 0u);                        // e >> 20
    x = mad_lo(fm1, xs, xs + (mad_lo(e, T.k2p12, 0u) >> 20));           // f·⌊x/M⌋ + slot − c
#else
    const uint32_t fm1 = mad_hi(mad_lo(e, T.k2p12, 0u), T.k2p12, 0u);   // (e >> 8) & 0xFFF
    x = mad_lo(fm1, xs, xs + (e >> 20));                                // f·⌊x/M⌋ + slot − c (LEA.HI)
#endif
    if (x < kLw) {
#if EQ_WMERGE
        x = mad_lo(x, T.k2p16, r.w);                                    // (x << 16) | w (FMA pipe)
#else
        x = __byte_perm(r.w, x, 0x5410);                                // (x << 16) | w (one PRMT)
#endif
        r.w = lds_u16(r.ring | (r.Q & (kWRing - 1)));
        r.Q += 2;
    }
    return e;
}

struct ChainW {
    uint32_t x;
    WordReader r;
    uint8_t* out;
    const uint16_t* sc;
    uint32_t row, col, cols;
    float s;
    uint16_t s16;
    bool i8;
    uint32_t n, i;
    uint32_t a, e;         // chunk payload byte range [a, e)
    uint32_t gs;           // layer positions between the chunk's 16-symbol groups: 16, or 512 (R17)
    bool active, runaway, fast;
};

// 4 symbols -> one word of codes (first symbol in the low byte)
__device__ __forceinline__ uint32_t decode4_w(ChainW& c, const DecTable& T) {
    const uint32_t a = decode_one_w(c.x, c.r, T);
    const uint32_t b = decode_one_w(c.x, c.r, T);
    const uint32_t d = decode_one_w(c.x, c.r, T);
    const uint32_t f = decode_one_w(c.x, c.r, T);
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(d, f, 0x0040), 0x5410);
}

}  // namespace eq
