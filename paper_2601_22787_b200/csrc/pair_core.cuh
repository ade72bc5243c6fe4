// pair_core.cuh — device side of the EQ_CODEC_PAIR decoder (reading R15), shared by
// the stand-alone decoder (rans_dec.cu, k_decode_p: §8(a) rows a7 + a8) and the decode-fused
// GEMM (qmatmul.cu, §8(f) row 1).
//
// The pair codec is the word codec's rANS (R14: L = 2^16, 16-bit words, M = 2^12) over PAIRS
// of consecutive symbols of a chunk for the block's 15 most frequent codes, with an escape
// (the top slots of the pair table) followed by the two codes coded with the single table.
// Per decoded pair: one pair-LUT lookup, one codes-table lookup, at most one word.
//
// Table buffer of a block (u16[512], include/entquant.h): [0,256) single frequencies,
// [256,481) pair frequencies by ra·15 + rb, [481] escape frequency, [482] K, [484,492) the 16
// rank codes as bytes.  Per CTA the decoder builds in shared memory (kPairSmemBytes):
//   lut[4096]   pair LUT, entry id(ra, rb) | (slot − c) << 8 | (f − 1) << 20 (escape id 0xFF),
//   lut[4096..] the 256 × u16 codes table id -> code(ra) | code(rb) << 8 (right after the LUT:
//               its address is the LUT's uniform base + a constant — a separate array's address
//               was rematerialised with four uniform instructions per pair step),
//   lut1[4096]  the single table's symbol per slot (escapes); while the tables are built it
//               first holds pcum[227], the pair table's cumulative frequencies;
//   cum[257]    u16, the single table's cumulative frequencies.
#pragma once
#include "decode_core.cuh"



namespace eq {

constexpr int kPairOff = 256, kFescIdx = 481, kKIdx = 482, kRankIdx = 484;
constexpr uint32_t kEscId = 225;                  // LUT id of the escape slots (codes-table word 225)

// The escape's codes-table word (R18): a code pair no kept pair can decode to — (c, c) for the
// smallest code c that is not one of the block's K ≤ 15 ranked codes (a kept pair has ranked
// codes only; every byte is a possible Int8 code, so no fixed sentinel would do).
__device__ __forceinline__ uint32_t escape_codes(const uint16_t* freq) {
    const uint32_t K = min((uint32_t)freq[kKIdx], 15u);
    const uint8_t* rc = reinterpret_cast<const uint8_t*>(freq + kRankIdx);
    uint32_t c = 0;
    for (; c < 16; ++c) {
        bool ranked = false;
        for (uint32_t k = 0; k < K; ++k) ranked |= rc[k] == c;
        if (!ranked) break;
    }
    return c | (c << 8);
}
constexpr int kPairLutWords = kM + 113;           // + the 225 × u16 codes table
constexpr uint32_t kEscVals = 0xFFFFFFFFu;        // the escape's value word (bf16 NaN pair: never a grid value)


constexpr uint32_t kPairSmemBytes = kPairLutWords * 4 + kM + 258 * 2;
// one contiguous table region: [pair LUT | codes | lut1 | cum | (R18 bf16) values], so every
// table address is the LUT base plus a constant (one register across the decode loop)
constexpr uint32_t kLut1Off = kPairLutWords * 4;  // byte offsets from the LUT base
constexpr uint32_t kCumOff = kLut1Off + kM;
constexpr int kPairValWords = 226;                // (bf16 output of R18) the bf16x2 value table
constexpr uint32_t kValOff = kPairSmemBytes;

struct PairTab {
    uint32_t lut_s;        // shared address of the pair LUT (the codes table follows at + 4·kM)
    uint32_t esc_lo;       // slot << 20 at and above which a pair step is the escape (0xFFFFFFFF: none)
    uint32_t fesc, cesc;   // escape frequency and cumulative start
    uint32_t k2p20, k2p12; // 2^20, 2^12 passed at run time (IMAD forms on the FMA pipe)
    uint32_t k2p10;        // 2^10 (TOPID entries)
};

// the LUT entry's 8-bit id of rank pair (ra, rb), ra, rb < 15: a bijection onto [0, 225) in
// anti-diagonal order, so the frequent pairs (small ranks) get consecutive ids and their
// codes-table words fall in distinct banks (−10 % shared wavefronts vs row-major ids)
__device__ __forceinline__ uint32_t pair_id(uint32_t ra, uint32_t rb) {
    const uint32_t d = ra + rb;
    if (d <= 14) return d * (d + 1) / 2 + ra;
    const uint32_t e = 28 - d;
    return 225 - (e + 1) * (e + 2) / 2 + ra - (d - 14);
}

// the grid value of a code (E4M3, R1; or Int8) as bf16 bits — exact: ≤ 4 / 7 significant bits
__device__ __forceinline__ uint32_t grid_bf16(uint32_t code, bool i8) {
    float v;
    if (i8) {
        v = (float)(int8_t)code;
    } else {
        __half_raw h = __nv_cvt_fp8_to_halfraw((__nv_fp8_storage_t)code, __NV_E4M3);
        v = __half2float(*reinterpret_cast<__half*>(&h));
    }
    return __bfloat16_as_ushort(__float2bfloat16_rn(v));
}

// two bf16 products in one instruction, each the RNE of the exact product (subnormals kept):
// s·v has at most 8 + 7 significant bits, so this is the bf16 RNE of P:142's s·Q — the same
// single rounding as the f32 product followed by one RNE.  The +0 addend maps the product of
// code 0x80 (−0) to +0 as the oracle's dequantiser does (R3); a nonzero product is unchanged.
__device__ __forceinline__ uint32_t mul_bf16x2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("fma.rn.bf16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(0u));
    return d;
}

__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// word renormalisation (R14): at most one 16-bit word per step, prefetched into r.w
__device__ __forceinline__ void renorm_w(uint32_t& x, WordReader& r) {
    if (x < kLw) {
        x = __byte_perm(r.w, x, 0x5410);                                // (x << 16) | w
        r.w = lds_u16(r.ring | (r.Q & (kWRing - 1)));
        r.Q += 2;
    }
}

// a single-table symbol (escape path and odd tails): symbol per slot, then its cum entries
__device__ __forceinline__ uint32_t decode_single_p(uint32_t& x, WordReader& r, const PairTab& T) {
    uint32_t lo, xs;
    asm("{ .reg .u64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0, %1}, t; }" : "=r"(lo), "=r"(xs) : "r"(x), "r"(T.k2p20));
    const uint32_t slot = lo >> 20;
    const uint32_t s = lds_u8(T.lut_s + kLut1Off + slot);
    const uint32_t cs = lds_u16(T.lut_s + kCumOff + 2 * s), ce = lds_u16(T.lut_s + kCumOff + 2 * s + 2);
    x = (ce - cs) * xs + slot - cs;
    renorm_w(x, r);
    return s;
}

// one pair step; returns the two codes in the low 16 bits (first symbol in the low byte).
// NARROW: the LUT entry holds 2·id | (slot − c) << 9 | (f − 1) << 20 (every kept pair has f ≤ 2048,
// pair_tables_build decides per block), so the codes-table offset is one LOP3 (e & 0x1FE)
// instead of an add and a mask; otherwise id | (slot − c) << 8 | (f − 1) << 20.
template <bool NARROW = false>
__device__ __forceinline__ uint32_t decode_pair(uint32_t& x, WordReader& r, const PairTab& T, const uint8_t* payload) {
    uint32_t lo, xs;
    asm("{ .reg .u64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0, %1}, t; }" : "=r"(lo), "=r"(xs) : "r"(x), "r"(T.k2p20));
    if (lo >= T.esc_lo) {                          // escape: its step, then two singles
        x = T.fesc * xs + (lo >> 20) - T.cesc;
        renorm_w(x, r);
        ring_step_w(r, payload);                   // up to 2 more words follow: keep the ring ahead
        const uint32_t a = decode_single_p(x, r, T);
        const uint32_t b = decode_single_p(x, r, T);
        return a | (b << 8);
    }
    const uint32_t e = lds_u32(T.lut_s + (lo >> 18));
    const uint32_t fm1 = mad_hi(e, T.k2p12, 0u);                        // e >> 20
    if (NARROW) {
        x = mad_lo(fm1, xs, xs + (mad_lo(e, T.k2p12, 0u) >> 21));       // f·⌊x/M⌋ + slot − c
        renorm_w(x, r);
        return lds_u16(T.lut_s + 4 * kM + (e & 0x1FEu));                // 2·id -> codes
    }
    x = mad_lo(fm1, xs, xs + (mad_lo(e, T.k2p12, 0u) >> 20));           // f·⌊x/M⌋ + slot − c
    renorm_w(x, r);
    return lds_u16(T.lut_s + 4 * kM + ((e & 0xFFu) << 1));              // pair id -> codes
}

// one pair step of EQ_CODEC_PAIR_G (R18): no escape branch — an escape is decoded as the pair
// table's symbol it is (its LUT entry holds its f and slot − c) and yields the codes sentinel;
// `esc` accumulates "this group had an escape" (one ISETP with a predicate OR per step)
// VALS (bf16 output): the pair's two grid values as bf16x2 from the value table instead of the codes.
// TOPID (narrow tables built with TOPID): entries (f − 1) | (slot − c) << 11 | id << 24, so ONE
// 64-bit product e·2^10 yields 4·id (high word: the value table offset) and (slot − c) << 21.
template <bool NARROW = false, bool VALS = false, bool TOPID = false>
__device__ __forceinline__ uint32_t decode_pair_g(uint32_t& x, WordReader& r, const PairTab& T, bool& esc) {
    uint32_t lo, xs;
    asm("{ .reg .u64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0, %1}, t; }" : "=r"(lo), "=r"(xs) : "r"(x), "r"(T.k2p20));
    esc |= lo >= T.esc_lo;
    const uint32_t e = lds_u32(T.lut_s + (lo >> 18));
    if (TOPID && NARROW) {
        uint32_t lo2, id4;
        asm("{ .reg .u64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0, %1}, t; }" : "=r"(lo2), "=r"(id4) : "r"(e), "r"(T.k2p10));
        x = mad_lo(e & 0x7FFu, xs, xs + (lo2 >> 21));                  // f·⌊x/M⌋ + slot − c
        renorm_w(x, r);
        // (ptxas adds the table base with one IADD whatever the form: a 64-bit addend to the
        // product costs a carry chain, a link-time constant address is not folded into the LDS)
        if (VALS) return lds_u32(T.lut_s + kValOff + id4);
        return lds_u16(T.lut_s + 4 * kM + (id4 >> 1));
    }
    const uint32_t fm1 = mad_hi(e, T.k2p12, 0u);                        // e >> 20
    if (NARROW) {
        x = mad_lo(fm1, xs, xs + (mad_lo(e, T.k2p12, 0u) >> 21));       // f·⌊x/M⌋ + slot − c
        renorm_w(x, r);
        if (VALS) return lds_u32(T.lut_s + kValOff + ((e & 0x1FEu) << 1));
        return lds_u16(T.lut_s + 4 * kM + (e & 0x1FEu));
    }
    x = mad_lo(fm1, xs, xs + (mad_lo(e, T.k2p12, 0u) >> 20));
    renorm_w(x, r);
    if (VALS) return lds_u32(T.lut_s + kValOff + ((e & 0xFFu) << 2));
    return lds_u16(T.lut_s + 4 * kM + ((e & 0xFFu) << 1));
}

// escapes per group whose singles need no ring step (see patch_escapes)
#ifndef EQ_FREE_ESC
#define EQ_FREE_ESC ((kWRing - 32 - 16) / 4)
#endif
constexpr uint32_t kFreeEsc = EQ_FREE_ESC;

// R18 patch for the value words of a group (bf16 output): v[k] is pair position k's bf16x2
__device__ __forceinline__ void patch_escapes_vals(uint32_t* v, uint32_t& x, WordReader& r, const PairTab& T,
                                                   const uint8_t* payload, bool i8) {
    uint32_t n = 0;
    #pragma unroll
    for (uint32_t k = 0; k < 8; ++k) {
        if (v[k] == kEscVals) {
            if (n++ >= kFreeEsc) ring_step_w(r, payload);     // as patch_escapes
            const uint32_t a = decode_single_p(x, r, T);
            const uint32_t b = decode_single_p(x, r, T);
            v[k] = grid_bf16(a, i8) | (grid_bf16(b, i8) << 16);
        }
    }
}

// R18, after a group's pair steps (and the group's ring step): each escaped position (codes
// sentinel), in position order, is replaced by its two codes (a, then b) decoded with the
// single table.  q[0..3] hold the group's 8 pair positions, two per word (position k in the
// half k & 1 of q[k >> 1]); only positions < m are pair positions of the group.
// Staging: at a group's start more than 32 landed bytes lie ahead of the reader (the segment
// issued at a boundary starts > read + kWRing − 32, decode_core.cuh), the 8 pair steps take at
// most 16 of them, so the first kFreeEsc escapes' two words each need no new segment — and no
// cp.async wait, which would stall on the segment just issued at the boundary; from the next
// escape on, one ring step (stage + wait) per escape as before.
__device__ __forceinline__ void patch_escapes(uint32_t* q, uint32_t m, uint32_t& x, WordReader& r, const PairTab& T,
                                              const uint8_t* payload) {
    uint32_t n = 0;
    #pragma unroll
    for (uint32_t k = 0; k < 8; ++k) {
        const uint32_t sh = 16 * (k & 1);
        // (the sentinel is read from the codes table here, off the fast path: no register
        // held across the decode loop)
        if (k < m && ((q[k >> 1] >> sh) & 0xFFFFu) == lds_u16(T.lut_s + 4 * kM + 2 * kEscId)) {
            if (n++ >= kFreeEsc) ring_step_w(r, payload);     // up to 2 more words: keep the ring ahead
            const uint32_t a = decode_single_p(x, r, T);
            const uint32_t b = decode_single_p(x, r, T);
            q[k >> 1] = (q[k >> 1] & ~(0xFFFFu << sh)) | ((a | (b << 8)) << sh);
        }
    }
}

// lut[slot] = entry(slot, s) for the s with cm[s] <= slot < cm[s + 1] (cm[0..NS], cm[NS] = kM),
// NT threads: thread t fills slots [S·t, S·t + S), S = kM / NT, one binary search then a forward
// walk over the symbol boundaries (zero-width symbols are stepped over), 16-byte stores
template <int NS, int NT, class F>
__device__ __forceinline__ void lut_walk(uint32_t* lut, const uint32_t* cm, F entry) {
    constexpr uint32_t S = kM / NT;
    static_assert(S >= 4 && S * NT == kM, "slots per thread");
    const uint32_t s0 = S * (uint32_t)threadIdx.x;
    int lo = 0, hi = NS - 1;                       // largest s with cm[s] <= s0
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (cm[mid] <= s0) lo = mid; else hi = mid - 1;
    }
    uint4* dst = reinterpret_cast<uint4*>(lut + s0);
    #pragma unroll 1
    for (uint32_t k = 0; k < S; k += 4) {
        uint32_t v[4];
        #pragma unroll
        for (int u = 0; u < 4; ++u) {
            while (cm[lo + 1] <= s0 + k + u) ++lo;
            v[u] = entry(s0 + k + u, lo);
        }
        dst[k >> 2] = make_uint4(v[0], v[1], v[2], v[3]);
    }
}

// The block's tables (PairSmem) from its table buffer `freq`.  ALL threads of the CTA call it
// (it holds the barriers); threads t < NT (NT ≥ 64, a power of two ≤ 1024) do the work: the
// single cum by a block scan, the pair cum (226 entries: kept pairs in (ra, rb) order, then the
// escape) by warp 0, then the LUT walks and the codes table.  The caller waits for the table
// stores (a barrier) before decoding.  Returns 0 on every thread for a corrupt table
// (EQ_EF_CORRUPT set once), else 1 (LUT entries id | (slot − c) << 8 | (f − 1) << 20) or, with
// NARROW_OK and every kept pair's f ≤ 2048, 2 (entries 2·id | (slot − c) << 9 | (f − 1) << 20).
// (Only the rank-(0,0) pair can exceed 2048 slots, when p(rank 0)² > ½.)
// (This sequence keeps the table bases in uniform registers through the decode loop; a variant
// scanning both tables concurrently made ptxas rematerialise them per pair step, −1.6 %.)
// pcum lives in lut1's space (the pair LUT walk is done, behind a barrier of the NT threads,
// before lut1 is filled); cesc returns the escape's cumulative start pcum[225].
// VALS: also the bf16x2 value table (kPairValWords words after the codes table) of format i8;
// TOPID: narrow entries laid out (f − 1) | (slot − c) << 11 | id << 24 (decode_pair_g).
template <int NT, bool ALL = false, bool NARROW_OK = false, bool VALS = false, bool TOPID = false>
__device__ __forceinline__ uint32_t pair_tables_build(const uint16_t* freq, uint32_t* lut, uint8_t* lut1,
                                                      uint16_t* cum, uint32_t& cesc, uint32_t* err,
                                                      bool i8 = false) {
    uint32_t* pcum = reinterpret_cast<uint32_t*>(lut1);
    static_assert(NT >= 64 && (NT & (NT - 1)) == 0 && NT <= 1024, "thread count");
    const int t = threadIdx.x;
    {                                              // cum[257]: exclusive prefix of the 256 frequencies
        __shared__ uint32_t wsum[8];
        const int lane = t & 31, w = t >> 5;
        for (int base = 0; base < 256; base += NT) {
            if ((ALL || t < NT) && base + t < 256) {
                uint32_t v = freq[base + t];
                #pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
                    if (lane >= d) v += o;
                }
                if (lane == 31) wsum[(base >> 5) + w] = v;
                cum[base + t + 1] = v;             // warp-local inclusive prefix for now
            }
        }
        __syncthreads();
        for (int base = 0; base < 256; base += NT) {
            const int idx = base + t;
            if ((ALL || t < NT) && idx < 256) {
                uint32_t add = 0;
                for (int q = 0; q < (idx >> 5); ++q) add += wsum[q];
                cum[idx + 1] += add;
            }
        }
        if (t == 0) cum[0] = 0;
    }
    __syncthreads();
    if (cum[256] != kM) {
        if (t == 0) atomicOr(err, EQ_EF_CORRUPT);
        return 0;
    }
    const uint32_t K = freq[kKIdx];
    __shared__ uint32_t s_fmax, s_cesc;
    if (t < 32) {                                  // 226-entry pair cum: (ra, rb) order, escape last
        uint32_t v[8], s = 0, fmax = 0;
        #pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int q = t * 8 + j;
            v[j] = (q < 225 && (uint32_t)(q / 15) < K && (uint32_t)(q % 15) < K) ? freq[kPairOff + q] : 0u;
            s += v[j];
            fmax = max(fmax, v[j]);
        }
        fmax = __reduce_max_sync(0xFFFFFFFFu, fmax);
        if (t == 0) s_fmax = fmax;
        uint32_t inc = s;
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
            if (t >= d) inc += o;
        }
        uint32_t run = inc - s;
        #pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int q = t * 8 + j;
            if (q < 225) pcum[q] = run;
            run += v[j];
        }
        if (t == 31) {
            pcum[225] = inc;
            pcum[226] = inc + freq[kFescIdx];
            s_cesc = inc;
        }
    }
    __syncthreads();
    if (pcum[226] != kM || K > 15) {
        if (t == 0) atomicOr(err, EQ_EF_CORRUPT);
        return 0;
    }
    const bool narrow = NARROW_OK && s_fmax <= 2048u && pcum[226] - pcum[225] <= 2048u;
    cesc = s_cesc;
    if (ALL || t < NT) {
        // escape slots: an ordinary entry (slot − c, f − 1) with id kEscId, whose codes-table
        // word is the sentinel escape_codes() and value word kEscVals.  R15 tests
        // for the escape before the lookup; R18 takes the step like any pair and patches later.
        const uint32_t idsh = narrow ? 1u : 0u, scsh = narrow ? 9u : 8u;
        lut_walk<226, NT>(lut, pcum, [&](uint32_t slot, int q) -> uint32_t {
            const uint32_t f = pcum[q + 1] - pcum[q];
            const uint32_t id = q < 225 ? pair_id((uint32_t)q / 15, (uint32_t)q % 15) : kEscId;
            if (TOPID && narrow) return (f - 1) | ((slot - pcum[q]) << 11) | (id << 24);
            return (id << idsh) | ((slot - pcum[q]) << scsh) | ((f - 1) << 20);
        });
        asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");     // pcum read by all: lut1 may be written
        constexpr uint32_t SP = kM / NT;           // symbol per slot: thread t fills [SP·t, SP·t + SP)
        const uint32_t s0 = SP * (uint32_t)t;
        int lo = 0, hi = 255;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (cum[mid] <= s0) lo = mid; else hi = mid - 1;
        }
        #pragma unroll
        for (uint32_t k4 = 0; k4 < SP; k4 += 4) {
            uint32_t w = 0;
            #pragma unroll
            for (uint32_t k = 0; k < 4; ++k) {
                while (cum[lo + 1] <= s0 + k4 + k) ++lo;
                w |= (uint32_t)lo << (8 * k);
            }
            *reinterpret_cast<uint32_t*>(lut1 + s0 + k4) = w;
        }
        const uint8_t* rcb = reinterpret_cast<const uint8_t*>(freq + kRankIdx);
        uint16_t* ctab = reinterpret_cast<uint16_t*>(lut + kM);
        for (int q = t; q < 225; q += NT)
            ctab[pair_id((uint32_t)q / 15, (uint32_t)q % 15)] = (uint16_t)(rcb[q / 15] | (rcb[q % 15] << 8));
        if (t == 0) ctab[kEscId] = (uint16_t)escape_codes(freq);
        if (VALS) {
            uint32_t* vtab = lut + kValOff / 4;
            for (int q = t; q < 225; q += NT)
                vtab[pair_id((uint32_t)q / 15, (uint32_t)q % 15)] = grid_bf16(rcb[q / 15], i8) | (grid_bf16(rcb[q % 15], i8) << 16);
            if (t == 0) vtab[kEscId] = kEscVals;
        }
    }
    return narrow ? 2u : 1u;
}

__device__ __forceinline__ PairTab pair_tab(const uint16_t* freq, const uint32_t* lut, const uint8_t* lut1,
                                            const uint16_t* cum, uint32_t cesc, uint32_t k2p20, uint32_t k2p12) {
    PairTab T;
    T.lut_s = (uint32_t)__cvta_generic_to_shared(lut);
    T.fesc = freq[kFescIdx];
    T.cesc = cesc;
    T.esc_lo = T.fesc ? (T.cesc << 20) : 0xFFFFFFFFu;
    T.k2p20 = k2p20;
    T.k2p12 = k2p12;
    T.k2p10 = k2p12 >> 2;
    return T;
}

}  // namespace eq
