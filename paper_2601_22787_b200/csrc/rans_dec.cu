// rans_dec.cu — §8(a) rows a7 + a8: chunk-parallel rANS decode (byte or 16-bit-word
// renormalisation, R9 / R14) of E4M3 symbol
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
#include "decode_core.cuh"
#include "pair_core.cuh"

#include <algorithm>
#include <cstring>
#include <memory>

namespace eq {

#ifndef EQ_DEC_CHAINS
#define EQ_DEC_CHAINS 1
#endif
constexpr int kChunksPerCta = 256;
constexpr int kChains = EQ_DEC_CHAINS;            // independent chunks per thread (ILP)
constexpr int kDecThreads = kChunksPerCta / kChains;
constexpr int kMaxDecBlocks = 48;

struct DecLayer {
    uint64_t out_off;      // byte offset of the layer in the arena
    ChunkGeom geom;        // chunking segment (layer or row, EQ_CHUNK_*) and chunks per segment
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
    uint32_t codec;        // EQ_CODEC_BYTE | EQ_CODEC_WORD | EQ_CODEC_PAIR (one per launch)
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
    uint32_t k2p20, k2p12, kneg2p14, k4, k64, k2p16;
    DecBlock b[kMaxDecBlocks];
};

// The block's decode LUT in shared memory from its 256 frequencies (all kDecThreads threads
// call it): exclusive prefix cum[257], then per slot the largest s with cum[s] ≤ slot,
// entry = s | (f_s − 1) << 8 | (slot − cum[s]) << 20 (LAYOUT 0) or
//         s | (slot − cum[s]) << 8 | (f_s − 1) << 20 (LAYOUT 1, decode_one_w).
// Returns false (EQ_EF_CORRUPT set once) if the frequencies do not sum to M.
// cum[257] = exclusive prefix of the block's 256 single-symbol frequencies (all NT threads);
// false (EQ_EF_CORRUPT set once) if they do not sum to M
template <int NT>
__device__ __forceinline__ bool build_cum(const DecBlock& B, uint32_t* cum, uint32_t* err) {
    static_assert(NT >= 256 || 256 % NT == 0, "thread count");
    const int t = threadIdx.x;
    {
        __shared__ uint32_t wsum[8];
        const int lane = t & 31, w = t >> 5;
        for (int base = 0; base < 256; base += NT) {
            if (base + t < 256) {
                uint32_t v = B.freq[base + t];
                #pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    uint32_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
                    if (lane >= d) v += o;
                }
                if (lane == 31) wsum[(base >> 5) + w] = v;
                cum[base + t + 1] = v;              // warp-local inclusive prefix for now
            }
        }
        __syncthreads();
        for (int base = 0; base < 256; base += NT) {
            const int idx = base + t;
            if (idx < 256) {
                uint32_t add = 0;
                for (int q = 0; q < (idx >> 5); ++q) add += wsum[q];
                cum[idx + 1] += add;
            }
        }
        if (t == 0) cum[0] = 0;
    }
    __syncthreads();
    if (cum[256] != kM) {                     // corrupt table: nothing decodable
        if (t == 0) atomicOr(err, EQ_EF_CORRUPT);
        return false;
    }
    return true;
}

template <int LAYOUT = 0, int NT = kDecThreads>
__device__ __forceinline__ bool build_lut(const DecBlock& B, uint32_t* lut, uint32_t* cum, uint32_t* err) {
    const int t = threadIdx.x;
    if (!build_cum<NT>(B, cum, err)) return false;
    auto entry = [&](uint32_t slot, int sym) -> uint32_t {
        const uint32_t fs = cum[sym + 1] - cum[sym];
        return LAYOUT == 0 ? ((uint32_t)sym | ((fs - 1) << 8) | ((slot - cum[sym]) << 20))
                           : ((uint32_t)sym | ((slot - cum[sym]) << 8) | ((fs - 1) << 20));
    };
    if (NT == 256) {
        // thread t fills slots [16t, 16t + 16): one binary search for the first slot's
        // symbol, then a forward walk over the symbol boundaries; 4 × 16-byte stores
        const uint32_t s0 = 16u * (uint32_t)t;
        int lo = 0, hi = 255;                  // largest s with cum[s] <= s0
        while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (cum[mid] <= s0) lo = mid; else hi = mid - 1;
        }
        uint4* dst = reinterpret_cast<uint4*>(lut + s0);
        #pragma unroll 1
        for (int k = 0; k < 16; k += 4) {            // 4 entries per 16-byte store (few live registers)
            uint32_t v[4];
            #pragma unroll
            for (int u = 0; u < 4; ++u) {
                while (cum[lo + 1] <= s0 + k + u) ++lo;
                v[u] = entry(s0 + k + u, lo);
            }
            dst[k >> 2] = make_uint4(v[0], v[1], v[2], v[3]);
        }
    } else {
        for (int slot = t; slot < (int)kM; slot += NT) {
            int lo = 0, hi = 255;              // largest s with cum[s] <= slot
            while (lo < hi) {
                int mid = (lo + hi + 1) >> 1;
                if (cum[mid] <= (uint32_t)slot) lo = mid; else hi = mid - 1;
            }
            lut[slot] = entry((uint32_t)slot, lo);
        }
    }
    return true;
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
    const uint64_t sym0 = chunk_start(Ly.geom, B.cs, chunk - Ly.chunk0, c.n);
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
    // 16 / 32-symbol groups with 32-byte stores need a 32-byte aligned chunk start (row chunks
    // start at row·cols + j·cs) and whole groups per row (bf16: one scale per group)
    c.fast = BF16 ? ((Ly.cols & 15) == 0 && ((sym0 | B.cs) & 15) == 0) : (((sym0 | B.cs) & 31) == 0);
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
    __shared__ __align__(16) uint32_t lut[kM];
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
    if (!build_lut<EQ_ZFAST ? 0 : 1>(B, lut, cum, P.err)) {
        stage_wait_all();
        return;
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


// ================================================================ EQ_CODEC_WORD decoder
// Same CTA/lane mapping, LUT and stores as k_decode; per lane a 128-byte (kWRing) staging
// ring, and word renormalisation (decode_one_w): no bit window, no per-pair refill.
template <bool BF16>
__device__ __forceinline__ void chain_setup_w(ChainW& c, const DecBlock& B, uint32_t chunk, uint32_t ring,
                                              uint8_t* arena, uint32_t* err) {
    c.active = chunk < B.n_chunks;
    c.runaway = false;
    c.i = 0;
    c.n = 0;
    if (!c.active) return;
    uint32_t l = 0;
    while (l + 1 < B.n_layers && chunk >= B.layer[l + 1].chunk0) ++l;
    const DecLayer& Ly = B.layer[l];
    const uint64_t sym0 = chunk_start(Ly.geom, B.cs, chunk - Ly.chunk0, c.n, &c.gs);
    const uint32_t a = __ldg(B.off + chunk), e = __ldg(B.off + chunk + 1);
    if (e < a || (uint64_t)e > B.payload_bytes || e - a < 4) {
        atomicOr(err, EQ_EF_TRUNCATED);
        c.active = false;
        return;
    }
    c.a = a;
    c.e = e;
    c.r.ring = ring;
    const uint32_t g0 = a & ~15u;
    #pragma unroll
    for (uint32_t q = 0; q < kWRing / 16; ++q) stage_segment_w(ring, B.payload, g0 + 16 * q);
    c.r.gn = g0 + kWRing;
    c.out = arena + Ly.out_off + sym0 * (BF16 ? 2 : 1);
    c.sc = B.scales + Ly.scale_off;
    c.cols = Ly.cols;
    c.row = (uint32_t)(sym0 / Ly.cols);
    c.col = (uint32_t)(sym0 % Ly.cols);
    c.s = BF16 ? bf16_bits_to_float(c.sc[c.row]) : 0.f;
    c.i8 = B.format == EQ_FMT_INT8;
    c.s16 = (BF16 && !c.i8) ? scale_f16(c.s) : 0;
    // 16 / 32-symbol groups with 32-byte stores need a 32-byte aligned chunk start (row chunks
    // start at row·cols + j·cs) and whole groups per row (bf16: one scale per group)
    c.fast = BF16 ? ((Ly.cols & 15) == 0 && ((sym0 | B.cs) & 15) == 0) : (((sym0 | B.cs) & 31) == 0);
    if (c.gs != kIlGroup) c.fast = true;           // R17 chunk: cs % 32 == 0, cols % 16 == 0 (validated)
}

// after the initial segments landed: 4-byte little-endian state, then the first word
__device__ __forceinline__ void chain_start_w(ChainW& c) {
    if (!c.active) return;
    const uint32_t m = kWRing - 1, A = c.a + kWBias;
    c.x = lds_u16(c.r.ring | (A & m)) | (lds_u16(c.r.ring | ((A + 2) & m)) << 16);
    c.r.w = lds_u16(c.r.ring | ((A + 4) & m));
    c.r.Q = A + 6;
}


template <bool BF16>
__device__ __forceinline__ void chain_finish_w(ChainW& c, const uint8_t* payload, const DecTable& T) {
    if (!c.active || c.runaway) return;
    if (c.fast) {
        const uint32_t G = BF16 ? 16 : 32;
        while (c.i + G <= c.n) {
            if (BF16) {
                uint32_t q[4];
                q[0] = decode4_w(c, T);
                q[1] = decode4_w(c, T);
                ring_step_w(c.r, payload);
                q[2] = decode4_w(c, T);
                q[3] = decode4_w(c, T);
                ring_step_w(c.r, payload);
                store16_bf16(c, q);
            } else {
                uint32_t q[8];
                #pragma unroll
                for (int k = 0; k < 8; ++k) {
                    q[k] = decode4_w(c, T);
                    if (k & 1) ring_step_w(c.r, payload);
                }
                st_out32(c.out + c.i, make_uint4(q[0], q[1], q[2], q[3]), make_uint4(q[4], q[5], q[6], q[7]));
            }
            c.i += G;
            if (c.r.Q > c.e + (2 + kWBias)) { c.runaway = true; return; }
        }
    }
    for (; c.i < c.n; ++c.i) {                  // generic / ragged tail: one symbol at a time
        const uint32_t sym = decode_one_w(c.x, c.r, T) & 0xFFu;
        if ((c.i & 7) == 7) ring_step_w(c.r, payload);
        store_one<BF16>(c.out, c.i, sym, c.s, c.i8);
        if (BF16 && ++c.col == c.cols) {
            c.col = 0;
            ++c.row;
            if (c.i + 1 < c.n) c.s = bf16_bits_to_float(c.sc[c.row]);
        }
        if (c.r.Q > c.e + (2 + kWBias)) { c.runaway = true; return; }
    }
}

#ifndef EQ_WTHREADS
#define EQ_WTHREADS 256             // chunks (= threads) per CTA of k_decode_w
#endif
#ifndef EQ_DECW_MIN_CTAS
#define EQ_DECW_MIN_CTAS 6          // 40 registers; 6 × (16 KB ring + 17 KB LUT) of shared memory
#endif
constexpr int kWThreads = EQ_WTHREADS;
constexpr int kWChains = 1;         // chunks per thread (2, interleaved for ILP, measured slower)
constexpr int kWChunksPerCta = kWThreads * kWChains;
constexpr uint32_t kDecWSmem = kWChunksPerCta * kWRing;     // dynamic: the staging rings

template <bool BF16>
__global__ void __launch_bounds__(kWThreads, EQ_DECW_MIN_CTAS)
k_decode_w(const __grid_constant__ DecParams P) {
    extern __shared__ __align__(128) uint8_t rings[];      // kWChunksPerCta × kWRing
    __shared__ __align__(16) uint32_t lut[kM];
    __shared__ uint32_t cum[257];

    uint32_t bi = 0;
    while (bi + 1 < P.n_blocks && blockIdx.x >= P.b[bi + 1].cta0) ++bi;
    const DecBlock& B = P.b[bi];
    const int t = threadIdx.x;

    ChainW ch[kWChains];        // setup first: the initial cp.async copies overlap the table build
    #pragma unroll
    for (int j = 0; j < kWChains; ++j) {
        const uint32_t slot = (uint32_t)(j * kWThreads + t);
        chain_setup_w<BF16>(ch[j], B, (blockIdx.x - B.cta0) * kWChunksPerCta + slot,
                            (uint32_t)__cvta_generic_to_shared(rings + slot * kWRing), P.arena, P.err);
    }
    stage_commit();
    if (!build_lut<EQ_WENTRY, kWThreads>(B, lut, cum, P.err)) {
        stage_wait_all();
        return;
    }
    stage_wait_all();
    __syncthreads();
    DecTable T;
    T.k2p20 = P.k2p20;
    T.k2p12 = P.k2p12;
    T.kneg2p14 = P.kneg2p14;
    T.k4 = P.k4;
    T.lut_s = (uint32_t)__cvta_generic_to_shared(lut);
    T.lutp = lut;
    T.f0 = cum[1];
    T.ez = (T.f0 - 1) << 8;
    T.zlim = T.lut_s + 4u * T.f0;
    T.zk = ((T.f0 - 1) << 20) - 64u * T.lut_s;
    T.k64 = P.k64;
    T.k2p16 = P.k2p16;

    #pragma unroll
    for (int j = 0; j < kWChains; ++j) chain_start_w(ch[j]);
    // each chain (one per thread) to its end: 16-symbol groups, then a ragged tail
    #pragma unroll
    for (int j = 0; j < kWChains; ++j) {
        if (ch[j].active && ch[j].r.Q > ch[j].e + (2 + kWBias)) ch[j].runaway = true;
        chain_finish_w<BF16>(ch[j], B.payload, T);
    }
    stage_wait_all();
    // integrity: final state L and every payload byte of the chunk consumed exactly
    #pragma unroll
    for (int j = 0; j < kWChains; ++j) {
        const ChainW& c = ch[j];
        if (c.active && (c.runaway || c.x != kLw || c.r.Q - (2u + kWBias) != c.e)) atomicOr(P.err, EQ_EF_CORRUPT);
    }
}


// ================================================================ EQ_CODEC_PAIR decoder (R15)
// Same CTA ↔ block and lane ↔ chunk mapping and staging as k_decode_w; the pair tables and the
// pair / single decode steps are in pair_core.cuh (shared with the fused GEMM).
#ifndef EQ_PAIR_VALS
#define EQ_PAIR_VALS 1              // R18 bf16: a bf16x2 value table (one HFMA2 per pair) instead of the codes
#endif
#ifndef EQ_PAIR_TOPID
#define EQ_PAIR_TOPID 1             // R18 bf16 values: narrow entries with the id on top (decode_pair_g)
#endif
// R18 (EQ_CODEC_PAIR_G) generic path: one group of len ≤ 16 symbols — its pair steps, the
// escaped pairs' codes, its odd last symbol — stored one symbol at a time (ragged tails and
// chunks without the 32-byte group stores; contiguous positions)
template <bool BF16, bool NARROW, bool TOPID>
__device__ __forceinline__ void group_generic_g(ChainW& c, const uint8_t* payload, const PairTab& T, uint32_t len) {
    const uint32_t m = len >> 1;
    uint32_t q[4] = {0u, 0u, 0u, 0u};
    bool esc = false;
    #pragma unroll
    for (uint32_t k = 0; k < 8; ++k) {
        if (k < m) {
            q[k >> 1] |= decode_pair_g<NARROW, false, TOPID>(c.x, c.r, T, esc) << (16 * (k & 1));
            if ((k & 3) == 3) ring_step_w(c.r, payload);
        }
    }
    if (esc) patch_escapes(q, m, c.x, c.r, T, payload);
    uint32_t last = 0;
    if (len & 1) {
        ring_step_w(c.r, payload);
        last = decode_single_p(c.x, c.r, T);
    }
    #pragma unroll
    for (uint32_t h = 0; h < 16; ++h) {
        if (h >= len) break;
        const uint32_t sym = h < 2 * m ? (q[h >> 2] >> (8 * (h & 3))) & 0xFFu : last;
        store_one<BF16>(c.out, c.i + h, sym, c.s, c.i8);
        if (BF16 && ++c.col == c.cols) {
            c.col = 0;
            ++c.row;
            if (c.i + h + 1 < c.n) c.s = bf16_bits_to_float(c.sc[c.row]);
        }
    }
    c.i += len;
}

template <bool BF16, bool NARROW, bool GROUPED>
__device__ __forceinline__ void chain_finish_p(ChainW& c, const uint8_t* payload, const PairTab& T) {
    if (!c.active || c.runaway) return;
    const uint32_t qlim = c.e + (2 + kWBias);
    if (c.fast) {
        // group loop with a down-counter and a running 32-byte output pointer; the runaway test
        // shares the loop test; the f16-scale dequant (the usual case) is tested first
        constexpr uint32_t G = BF16 ? 16 : 32;
        const uint32_t ng0 = (c.n - c.i) / G;
        const bool tail = c.i + ng0 * G < c.n;     // symbols after the groups (they need the row's scale)
        uint32_t ng = ng0;
        uint8_t* o = c.out + (uint64_t)c.i * (BF16 ? 2 : 1);
        uint32_t s16 = c.i8 ? 0u : (uint32_t)c.s16;
        constexpr bool VALS = BF16 && GROUPED && EQ_PAIR_VALS;
        uint32_t s2 = VALS ? c.sc[c.row] * 0x10001u : 0u;     // the row's bf16 scale, twice
        while (ng != 0 && c.r.Q <= qlim) {
            if (VALS) {                            // R18 + bf16: value words, one bf16x2 product per pair
                uint32_t v[8];
                bool esc = false;
                #pragma unroll
                for (int k = 0; k < 8; ++k) v[k] = decode_pair_g<NARROW, true, EQ_PAIR_TOPID>(c.x, c.r, T, esc);
                ring_step_w(c.r, payload);
                if (esc) patch_escapes_vals(v, c.x, c.r, T, payload, c.i8);
                st_out32(o, make_uint4(mul_bf16x2(v[0], s2), mul_bf16x2(v[1], s2), mul_bf16x2(v[2], s2),
                                       mul_bf16x2(v[3], s2)),
                         make_uint4(mul_bf16x2(v[4], s2), mul_bf16x2(v[5], s2), mul_bf16x2(v[6], s2),
                                    mul_bf16x2(v[7], s2)));
                c.col += c.gs;
                if (c.col >= c.cols) {
                    do {
                        c.col -= c.cols;
                        ++c.row;
                    } while (c.col >= c.cols);
                    if (ng > 1 || tail) s2 = c.sc[c.row] * 0x10001u;
                }
                o += 2 * c.gs;
                --ng;
                continue;
            }
            uint32_t q[8];
            bool esc = false;
            #pragma unroll
            for (int k = 0; k < (BF16 ? 4 : 8); ++k) {
                uint32_t a, b;
                if (GROUPED) {
                    a = decode_pair_g<NARROW>(c.x, c.r, T, esc);
                    b = decode_pair_g<NARROW>(c.x, c.r, T, esc);
                } else {
                    a = decode_pair<NARROW>(c.x, c.r, T, payload);
                    b = decode_pair<NARROW>(c.x, c.r, T, payload);
                }
                q[k] = __byte_perm(a, b, 0x5410);
                if ((k & 3) == 3) {
                    ring_step_w(c.r, payload);
                    if (GROUPED) {                 // R18: the group's escaped codes follow its pair steps
                        if (esc) patch_escapes(q + (k - 3), 8, c.x, c.r, T, payload);
                        esc = false;
                    }
                }
            }
            if (BF16) {
                uint4 lo, hi;
                if (s16) {
                    const uint16_t h = (uint16_t)s16;
                    lo = make_uint4(dequant2_h(q[0], h), dequant2_h(q[0] >> 16, h), dequant2_h(q[1], h), dequant2_h(q[1] >> 16, h));
                    hi = make_uint4(dequant2_h(q[2], h), dequant2_h(q[2] >> 16, h), dequant2_h(q[3], h), dequant2_h(q[3] >> 16, h));
                } else if (c.i8) {
                    lo = make_uint4(dequant2_i8(q[0], c.s), dequant2_i8(q[0] >> 16, c.s), dequant2_i8(q[1], c.s),
                                    dequant2_i8(q[1] >> 16, c.s));
                    hi = make_uint4(dequant2_i8(q[2], c.s), dequant2_i8(q[2] >> 16, c.s), dequant2_i8(q[3], c.s),
                                    dequant2_i8(q[3] >> 16, c.s));
                } else {
                    lo = make_uint4(dequant2(q[0], c.s), dequant2(q[0] >> 16, c.s), dequant2(q[1], c.s), dequant2(q[1] >> 16, c.s));
                    hi = make_uint4(dequant2(q[2], c.s), dequant2(q[2] >> 16, c.s), dequant2(q[3], c.s), dequant2(q[3] >> 16, c.s));
                }
                st_out32(o, lo, hi);
                c.col += c.gs;                         // the next group: 16 symbols on, or 512 (R17)
                if (c.col >= c.cols) {                 // next row: its scale (unless this was the last group)
                    do {
                        c.col -= c.cols;
                        ++c.row;
                    } while (c.col >= c.cols);
                    if (ng > 1 || tail) {
                        c.s = bf16_bits_to_float(c.sc[c.row]);
                        s16 = c.i8 ? 0u : (uint32_t)scale_f16(c.s);
                    }
                }
            } else if (c.gs == kIlGroup) {
                st_out32(o, make_uint4(q[0], q[1], q[2], q[3]), make_uint4(q[4], q[5], q[6], q[7]));
            } else {                                   // R17: the two groups are 512 positions apart
                st_out(reinterpret_cast<uint4*>(o), make_uint4(q[0], q[1], q[2], q[3]));
                st_out(reinterpret_cast<uint4*>(o + c.gs), make_uint4(q[4], q[5], q[6], q[7]));
            }
            o += 2 * c.gs;                             // 16 bf16 / 32 FP8 symbols on (32 B if contiguous)
            --ng;
        }
        c.i += (ng0 - ng) * G;
        if (ng != 0) { c.runaway = true; return; }
        if (VALS && ng0 != 0 && tail) {            // the tail's row scale (s2 tracked the rows)
            c.s = bf16_bits_to_float(c.sc[c.row]);
            s16 = c.i8 ? 0u : (uint32_t)scale_f16(c.s);
        }
        c.s16 = (uint16_t)s16;
        if (c.r.Q > qlim) { c.runaway = true; return; }
    }
    if (GROUPED) {                                 // generic / ragged tail, group by group (R18)
        while (c.i < c.n) {
            group_generic_g<BF16, NARROW, BF16 && EQ_PAIR_VALS && EQ_PAIR_TOPID>(c, payload, T, min(16u, c.n - c.i));
            if (c.r.Q > qlim) { c.runaway = true; return; }
        }
        return;
    }
    uint32_t k = 0;                                // generic / ragged tail
    for (; c.i + 2 <= c.n; c.i += 2) {
        const uint32_t ab = decode_pair<NARROW>(c.x, c.r, T, payload);
        if ((++k & 7) == 0) ring_step_w(c.r, payload);
        #pragma unroll
        for (int h = 0; h < 2; ++h) {
            store_one<BF16>(c.out, c.i + h, (ab >> (8 * h)) & 0xFFu, c.s, c.i8);
            if (BF16 && ++c.col == c.cols) {
                c.col = 0;
                ++c.row;
                if (c.i + h + 1 < c.n) c.s = bf16_bits_to_float(c.sc[c.row]);
            }
        }
        if (c.r.Q > qlim) { c.runaway = true; return; }
    }
    if (c.i < c.n) {                               // odd chunk: the last symbol is a single
        const uint32_t s1 = decode_single_p(c.x, c.r, T);
        store_one<BF16>(c.out, c.i, s1, c.s, c.i8);
        ++c.i;
    }
}

#ifndef EQ_PAIR_NARROW
#define EQ_PAIR_NARROW 1            // 2·id LUT entries when every kept pair has f ≤ 2048 (one add fewer per pair)
#endif
#ifndef EQ_PTHREADS
#define EQ_PTHREADS 256             // chunks (= threads) per CTA of k_decode_p
#endif
#ifndef EQ_DECP_MIN_CTAS
#define EQ_DECP_MIN_CTAS 5          // shared memory (40 KB: pair LUT, byte single LUT, rings) allows 5 CTAs/SM: 48 registers
#endif
constexpr int kPThreads = EQ_PTHREADS;
constexpr uint32_t kDecPSmem = kPThreads * kWRing;          // dynamic: the staging rings
template <bool BF16, bool GROUPED>
__global__ void __launch_bounds__(kPThreads, EQ_DECP_MIN_CTAS)
k_decode_p(const __grid_constant__ DecParams P) {
    extern __shared__ __align__(128) uint8_t rings[];      // kPThreads × kWRing
    constexpr bool VALS = BF16 && GROUPED && EQ_PAIR_VALS;
    // the contiguous table region of pair_core.cuh: pair LUT + codes, lut1 (first the pair cum,
    // see pair_tables_build), cum, and for R18 bf16 the value table
    __shared__ __align__(16) uint8_t tabs[kPairSmemBytes + (VALS ? 4 * kPairValWords : 0)];
    uint32_t* lut = reinterpret_cast<uint32_t*>(tabs);
    uint8_t* lut1 = tabs + kLut1Off;
    uint16_t* cum = reinterpret_cast<uint16_t*>(tabs + kCumOff);

    uint32_t bi = 0;
    while (bi + 1 < P.n_blocks && blockIdx.x >= P.b[bi + 1].cta0) ++bi;
    const DecBlock& B = P.b[bi];
    const int t = threadIdx.x;
    ChainW c;                                      // setup first: the initial copies overlap the table build
    chain_setup_w<BF16>(c, B, (blockIdx.x - B.cta0) * kPThreads + t,
                        (uint32_t)__cvta_generic_to_shared(rings + t * kWRing), P.arena, P.err);
    stage_commit();
    uint32_t cesc;
    const uint32_t mode = pair_tables_build<kPThreads, true, EQ_PAIR_NARROW, VALS, VALS && EQ_PAIR_TOPID>(
        B.freq, lut, lut1, cum, cesc, P.err, B.format == EQ_FMT_INT8);
    if (!mode) {
        stage_wait_all();
        return;
    }
    stage_wait_all();
    __syncthreads();
    const PairTab T = pair_tab(B.freq, lut, lut1, cum, cesc, P.k2p20, P.k2p12);
    chain_start_w(c);
    if (EQ_PAIR_NARROW && mode == 2) chain_finish_p<BF16, true, GROUPED>(c, B.payload, T);    // CTA-uniform
    else chain_finish_p<BF16, false, GROUPED>(c, B.payload, T);
    stage_wait_all();
    if (c.active && (c.runaway || c.x != kLw || c.r.Q - (2u + kWBias) != c.e)) atomicOr(P.err, EQ_EF_CORRUPT);
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
    if (blk.codec > EQ_CODEC_PAIR_G || blk.chunk_mode > EQ_CHUNK_INTERLEAVED) return EQ_ERR_ARG;
    if (blk.chunk_mode == EQ_CHUNK_INTERLEAVED && (!is_pair_codec(blk.codec) || blk.chunk_symbols % 32 != 0))
        return EQ_ERR_ARG;                         // R17 is decoded by k_decode_p only
    if (blk.chunk_mode == EQ_CHUNK_INTERLEAVED)    // R17: whole 16-symbol groups per row
        for (uint32_t l = 0; l < blk.n_layers && l < EQ_MAX_LAYERS; ++l)
            if (blk.layer_cols[l] % 16 != 0) return EQ_ERR_SHAPE;
    d.format = blk.format;
    d.codec = blk.codec;
    d.cs = blk.chunk_symbols;
    d.n_layers = blk.n_layers;
    d.cta0 = cta0;
    uint32_t chunk = 0, srow = 0;
    for (uint32_t l = 0; l < EQ_MAX_LAYERS; ++l) {
        DecLayer& L = d.layer[l];
        if (l < blk.n_layers) {
            L.out_off = offs[l];
            L.geom = chunk_geom(blk.chunk_mode, blk.layer_rows[l], blk.layer_cols[l], blk.chunk_symbols);
            L.chunk0 = chunk;
            L.cols = (uint32_t)blk.layer_cols[l];
            L.scale_off = srow;
            chunk += (uint32_t)layer_chunks(blk.chunk_mode, blk.layer_rows[l], blk.layer_cols[l], blk.chunk_symbols);
            srow += (uint32_t)blk.layer_rows[l];
        } else {
            L = DecLayer{0, ChunkGeom{1, 1}, chunk, 1, srow, 0};
        }
    }
    if (chunk != blk.n_chunks) return EQ_ERR_SHAPE;
    d.n_chunks = chunk;
    return EQ_OK;
}

static const void* pair_kernel(bool bf16, bool grouped) {
    return bf16 ? (grouped ? (const void*)k_decode_p<true, true> : (const void*)k_decode_p<true, false>)
                : (grouped ? (const void*)k_decode_p<false, true> : (const void*)k_decode_p<false, false>);
}

extern "C" eq_status eq_decode_lanes(uint32_t codec, uint32_t out_dtype, int device, uint64_t* lanes) {
    if (!lanes || codec > EQ_CODEC_PAIR_G || (out_dtype != EQ_OUT_FP8 && out_dtype != EQ_OUT_BF16)) return EQ_ERR_ARG;
    const bool bf = out_dtype == EQ_OUT_BF16;
    const void* fn;
    int threads, per;
    size_t dyn;
    if (is_pair_codec(codec)) {
        fn = pair_kernel(bf, codec == EQ_CODEC_PAIR_G);
        threads = kPThreads, per = kPThreads, dyn = kDecPSmem;
    } else if (codec == EQ_CODEC_WORD) {
        fn = bf ? (const void*)k_decode_w<true> : (const void*)k_decode_w<false>;
        threads = kWThreads, per = kWChunksPerCta, dyn = kDecWSmem;
    } else {
        fn = bf ? (const void*)k_decode<true> : (const void*)k_decode<false>;
        threads = kDecThreads, per = kChunksPerCta, dyn = 0;
    }
    int sms = 0, ctas = 0;
    EQ_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    if (dyn) EQ_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
    EQ_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, fn, threads, dyn));
    *lanes = (uint64_t)sms * (uint64_t)ctas * (uint64_t)per;
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
    const uint32_t codec = blocks[0].codec;
    for (uint32_t b = 1; b < n_blocks; ++b)
        if (blocks[b].codec != codec) return EQ_ERR_ARG;       // one codec per call
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
        P.k64 = 64u;
        P.k2p16 = 1u << 16;
        uint32_t ctas = 0;
        for (uint32_t k = 0; k < nb; ++k) {
            EQ_TRY(fill_desc(blocks[b0 + k], all.get() + (size_t)(b0 + k) * EQ_MAX_LAYERS, P.b[k], ctas));
            const uint32_t per = is_pair_codec(codec) ? (uint32_t)kPThreads
                               : codec == EQ_CODEC_WORD ? (uint32_t)kWChunksPerCta : (uint32_t)kChunksPerCta;
            ctas += (P.b[k].n_chunks + per - 1) / per;
        }
        // blocks with zero chunks cannot exist (layers are non-empty); ctas > 0
        if (is_pair_codec(codec)) {
            const bool bi = out_dtype == EQ_OUT_BF16, g = codec == EQ_CODEC_PAIR_G;
            const uint32_t dyn = kDecPSmem;
            EQ_CUDA_TRY(cudaFuncSetAttribute(pair_kernel(bi, g), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
            if (bi && g) k_decode_p<true, true><<<ctas, kPThreads, dyn, st>>>(P);
            else if (bi) k_decode_p<true, false><<<ctas, kPThreads, dyn, st>>>(P);
            else if (g) k_decode_p<false, true><<<ctas, kPThreads, dyn, st>>>(P);
            else k_decode_p<false, false><<<ctas, kPThreads, dyn, st>>>(P);
        } else if (codec == EQ_CODEC_WORD) {
            const int bi = out_dtype == EQ_OUT_BF16 ? 1 : 0;
            // (6 CTAs/SM: for the 8B layer set 7.5 waves; forcing 5 CTAs/SM for exactly 9 waves
            // measured 2.3 % slower — the tail wave runs faster, the lost latency hiding costs more)
            const uint32_t dyn = kDecWSmem;
            EQ_CUDA_TRY(cudaFuncSetAttribute(bi ? (const void*)k_decode_w<true> : (const void*)k_decode_w<false>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
            if (bi)
                k_decode_w<true><<<ctas, kWThreads, dyn, st>>>(P);
            else
                k_decode_w<false><<<ctas, kWThreads, dyn, st>>>(P);
        } else if (out_dtype == EQ_OUT_BF16) {
            k_decode<true><<<ctas, kDecThreads, 0, st>>>(P);
        } else {
            k_decode<false><<<ctas, kDecThreads, 0, st>>>(P);
        }
        EQ_CUDA_TRY(cudaGetLastError());
    }
    return EQ_OK;
}
