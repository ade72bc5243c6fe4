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

constexpr int kDecThreads = 256;
constexpr int kMaxDecBlocks = 48;

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
    uint64_t word_end;     // index of the first 32-bit word that must not be read
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
    DecBlock b[kMaxDecBlocks];
};

// ---------------------------------------------------------------- per-lane bit reader
// Upcoming payload bits, most significant first, in a 64-bit window (hi:lo) holding nb
// valid bits.  A symbol consumes k ∈ {0,8,16} bits with funnel shifts (branch-free);
// refill() runs after every PAIR of symbols and restores nb ≥ 32.
// The lane's compressed bytes are staged in a 64-byte shared-memory ring by cp.async
// (16-byte segments issued warp-uniformly every 8 symbols, ≥ 8 symbols before use), so
// no register ever waits on a global load (the warp-level scoreboard would otherwise
// serialise the lanes' independent refills).
constexpr int kRingWords = 16;
struct BitReader {
    uint32_t hi, lo;
    int nb;
    uint32_t wi4;          // 4 × (absolute index of the next payload word to insert)
    uint32_t gs;           // next 16-byte payload segment to stage
    uint32_t ring;         // shared address of this lane's ring (64-byte aligned)

    __device__ __forceinline__ void refill() {
        if (nb < 32) {                              // predicated, not a divergent branch
            uint32_t w;
            asm("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(ring | (wi4 & 0x3Cu)));
            w = bswap32(w);
            hi |= w >> nb;                          // lo is empty when nb < 32
            lo = __funnelshift_r(0u, w, nb);        // = w << (32 − nb)
            nb += 32;
            wi4 += 4;
        }
    }
};

__device__ __forceinline__ void stage_segment(uint32_t ring, const uint8_t* payload, uint32_t seg) {
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(ring | ((seg & 3u) << 4)),
                 "l"(payload + (uint64_t)seg * 16));
}
__device__ __forceinline__ void stage_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void stage_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Every 8 symbols: the copies of the previous boundary have landed (wait_all); stage one
// more segment if fewer than 13 words lie ahead of the reader (≤ 4 words are consumed per
// 8 symbols, so the words needed before the next boundary are always already landed and
// the ring never overwrites an unread word).
__device__ __forceinline__ void ring_boundary(BitReader& br, const uint8_t* payload) {
    stage_wait_all();
    if (br.gs * 16u <= br.wi4 + 48u) {
        stage_segment(br.ring, payload, br.gs);
        ++br.gs;
    }
    stage_commit();
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// One rANS decode step (Alg. 2 l.1): slot lookup, state update, byte renormalisation.
// LUT entry e: sym | (f−1) << 8 | (slot − c_sym) << 20; returns e (sym in the low byte).
// Field extraction and x>>12 use IMAD.HI (FMA pipe) to balance the integer ALU pipe.
__device__ __forceinline__ uint32_t decode_one(uint32_t& x, BitReader& br, uint32_t lut_s) {
    const uint32_t e = lds_u32(lut_s + (x & (kM - 1)) * 4u);
    const uint32_t xs = __umulhi(x, 1u << 20);             // x >> 12
    const uint32_t fm1 = __umulhi(e << 12, 1u << 12);      // (e >> 8) & 0xFFF
    x = fm1 * xs + (xs + (e >> 20));                       // f·⌊x/M⌋ + slot − c
    // bytes to read: 0 if x ≥ 2^23, 1 if x ≥ 2^15, else 2 (after a step x ≥ 2^11)
    const uint32_t k = (uint32_t)(__clz(x) - 1) & 0x18u;
    x = __funnelshift_lc(br.hi, x, k);
    br.hi = __funnelshift_lc(br.lo, br.hi, k);
    br.lo = br.lo << k;
    br.nb -= (int)k;
    return e;
}

template <bool BF16>
__device__ __forceinline__ void store_one(uint8_t* out, uint64_t i, uint32_t sym, float s) {
    if (BF16) {
        __half_raw h = __nv_cvt_fp8_to_halfraw((__nv_fp8_storage_t)sym, __NV_E4M3);
        float v = __half2float(*reinterpret_cast<__half*>(&h));
        reinterpret_cast<uint16_t*>(out)[i] = float_to_bf16_bits(__fmul_rn(s, v));
    } else {
        out[i] = (uint8_t)sym;
    }
}

// decoded output is written once and never re-read by this kernel: evict-first in L2 so
// it does not push the (re-read) compressed input out of the cache
#ifndef EQ_CS_STORES
#define EQ_CS_STORES 1
#endif
__device__ __forceinline__ void st_out(uint4* p, uint4 v) {
#if EQ_CS_STORES
    __stcs(p, v);
#else
    *p = v;
#endif
}

// 4 symbols -> one word of codes (first symbol in the low byte), two refills
__device__ __forceinline__ uint32_t decode4(uint32_t& x, BitReader& br, uint32_t lut_s) {
    const uint32_t a = decode_one(x, br, lut_s);
    const uint32_t b = decode_one(x, br, lut_s);
    br.refill();
    const uint32_t c = decode_one(x, br, lut_s);
    const uint32_t d = decode_one(x, br, lut_s);
    br.refill();
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// Q† on two codes: exact e4m3 -> f32, one exact f32 product each, one RNE to bf16 each
__device__ __forceinline__ uint32_t dequant2(uint32_t pair, float s) {
    const float2 v = e4m3x2_to_float2(pair);
    __nv_bfloat162 b = __floats2bfloat162_rn(__fmul_rn(s, v.x), __fmul_rn(s, v.y));
    return *reinterpret_cast<uint32_t*>(&b);
}

template <bool BF16>
__global__ void __launch_bounds__(kDecThreads)
k_decode(const __grid_constant__ DecParams P) {
    __shared__ uint32_t lut[kM];
    __shared__ uint32_t cum[257];

    uint32_t bi = 0;
    while (bi + 1 < P.n_blocks && blockIdx.x >= P.b[bi + 1].cta0) ++bi;
    const DecBlock& B = P.b[bi];

    // ---- table: exclusive prefix of the 256 frequencies, then the slot LUT
    const int t = threadIdx.x;
    {
        uint32_t v = B.freq[t];
        #pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            uint32_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
            if ((t & 31) >= d) v += o;
        }
        __shared__ uint32_t wsum[kDecThreads / 32];
        if ((t & 31) == 31) wsum[t >> 5] = v;
        __syncthreads();
        uint32_t add = 0;
        for (int w = 0; w < (t >> 5); ++w) add += wsum[w];
        cum[t + 1] = v + add;
        if (t == 0) cum[0] = 0;
    }
    __syncthreads();
    if (cum[256] != kM) {                     // corrupt table: nothing decodable
        if (t == 0) atomicOr(P.err, EQ_EF_CORRUPT);
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
    __syncthreads();
    const uint32_t lut_s = (uint32_t)__cvta_generic_to_shared(lut);

    // ---- this lane's chunk
    const uint32_t c = (blockIdx.x - B.cta0) * kDecThreads + t;
    if (c >= B.n_chunks) return;
    uint32_t l = 0;
    while (l + 1 < B.n_layers && c >= B.layer[l + 1].chunk0) ++l;
    const DecLayer& Ly = B.layer[l];
    const uint64_t sym0 = (uint64_t)(c - Ly.chunk0) * B.cs;
    const uint32_t n = (uint32_t)min((uint64_t)B.cs, Ly.size - sym0);

    const uint64_t a = __ldg(B.off + c), e = __ldg(B.off + c + 1);
    if (e < a || e > B.payload_bytes || e - a < 4) {
        atomicOr(P.err, EQ_EF_TRUNCATED);
        return;
    }
    // ---- stage the first 64 bytes of the chunk and read the state
    BitReader br;
    uint32_t x;
    {
        __shared__ __align__(64) uint32_t rings[kDecThreads * kRingWords];
        br.ring = (uint32_t)__cvta_generic_to_shared(rings + t * kRingWords);
        const uint32_t s0 = (uint32_t)(a >> 4);
        #pragma unroll
        for (int q = 0; q < 4; ++q) stage_segment(br.ring, B.payload, s0 + q);
        stage_commit();
        stage_wait_all();
        br.gs = s0 + 4;
        const uint32_t wa = (uint32_t)(a >> 2);
        uint32_t h, m;
        asm("ld.shared.u32 %0, [%1];" : "=r"(h) : "r"(br.ring | ((wa * 4u) & 0x3Cu)));
        asm("ld.shared.u32 %0, [%1];" : "=r"(m) : "r"(br.ring | (((wa + 1) * 4u) & 0x3Cu)));
        h = bswap32(h);
        m = bswap32(m);
        const uint32_t sh = (uint32_t)(a & 3) * 8;
        x = bswap32(__funnelshift_lc(m, h, sh));   // 4-byte little-endian initial state
        br.hi = m << sh;                            // remaining bytes of word 1
        br.lo = 0;
        br.nb = 32 - (int)sh;
        br.wi4 = (wa + 2) * 4u;
        br.refill();                                // nb ≥ 32 from here on, at pair starts
    }
    // a corrupt chunk may read past its end: stop (and flag) once 64 bytes beyond it
    const uint32_t wlimit4 = (uint32_t)((e >> 2) + 16) * 4u;

    const uint32_t esz = BF16 ? 2 : 1;
    uint8_t* out = P.arena + Ly.out_off + sym0 * esz;
    const uint16_t* sc = B.scales + Ly.scale_off;
    uint32_t row = (uint32_t)(sym0 / Ly.cols), col = (uint32_t)(sym0 % Ly.cols);
    float s = BF16 ? bf16_bits_to_float(sc[row]) : 0.f;

    uint32_t i = 0;
    bool runaway = false;
    if (BF16) {
        if ((Ly.cols & 15) == 0 && (B.cs & 15) == 0) {
            for (; i + 16 <= n; i += 16) {
                const uint32_t q0 = decode4(x, br, lut_s), q1 = decode4(x, br, lut_s);
                ring_boundary(br, B.payload);
                const uint32_t q2 = decode4(x, br, lut_s), q3 = decode4(x, br, lut_s);
                ring_boundary(br, B.payload);
                uint4* dst = reinterpret_cast<uint4*>(out + (uint64_t)i * 2);
                st_out(dst, make_uint4(dequant2(q0, s), dequant2(q0 >> 16, s), dequant2(q1, s), dequant2(q1 >> 16, s)));
                st_out(dst + 1, make_uint4(dequant2(q2, s), dequant2(q2 >> 16, s), dequant2(q3, s), dequant2(q3 >> 16, s)));
                col += 16;
                if (col >= Ly.cols) {
                    col -= Ly.cols;
                    ++row;
                    if (i + 16 < n) s = bf16_bits_to_float(sc[row]);
                }
                if (br.wi4 > wlimit4) { runaway = true; break; }
            }
        }
    } else {
        if ((B.cs & 31) == 0) {
            for (; i + 32 <= n; i += 32) {
                uint32_t q[8];
                #pragma unroll
                for (int k = 0; k < 8; ++k) {
                    q[k] = decode4(x, br, lut_s);
                    if (k & 1) ring_boundary(br, B.payload);
                }
                uint4* dst = reinterpret_cast<uint4*>(out + i);
                st_out(dst, make_uint4(q[0], q[1], q[2], q[3]));
                st_out(dst + 1, make_uint4(q[4], q[5], q[6], q[7]));
                if (br.wi4 > wlimit4) { runaway = true; break; }
            }
        }
    }
    if (!runaway) {
        for (; i < n; ++i) {                   // generic / ragged tail: one symbol at a time
            const uint32_t sym = decode_one(x, br, lut_s) & 0xFFu;
            br.refill();
            if ((i & 7) == 7) ring_boundary(br, B.payload);
            store_one<BF16>(out, i, sym, s);
            if (BF16 && ++col == Ly.cols) {
                col = 0;
                ++row;
                if (i + 1 < n) s = bf16_bits_to_float(sc[row]);
            }
            if (br.wi4 > wlimit4) { runaway = true; break; }
        }
    }
    // integrity: final state L and every payload byte of the chunk consumed exactly
    // (bits inserted into the window = 32·(words inserted) − 8·misalignment)
    stage_wait_all();
    const int64_t inserted = 8ll * (int64_t)(br.wi4 - (uint32_t)(a >> 2) * 4u) - 8ll * (int64_t)(a & 3);
    const int64_t consumed = inserted - br.nb;            // includes the 32-bit state
    if (runaway || x != kL || consumed != 8ll * (int64_t)(e - a)) atomicOr(P.err, EQ_EF_CORRUPT);
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
    d.word_end = blk.payload_cap / 4;
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
        uint32_t ctas = 0;
        for (uint32_t k = 0; k < nb; ++k) {
            EQ_TRY(fill_desc(blocks[b0 + k], all.get() + (size_t)(b0 + k) * EQ_MAX_LAYERS, P.b[k], ctas));
            ctas += (P.b[k].n_chunks + kDecThreads - 1) / kDecThreads;
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
