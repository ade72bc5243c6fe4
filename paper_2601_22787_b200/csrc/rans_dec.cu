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
struct BitReader {
    uint64_t bb;           // upcoming bits, next byte in bits 63..56
    int nb;                // valid bits in bb
    uint32_t used;         // payload bits consumed after the 4-byte state
    const uint32_t* wp;    // next aligned word
    const uint32_t* wend;  // first word that must not be read

    __device__ __forceinline__ uint32_t load_word() {
        uint32_t w = (wp < wend) ? __ldg(wp) : 0u;
        ++wp;
        return bswap32(w);
    }
    __device__ __forceinline__ void refill() {
        if (nb <= 32) {
            bb |= (uint64_t)load_word() << (32 - nb);
            nb += 32;
        }
    }
};

__device__ __forceinline__ uint32_t decode_one(uint32_t& x, BitReader& br, const uint32_t* lut) {
    uint32_t e = lut[x & (kM - 1)];
    uint32_t xs = x >> kProbBits;
    x = ((e >> 8) & 0xFFFu) * xs + xs + (e >> 20);
    if (x < kL) {
        uint32_t k = (x < (1u << 15)) ? 16u : 8u;
        x = (x << k) | (uint32_t)(br.bb >> (64 - k));
        br.bb <<= k;
        br.nb -= (int)k;
        br.used += k;
        br.refill();
    }
    return e & 0xFFu;
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
    uint32_t f = B.freq[t];
    {
        uint32_t v = f;
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
    BitReader br;
    br.wp = reinterpret_cast<const uint32_t*>(B.payload) + (a >> 2);
    br.wend = reinterpret_cast<const uint32_t*>(B.payload) + B.word_end;
    {
        const uint32_t sh = (uint32_t)(a & 3) * 8;
        uint64_t hi = br.load_word(), lo = br.load_word();
        br.bb = ((hi << 32) | lo) << sh;
        br.nb = 64 - (int)sh;
    }
    uint32_t x = bswap32((uint32_t)(br.bb >> 32));   // 4-byte little-endian state
    br.bb <<= 32;
    br.nb -= 32;
    br.used = 0;
    br.refill();

    const uint32_t esz = BF16 ? 2 : 1;
    uint8_t* out = P.arena + Ly.out_off + sym0 * esz;
    const uint16_t* sc = B.scales + Ly.scale_off;
    uint32_t row = (uint32_t)(sym0 / Ly.cols), col = (uint32_t)(sym0 % Ly.cols);
    float s = BF16 ? bf16_bits_to_float(sc[row]) : 0.f;

    uint32_t i = 0;
    if ((Ly.cols & 15) == 0 && (B.cs & 15) == 0) {
        for (; i + 16 <= n; i += 16) {
            uint32_t w[4];
            #pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t acc = 0;
                #pragma unroll
                for (int r = 0; r < 4; ++r) acc |= decode_one(x, br, lut) << (8 * r);
                w[q] = acc;
            }
            if (BF16) {
                uint32_t o[8];
                #pragma unroll
                for (int q = 0; q < 4; ++q) {
                    float2 v0 = e4m3x2_to_float2(w[q] & 0xFFFFu);
                    float2 v1 = e4m3x2_to_float2(w[q] >> 16);
                    __nv_bfloat162 b0 = __floats2bfloat162_rn(__fmul_rn(s, v0.x), __fmul_rn(s, v0.y));
                    __nv_bfloat162 b1 = __floats2bfloat162_rn(__fmul_rn(s, v1.x), __fmul_rn(s, v1.y));
                    o[2 * q] = *reinterpret_cast<uint32_t*>(&b0);
                    o[2 * q + 1] = *reinterpret_cast<uint32_t*>(&b1);
                }
                uint4* dst = reinterpret_cast<uint4*>(out + (uint64_t)i * 2);
                dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
                dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
                col += 16;
                if (col >= Ly.cols) {
                    col -= Ly.cols;
                    ++row;
                    if (i + 16 < n) s = bf16_bits_to_float(sc[row]);
                }
            } else {
                *reinterpret_cast<uint4*>(out + i) = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    }
    for (; i < n; ++i) {                       // generic / ragged tail: one symbol at a time
        uint32_t sym = decode_one(x, br, lut);
        store_one<BF16>(out, i, sym, s);
        if (BF16 && ++col == Ly.cols) {
            col = 0;
            ++row;
            if (i + 1 < n) s = bf16_bits_to_float(sc[row]);
        }
    }
    if (x != kL || 4ull + (br.used >> 3) != e - a) atomicOr(P.err, EQ_EF_CORRUPT);
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
    if ((reinterpret_cast<uintptr_t>(blk.payload) & 3) != 0) return EQ_ERR_ARG;
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
