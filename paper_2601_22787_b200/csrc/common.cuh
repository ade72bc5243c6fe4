// common.cuh — shared device helpers of libentquant (sm_100a).  No code here is shared
// with the oracle (oracle/ is a separate CPU program).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp8.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/entquant.h"

namespace eq {

constexpr uint32_t kL = 1u << 23;            // rANS lower bound, EQ_CODEC_BYTE (R9)
constexpr uint32_t kLw = 1u << 16;           // rANS lower bound, EQ_CODEC_WORD (R14)
// the pair codecs share tables and decoder (R15; R18 only reorders a group's steps)
__host__ __device__ constexpr bool is_pair_codec(uint32_t codec) {
    return codec == EQ_CODEC_PAIR || codec == EQ_CODEC_PAIR_G;
}
constexpr uint32_t kProbBits = 12;
constexpr uint32_t kM = 1u << kProbBits;
constexpr float kQmax = 448.0f;              // E4M3 Q_max

#define EQ_CUDA_TRY(expr)                                   \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return EQ_ERR_CUDA;          \
    } while (0)

#define EQ_TRY(expr)                                        \
    do {                                                    \
        eq_status _s = (expr);                              \
        if (_s != EQ_OK) return _s;                         \
    } while (0)

// Chunk geometry of one layer: chunking restarts every `seg` symbols — the
// whole layer (EQ_CHUNK_LAYER, EQ_CHUNK_INTERLEAVED) or one row (EQ_CHUNK_ROW) — so a segment
// holds cps = ceil(seg / cs) chunks, all of cs symbols but the last.  Under EQ_CHUNK_INTERLEAVED
// (R17) the first nil = 32·⌊seg / 32cs⌋ chunks of the layer are interleaved: chunk k < nil is
// chunk j = k mod 32 of super-chunk s = ⌊k / 32⌋ and holds the super-chunk's 16-symbol groups
// j, j + 32, …, i.e. symbol i sits at s·32cs + (⌊i/16⌋·32 + j)·16 + i mod 16.
constexpr uint32_t kIlWays = 32, kIlGroup = 16;
struct ChunkGeom {
    uint64_t seg;          // segment length in symbols
    uint32_t cps;          // chunks per segment
    uint32_t nil;          // leading interleaved chunks of the layer (EQ_CHUNK_INTERLEAVED), else 0
};
__host__ __device__ __forceinline__ ChunkGeom chunk_geom(uint32_t mode, uint64_t rows, uint64_t cols, uint32_t cs) {
    const uint64_t seg = mode == EQ_CHUNK_ROW ? cols : rows * cols;
    const uint32_t nil = mode == EQ_CHUNK_INTERLEAVED ? (uint32_t)(seg / ((uint64_t)kIlWays * cs)) * kIlWays : 0u;
    return ChunkGeom{seg, (uint32_t)((seg + cs - 1) / cs), nil};
}
__host__ __device__ __forceinline__ uint64_t layer_chunks(uint32_t mode, uint64_t rows, uint64_t cols, uint32_t cs) {
    const ChunkGeom g = chunk_geom(mode, rows, cols, cs);
    return (rows * cols / g.seg) * g.cps;
}
// first symbol (within the layer) and length of the layer's local chunk k; *gstride = layer
// positions between consecutive 16-symbol groups of the chunk (16: contiguous; 512: R17)
__host__ __device__ __forceinline__ uint64_t chunk_start(const ChunkGeom& g, uint32_t cs, uint32_t k, uint32_t& n,
                                                         uint32_t* gstride = nullptr) {
    if (k < g.nil) {
        if (gstride) *gstride = kIlWays * kIlGroup;
        n = cs;
        return (uint64_t)(k / kIlWays) * kIlWays * cs + (uint64_t)(k % kIlWays) * kIlGroup;
    }
    if (gstride) *gstride = kIlGroup;
    const uint32_t s = k / g.cps, j = k - s * g.cps;
    const uint64_t a = (uint64_t)j * cs;
    n = (uint32_t)(g.seg - a < cs ? g.seg - a : cs);
    return (uint64_t)s * g.seg + a;
}

__device__ __forceinline__ float bf16_bits_to_float(uint32_t b) {
    return __uint_as_float(b << 16);
}

// round-to-nearest-even f32 -> bf16 bits (hardware cvt.rn.bf16.f32; subnormals kept)
__device__ __forceinline__ uint16_t float_to_bf16_bits(float f) {
    __nv_bfloat16 h = __float2bfloat16_rn(f);
    return *reinterpret_cast<uint16_t*>(&h);
}

// Two E4M3 codes (lo byte = first) from two floats: cvt.rn.satfinite.e4m3x2.f32, which
// clamps to ±448 before rounding (R2) and rounds to nearest even; then −0 (0x80) -> +0.
__device__ __forceinline__ uint32_t e4m3x2_from_float2(float a, float b) {
    __nv_fp8x2_storage_t p = __nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
    uint32_t u = (uint32_t)p;
    if ((u & 0xFFu) == 0x80u) u &= 0xFF00u;
    if ((u & 0xFF00u) == 0x8000u) u &= 0x00FFu;
    return u;
}

// Two E4M3 codes as cvt.rn.satfinite.e4m3x2.f32 gives them (−0 kept as 0x80)
__device__ __forceinline__ uint32_t e4m3x2_sat(float a, float b) {
    return (uint32_t)__nv_cvt_float2_to_fp8x2(make_float2(a, b), __NV_SATFINITE, __NV_E4M3);
}

// Two E4M3 codes (packed lo/hi byte) to two exact floats via the f16 path (exact).
__device__ __forceinline__ float2 e4m3x2_to_float2(uint32_t pair) {
    __half2_raw h = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(pair & 0xFFFFu), __NV_E4M3);
    __half2 hh = *reinterpret_cast<__half2*>(&h);
    return __half22float2(hh);
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// Int8: clamp to ±127, round half to even (the f32 quotient of bf16 values
// is ≥ 2^-9 relative away from any half-integer unless exactly on it, so fl32 suffices)
__device__ __forceinline__ uint32_t int8x2_from_float2(float a, float b) {
    const int ia = __float2int_rn(fminf(fmaxf(a, -127.f), 127.f));
    const int ib = __float2int_rn(fminf(fmaxf(b, -127.f), 127.f));
    return ((uint32_t)ia & 0xFFu) | (((uint32_t)ib & 0xFFu) << 8);
}
__device__ __forceinline__ float2 int8x2_to_float2(uint32_t pair) {
    return make_float2((float)(int8_t)(pair & 0xFFu), (float)(int8_t)((pair >> 8) & 0xFFu));
}
template <uint32_t FMT>
__device__ __forceinline__ uint32_t codes2(float a, float b) {
    return FMT == EQ_FMT_INT8 ? int8x2_from_float2(a, b) : e4m3x2_from_float2(a, b);
}
template <uint32_t FMT>
__device__ __forceinline__ float2 values2(uint32_t pair) {
    return FMT == EQ_FMT_INT8 ? int8x2_to_float2(pair) : e4m3x2_to_float2(pair);
}


}  // namespace eq
