// qmatmul.cu — §8(f) NEXT row 1 / config 4: QMatMul of Alg. 2 l.3 fused with the
// entropy decode and dequantisation of l.1-2: Y = X · Ŵᵀ for one layer of a compressed block,
// where Ŵ = RNE_bf16(s_row · value(code)) is never written to HBM.  The paper runs a Marlin
// FP8 GEMM (W8A16) on the buffer nvCOMP decoded into; here the decoded rows go
// straight into tcgen05 shared-memory operand tiles.
//
// CTA = 128 threads = 128 output channels (lane = weight row = one rANS chunk sequence, which
// needs row-aligned chunks: K % chunk_symbols == 0).  Per 64-column K step:
//   1. each lane decodes + dequantises the next 64 symbols of its row into the A tile
//      (bf16, K-major, SWIZZLE_128B canonical UMMA layout: 8-row × 128 B atoms, 16-byte
//      chunk j of row r stored at chunk j ^ (r & 7));
//   2. the 128 threads stage X[:, k0:k0+64] (bf16, K-major, same layout) as the B tile;
//   3. fence.proxy.async, barrier; one thread issues 4 × tcgen05.mma.cta_group::1.kind::f16
//      (M=128, N=batch padded to 8, K=16 each) accumulating fp32 in TMEM, then
//      tcgen05.commit → mbarrier of the stage.  Two stages: the decode of step t+1 overlaps
//      the MMAs of step t.
// Epilogue: tcgen05.ld 32x32b (warp w reads TMEM lanes 32w..32w+31 = rows) → fp32 Y[b][row].
#include "common.cuh"
#include "decode_core.cuh"

#include <algorithm>
#include <cstring>

namespace eq {

constexpr int kQThreads = 128;
constexpr int kQK = 64;                       // K columns per step (one 128-byte swizzle row)
constexpr int kATile = kQThreads * kQK * 2;   // 16 KB per stage

struct QmmParams {
    const uint8_t* payload;
    const uint32_t* off;
    const uint16_t* freq;
    const uint16_t* scales;   // this layer's first row
    uint64_t payload_bytes;
    const uint16_t* x;        // bf16 [n_real][K]
    float* y;                 // fp32 [n_real][rows]
    uint32_t* err;
    uint32_t format, cs, chunk0, rows, K, n_pad, n_real, idesc, tmem_cols;
    uint32_t k2p20, k2p12, kneg2p14, k4;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: start >> 4, LBO = 1 (unused for
// swizzled K-major), SBO = 1024 B (stride between 8-row atoms), version 1, layout type 2
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024u >> 4) << 32) |
           ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
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

// one lane's 64 decoded + dequantised symbols -> its row of the swizzled A tile
__device__ __forceinline__ void decode_step(Chain& c, const DecTable& T, const uint8_t* payload, uint8_t* a_tile,
                                            uint32_t r) {
    uint8_t* row = a_tile + (r >> 3) * 1024 + (r & 7) * 128;
    #pragma unroll
    for (int g = 0; g < 4; ++g) {                       // 4 × 16 symbols
        uint32_t q[4];
        q[0] = decode4(c, T);
        q[1] = decode4(c, T);
        stage_wait_all(); ring_issue(c.br, payload); stage_commit();
        q[2] = decode4(c, T);
        q[3] = decode4(c, T);
        stage_wait_all(); ring_issue(c.br, payload); stage_commit();
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
            lo = make_uint4(dequant2(q[0], c.s), dequant2(q[0] >> 16, c.s), dequant2(q[1], c.s),
                            dequant2(q[1] >> 16, c.s));
            hi = make_uint4(dequant2(q[2], c.s), dequant2(q[2] >> 16, c.s), dequant2(q[3], c.s),
                            dequant2(q[3] >> 16, c.s));
        }
        const uint32_t j0 = 2 * g, j1 = 2 * g + 1;     // 16-byte chunks of this 16-symbol group
        *reinterpret_cast<uint4*>(row + ((j0 ^ (r & 7)) << 4)) = lo;
        *reinterpret_cast<uint4*>(row + ((j1 ^ (r & 7)) << 4)) = hi;
        c.i += 16;
    }
}

// start decoding chunk `chunk` (payload bytes, ring staging, first state) for this lane
__device__ __forceinline__ bool chunk_begin(Chain& c, const QmmParams& P, uint32_t chunk, uint32_t ring) {
    c.i = 0;
    c.n = P.cs;
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
    // the previous chunk's look-ahead copies target the same ring slots and copies of
    // different groups are not ordered: drain them before staging the new chunk
    stage_wait_all();
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
    if (c.br.wi4 > c.wlimit4 || c.x != kL || consumed != 8ll * (int64_t)(c.e - c.a)) atomicOr(err, EQ_EF_CORRUPT);
}

__global__ void __launch_bounds__(kQThreads, 1) k_qmatmul(const __grid_constant__ QmmParams P) {
    extern __shared__ __align__(1024) uint8_t dsm_raw[];
    // SWIZZLE_128B atoms are addressed by absolute shared-address bits: align the carve-out
    uint8_t* dsm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
    // layout: [A stage 0 | A stage 1 | B stage 0 | B stage 1 | LUT | rings | cum | bars | tmem]
    uint8_t* a_tiles = dsm;                                          // 2 × 16 KB, 1024-aligned
    uint8_t* b_tiles = dsm + 2 * kATile;                             // 2 × n_pad × 128 B
    const uint32_t b_tile_bytes = P.n_pad * 128u;
    uint8_t* tail = b_tiles + 2 * ((b_tile_bytes + 1023) & ~1023u);
    uint32_t* lut = reinterpret_cast<uint32_t*>(tail);               // 16 KB
    uint32_t* rings = lut + kM;                                      // 128 × 64 B
    uint32_t* cum = rings + kQThreads * kRingWords;                  // 257
    uint64_t* bars = reinterpret_cast<uint64_t*>(cum + 260);         // 2 mbarriers (8-aligned)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);

    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const uint32_t row0 = blockIdx.x * kQThreads;

    // ---- TMEM accumulator (warp 0), mbarriers (thread 0)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(P.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (t == 0) {
        mbar_init(smem_u32(&bars[0]), 1);
        mbar_init(smem_u32(&bars[1]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // ---- block LUT (as in k_decode)
    {
        __shared__ uint32_t wsum[8];
        for (int base = 0; base < 256; base += kQThreads) {
            uint32_t v = P.freq[base + t];
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                uint32_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
                if (lane >= d) v += o;
            }
            if (lane == 31) wsum[(base >> 5) + warp] = v;
            cum[base + t + 1] = v;
        }
        __syncthreads();
        for (int base = 0; base < 256; base += kQThreads) {
            const int idx = base + t;
            uint32_t add = 0;
            for (int q = 0; q < (idx >> 5); ++q) add += wsum[q];
            cum[idx + 1] += add;
        }
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
            lut[slot] = (uint32_t)lo | ((fs - 1) << 8) | (((uint32_t)slot - cum[lo]) << 20);
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

    // ---- this lane's row
    const uint32_t r = (uint32_t)t;                 // row within the tile = TMEM lane
    const uint32_t grow = row0 + r;
    const uint32_t cpr = P.K / P.cs;                // chunks per row
    const uint32_t ring = smem_u32(rings + t * kRingWords);
    Chain c;
    c.sc = P.scales;
    c.i8 = P.format == EQ_FMT_INT8;
    c.s = bf16_bits_to_float(P.scales[grow]);
    c.s16 = c.i8 ? 0 : scale_f16(c.s);
    c.active = false;
    const uint32_t steps = P.K / kQK, steps_per_chunk = P.cs / kQK;

    for (uint32_t st = 0; st < steps; ++st) {
        const uint32_t s = st & 1;
        if (st % steps_per_chunk == 0) {
            if (st) chunk_end(c, P.err);
            if (table_ok) chunk_begin(c, P, P.chunk0 + grow * cpr + st / steps_per_chunk, ring);
        }
        if (st >= 2) mbar_wait(smem_u32(&bars[s]), ((st - 2) >> 1) & 1);   // MMA of step st-2 done
        uint8_t* a_tile = a_tiles + s * kATile;
        uint8_t* b_tile = b_tiles + s * ((b_tile_bytes + 1023) & ~1023u);
        if (c.active) decode_step(c, T, P.payload, a_tile, r);
        // activations X[:, k0:k0+64] -> B tile (rows = batch, zero-padded)
        const uint32_t k0 = st * kQK;
        for (uint32_t piece = t; piece < P.n_pad * 8; piece += kQThreads) {
            const uint32_t b = piece >> 3, j = piece & 7;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (b < P.n_real) v = __ldg(reinterpret_cast<const uint4*>(P.x + (uint64_t)b * P.K + k0) + j);
            *reinterpret_cast<uint4*>(b_tile + (b >> 3) * 1024 + (b & 7) * 128 + ((j ^ (b & 7)) << 4)) = v;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (t == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t da = umma_desc_sw128(smem_u32(a_tile)), db = umma_desc_sw128(smem_u32(b_tile));
            #pragma unroll
            for (int kk = 0; kk < kQK / 16; ++kk) {
                const uint32_t acc = (st > 0 || kk > 0) ? 1u : 0u;
                // +32 bytes per K=16 slice inside the swizzle atom (start address field in 16 B units)
                asm volatile(
                    "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(
                        tmem),
                    "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(P.idesc), "r"(acc));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&bars[s]))
                         : "memory");
        }
    }
    chunk_end(c, P.err);
    stage_wait_all();
    // ---- wait for the last MMA, read the accumulator
    const uint32_t last = steps - 1;
    mbar_wait(smem_u32(&bars[last & 1]), (last >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (uint32_t col = 0; col < P.n_pad; col += 8) {
        uint32_t v[8];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + col;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        #pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t b = col + q;
            if (b < P.n_real) P.y[(uint64_t)b * P.rows + grow] = __uint_as_float(v[q]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(P.tmem_cols));
}

}  // namespace eq

using namespace eq;

extern "C" eq_status eq_qmatmul(const eq_block* blk, uint32_t layer, const void* x, uint32_t batch, float* y,
                                uint32_t* d_err, eq_stream_t stream) {
    if (!blk || !x || !y || !d_err || layer >= blk->n_layers || layer >= EQ_MAX_LAYERS) return EQ_ERR_ARG;
    if (!blk->payload || !blk->chunk_off || !blk->freq || !blk->scales || blk->format > EQ_FMT_INT8) return EQ_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(blk->payload) & 15) != 0) return EQ_ERR_ARG;
    if ((reinterpret_cast<uintptr_t>(x) & 15) != 0) return EQ_ERR_ARG;
    if (blk->payload_cap < blk->payload_bytes + EQ_PAYLOAD_SLACK) return EQ_ERR_BUFFER;
    const int64_t rows = blk->layer_rows[layer], K = blk->layer_cols[layer];
    const uint32_t cs = blk->chunk_symbols;
    if (batch < 1 || batch > 256) return EQ_ERR_SHAPE;
    if (rows % kQThreads != 0 || K % kQK != 0 || cs % kQK != 0 || K % cs != 0) return EQ_ERR_SHAPE;
    uint32_t chunk0 = 0;
    uint64_t srow = 0;
    for (uint32_t l = 0; l < layer; ++l) {
        chunk0 += (uint32_t)(((uint64_t)blk->layer_rows[l] * blk->layer_cols[l] + cs - 1) / cs);
        srow += (uint64_t)blk->layer_rows[l];
    }
    QmmParams P;
    memset(&P, 0, sizeof(P));
    P.payload = blk->payload;
    P.off = blk->chunk_off;
    P.freq = blk->freq;
    P.scales = blk->scales + srow;
    P.payload_bytes = blk->payload_bytes;
    P.x = static_cast<const uint16_t*>(x);
    P.y = y;
    P.err = d_err;
    P.format = blk->format;
    P.cs = cs;
    P.chunk0 = chunk0;
    P.rows = (uint32_t)rows;
    P.K = (uint32_t)K;
    P.n_pad = (batch + 7) & ~7u;
    P.n_real = batch;
    P.tmem_cols = 32;
    while (P.tmem_cols < P.n_pad) P.tmem_cols <<= 1;
    // instruction descriptor, kind::f16: D f32, A = B = bf16, both K-major, N, M = 128
    P.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((P.n_pad >> 3) << 17) | ((128u >> 4) << 24);
    P.k2p20 = 1u << 20;
    P.k2p12 = 1u << 12;
    P.kneg2p14 = 0u - (1u << 14);
    P.k4 = 4u;
    const uint32_t b_tile = ((P.n_pad * 128u + 1023u) & ~1023u);
    const size_t smem = 2 * kATile + 2 * b_tile + kM * 4 + kQThreads * kRingWords * 4 + 260 * 4 + 2 * 8 + 16 + 1024;
    EQ_CUDA_TRY(cudaFuncSetAttribute(k_qmatmul, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_qmatmul<<<(unsigned)(rows / kQThreads), kQThreads, smem, (cudaStream_t)stream>>>(P);
    EQ_CUDA_TRY(cudaGetLastError());
    return EQ_OK;
}
