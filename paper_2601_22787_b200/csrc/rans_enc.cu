// rans_enc.cu — §8(a) row a6: per-chunk rANS encoding (Alg. 1 l.4-5, P:212-213;
// S:316-324) of the block's concatenated E4M3 symbol stream (App. A.1).
// Wire formats: 32-bit state, M = 2^12, cum in code order; per chunk the symbols are coded
// in reverse from x = L, units of b emitted while x ≥ ((L>>12)·b)·f; the final state is
// stored first (little-endian), followed by the units in decode order.
//   EQ_CODEC_BYTE (R9):  L = 2^23, b = 2^8;   EQ_CODEC_WORD (R14): L = 2^16, b = 2^16 (LE).
// Chunks of cs symbols restart at each layer start (R10), and at each row start under
// EQ_CHUNK_ROW.
//
// Two passes, one thread per chunk: (1) exact byte count per chunk, (2) exclusive scan
// into chunk offsets, (3) encode again writing back-to-front straight into the final
// payload position — no worst-case scratch, no compaction copy.
#include "common.cuh"

#include <algorithm>

namespace eq {

constexpr int kEncThreads = 128;

struct EncParams {
    const uint8_t* codes;
    uint8_t* payload;
    uint32_t* chunk_off;
    uint32_t* sizes;
    const uint16_t* freq;
    uint32_t* err;
    unsigned long long* total;
    uint64_t payload_cap;
    uint32_t n_chunks;
    uint32_t cs;
    uint32_t n_layers;
    uint32_t chunk0[EQ_MAX_LAYERS + 1];
    uint64_t sym_base[EQ_MAX_LAYERS];
    ChunkGeom geom[EQ_MAX_LAYERS];
};

__device__ __forceinline__ void chunk_range(const EncParams& P, uint32_t c, uint64_t& base, uint32_t& n,
                                            uint32_t& gstride) {
    uint32_t l = 0;
    while (l + 1 < P.n_layers && c >= P.chunk0[l + 1]) ++l;
    base = P.sym_base[l] + chunk_start(P.geom[l], P.cs, c - P.chunk0[l], n, &gstride);
}

// symbol i of a chunk: contiguous (gstride 16) or R17-interleaved (gstride 512) 16-symbol groups
struct ChunkSyms {
    const uint8_t* p;
    uint32_t gstride;
    __device__ __forceinline__ uint32_t operator[](int64_t i) const {
        return p[(uint64_t)(i >> 4) * gstride + (uint64_t)(i & 15)];
    }
};

__device__ __forceinline__ void load_table(const EncParams& P, uint32_t* sf, uint32_t* scum) {
    // sf[s] = freq, scum[s] = cumulative (code order); one warp scans, others wait
    if (threadIdx.x < 32) {
        uint32_t run = 0;
        for (int b = 0; b < 256; b += 32) {
            uint32_t f = P.freq[b + threadIdx.x], v = f;
            #pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                uint32_t o = __shfl_up_sync(0xFFFFFFFFu, v, d);
                if ((int)threadIdx.x >= d) v += o;
            }
            sf[b + threadIdx.x] = f;
            scum[b + threadIdx.x] = run + v - f;
            run += __shfl_sync(0xFFFFFFFFu, v, 31);
        }
    }
    __syncthreads();
}

template <bool WRITE, bool WORD>
__global__ void __launch_bounds__(kEncThreads) k_encode(const __grid_constant__ EncParams P) {
    __shared__ uint32_t sf[256], scum[256];
    load_table(P, sf, scum);
    const uint32_t c = blockIdx.x * kEncThreads + threadIdx.x;
    if (c >= P.n_chunks) return;
    uint64_t base;
    uint32_t n;
    uint32_t gstride;
    chunk_range(P, c, base, n, gstride);
    const ChunkSyms sym{P.codes + base, gstride};
    uint8_t* dst = nullptr;
    uint64_t end = 0, beg = 0;
    if (WRITE) {
        beg = P.chunk_off[c];
        end = P.chunk_off[c + 1];
        if (end + EQ_PAYLOAD_SLACK > P.payload_cap) {
            atomicOr(P.err, EQ_EF_BUFFER);
            return;
        }
        dst = P.payload + end;
    }
    uint32_t x = WORD ? kLw : kL, bytes = 0;
    for (int64_t i = (int64_t)n - 1; i >= 0; --i) {
        const uint32_t s = sym[i];
        const uint32_t f = sf[s];
        if (f == 0) {
            atomicOr(P.err, EQ_EF_UNKNOWN_SYMBOL);
            break;
        }
        if (WORD) {
            // x_max = 2^20·f ≤ 2^32: at most one word (x < 2^32 → x >> 16 < 2^16 ≤ 2^20·f)
            if ((uint64_t)x >= ((uint64_t)(kLw >> kProbBits) << 16) * f) {
                if (WRITE) {
                    dst -= 2;
                    dst[0] = (uint8_t)(x & 0xFFu);
                    dst[1] = (uint8_t)((x >> 8) & 0xFFu);
                }
                bytes += 2;
                x >>= 16;
            }
        } else {
            const uint32_t x_max = ((kL >> kProbBits) << 8) * f;
            while (x >= x_max) {
                if (WRITE) *--dst = (uint8_t)(x & 0xFFu);
                ++bytes;
                x >>= 8;
            }
        }
        x = (x / f) * kM + (x % f) + scum[s];
    }
    if (WRITE) {
        if (end - beg != (uint64_t)bytes + 4) {
            atomicOr(P.err, EQ_EF_BUFFER);
            return;
        }
        dst -= 4;
        dst[0] = (uint8_t)x;
        dst[1] = (uint8_t)(x >> 8);
        dst[2] = (uint8_t)(x >> 16);
        dst[3] = (uint8_t)(x >> 24);
    } else {
        P.sizes[c] = bytes + 4;
    }
}

// EQ_CODEC_PAIR (R15): pairs (s[2i], s[2i+1]) of ranked codes whose pair is kept are one
// pair-table symbol, other pairs the escape followed by the two codes (single table), an
// odd tail one single; all word-codec rANS steps, in reverse (escaped pair: b, a, escape).
// EQ_CODEC_PAIR_G (R18): the same steps, per 16-symbol group in the decode order "the group's
// pair steps, then the codes (a, b) of each escaped pair in position order, then an odd last
// symbol"; the encoder walks that order backwards, last group first.
// Table buffer layout as in include/entquant.h (P.freq points at 512 u16).
struct WordEmitter {
    uint32_t x, bytes;
    uint8_t* dst;
    template <bool WRITE>
    __device__ __forceinline__ void put(uint32_t f, uint32_t c) {
        if ((uint64_t)x >= ((uint64_t)(kLw >> kProbBits) << 16) * f) {
            if (WRITE) {
                dst -= 2;
                dst[0] = (uint8_t)(x & 0xFFu);
                dst[1] = (uint8_t)((x >> 8) & 0xFFu);
            }
            bytes += 2;
            x >>= 16;
        }
        x = (x / f) * kM + (x % f) + c;
    }
};

template <bool WRITE, bool GROUPED>
__global__ void __launch_bounds__(kEncThreads) k_encode_pair(const __grid_constant__ EncParams P) {
    __shared__ uint32_t sf[256], scum[256];
    __shared__ uint32_t pf[225], pcum[225];
    __shared__ int32_t rank[256];
    __shared__ uint32_t fesc_s, cesc_s;
    load_table(P, sf, scum);
    const uint32_t K = P.freq[482];
    const uint8_t* rc = reinterpret_cast<const uint8_t*>(P.freq + 484);
    for (int i = threadIdx.x; i < 256; i += kEncThreads) rank[i] = -1;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint32_t r = 0; r < K; ++r) rank[rc[r]] = (int32_t)r;
        uint32_t run = 0;
        for (int q = 0; q < 225; ++q) {
            const bool on = (uint32_t)(q / 15) < K && (uint32_t)(q % 15) < K;
            pf[q] = on ? P.freq[256 + q] : 0;
            pcum[q] = run;
            run += pf[q];
        }
        cesc_s = run;
        fesc_s = P.freq[481];
    }
    __syncthreads();
    const uint32_t c = blockIdx.x * kEncThreads + threadIdx.x;
    if (c >= P.n_chunks) return;
    uint64_t base;
    uint32_t n;
    uint32_t gstride;
    chunk_range(P, c, base, n, gstride);
    const ChunkSyms sym{P.codes + base, gstride};
    uint64_t end = 0, beg = 0;
    WordEmitter E{kLw, 0, nullptr};
    if (WRITE) {
        beg = P.chunk_off[c];
        end = P.chunk_off[c + 1];
        if (end + EQ_PAYLOAD_SLACK > P.payload_cap) {
            atomicOr(P.err, EQ_EF_BUFFER);
            return;
        }
        E.dst = P.payload + end;
    }
    bool bad = false;
    if (GROUPED) {
        for (int64_t g0 = (int64_t)((n - 1) & ~15u); n > 0 && g0 >= 0 && !bad; g0 -= 16) {
            const uint32_t len = min(16u, n - (uint32_t)g0), m = len / 2;
            uint32_t esc = 0;                      // escaped pair positions of the group
            for (uint32_t k = 0; k < m; ++k) {
                const uint32_t a = sym[g0 + 2 * k], b = sym[g0 + 2 * k + 1];
                if (sf[a] == 0 || sf[b] == 0) { bad = true; break; }
                const int ra = rank[a], rb = rank[b];
                if (!(ra >= 0 && rb >= 0 && pf[ra * 15 + rb] > 0)) {
                    if (fesc_s == 0) { bad = true; break; }
                    esc |= 1u << k;
                }
            }
            if (bad) break;
            if (len & 1) {                         // the odd last symbol (decoded last)
                const uint32_t s = sym[g0 + len - 1];
                if (sf[s] == 0) { bad = true; break; }
                E.put<WRITE>(sf[s], scum[s]);
            }
            for (int k = (int)m - 1; k >= 0; --k)  // the escaped pairs' codes, b then a
                if (esc >> k & 1) {
                    const uint32_t a = sym[g0 + 2 * k], b = sym[g0 + 2 * k + 1];
                    E.put<WRITE>(sf[b], scum[b]);
                    E.put<WRITE>(sf[a], scum[a]);
                }
            for (int k = (int)m - 1; k >= 0; --k) {  // the group's pair steps
                if (esc >> k & 1) {
                    E.put<WRITE>(fesc_s, cesc_s);
                } else {
                    const int q = rank[sym[g0 + 2 * k]] * 15 + rank[sym[g0 + 2 * k + 1]];
                    E.put<WRITE>(pf[q], pcum[q]);
                }
            }
        }
    } else if (n & 1) {
        const uint32_t s = sym[n - 1];
        if (sf[s] == 0) bad = true;
        else E.put<WRITE>(sf[s], scum[s]);
    }
    for (int64_t i = GROUPED ? -1 : (int64_t)(n / 2) - 1; i >= 0 && !bad; --i) {
        const uint32_t a = sym[2 * i], b = sym[2 * i + 1];
        if (sf[a] == 0 || sf[b] == 0) { bad = true; break; }
        const int ra = rank[a], rb = rank[b];
        const int q = ra * 15 + rb;
        if (ra >= 0 && rb >= 0 && pf[q] > 0) {
            E.put<WRITE>(pf[q], pcum[q]);
        } else {
            if (fesc_s == 0) { bad = true; break; }
            E.put<WRITE>(sf[b], scum[b]);
            E.put<WRITE>(sf[a], scum[a]);
            E.put<WRITE>(fesc_s, cesc_s);
        }
    }
    if (bad) {
        atomicOr(P.err, EQ_EF_UNKNOWN_SYMBOL);
        return;
    }
    if (WRITE) {
        if (end - beg != (uint64_t)E.bytes + 4) {
            atomicOr(P.err, EQ_EF_BUFFER);
            return;
        }
        uint8_t* d = E.dst - 4;
        d[0] = (uint8_t)E.x;
        d[1] = (uint8_t)(E.x >> 8);
        d[2] = (uint8_t)(E.x >> 16);
        d[3] = (uint8_t)(E.x >> 24);
    } else {
        P.sizes[c] = E.bytes + 4;
    }
}

// exclusive scan of sizes -> chunk_off[0..n], total; one CTA, fixed segments (deterministic)
__global__ void __launch_bounds__(1024) k_scan(const uint32_t* __restrict__ sizes, uint32_t n,
                                               uint32_t* __restrict__ off, unsigned long long* total,
                                               uint32_t* err) {
    __shared__ unsigned long long part[1024];
    const uint32_t t = threadIdx.x;
    const uint32_t per = (n + 1023) / 1024;
    const uint32_t a = min(n, t * per), b = min(n, a + per);
    unsigned long long s = 0;
    for (uint32_t i = a; i < b; ++i) s += sizes[i];
    part[t] = s;
    __syncthreads();
    for (uint32_t d = 1; d < 1024; d <<= 1) {       // Hillis-Steele inclusive scan
        unsigned long long v = t >= d ? part[t - d] : 0ull;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    unsigned long long run = t ? part[t - 1] : 0ull;
    for (uint32_t i = a; i < b; ++i) {
        if (run > 0xFFFFFFFFull) atomicOr(err, EQ_EF_BUFFER);
        off[i] = (uint32_t)run;
        run += sizes[i];
    }
    if (t == 1023) {
        off[n] = (uint32_t)part[1023];
        *total = part[1023];
        if (part[1023] > 0xFFFFFFFFull) atomicOr(err, EQ_EF_BUFFER);
    }
}

}  // namespace eq

using namespace eq;

extern "C" eq_status eq_rans_encode(const uint8_t* codes, const eq_block* blk, uint32_t* chunk_sizes,
                                    uint64_t* payload_bytes_dev, uint32_t* d_err, eq_stream_t stream) {
    if (!codes || !blk || !chunk_sizes || !payload_bytes_dev || !d_err) return EQ_ERR_ARG;
    if (!blk->payload || !blk->chunk_off || !blk->freq) return EQ_ERR_ARG;
    if (blk->n_layers == 0 || blk->n_layers > EQ_MAX_LAYERS) return EQ_ERR_ARG;
    if (blk->chunk_symbols == 0 || blk->chunk_symbols > 262144u) return EQ_ERR_ARG;
    if (blk->codec > EQ_CODEC_PAIR_G || blk->chunk_mode > EQ_CHUNK_INTERLEAVED) return EQ_ERR_ARG;
    if (blk->chunk_mode == EQ_CHUNK_INTERLEAVED && (!is_pair_codec(blk->codec) || blk->chunk_symbols % 32 != 0))
        return EQ_ERR_ARG;
    EncParams P;
    memset(&P, 0, sizeof(P));
    P.codes = codes;
    P.payload = blk->payload;
    P.chunk_off = blk->chunk_off;
    P.sizes = chunk_sizes;
    P.freq = blk->freq;
    P.err = d_err;
    P.total = (unsigned long long*)payload_bytes_dev;
    P.payload_cap = blk->payload_cap;
    P.cs = blk->chunk_symbols;
    P.n_layers = blk->n_layers;
    uint64_t base = 0;
    uint32_t chunk = 0;
    for (uint32_t l = 0; l < blk->n_layers; ++l) {
        if (blk->layer_rows[l] < 1 || blk->layer_cols[l] < 1) return EQ_ERR_SHAPE;
        if (blk->chunk_mode == EQ_CHUNK_INTERLEAVED && blk->layer_cols[l] % 16 != 0) return EQ_ERR_SHAPE;
        const uint64_t sz = (uint64_t)blk->layer_rows[l] * (uint64_t)blk->layer_cols[l];
        P.chunk0[l] = chunk;
        P.sym_base[l] = base;
        P.geom[l] = chunk_geom(blk->chunk_mode, blk->layer_rows[l], blk->layer_cols[l], P.cs);
        chunk += (uint32_t)layer_chunks(blk->chunk_mode, blk->layer_rows[l], blk->layer_cols[l], P.cs);
        base += sz;
    }
    P.chunk0[blk->n_layers] = chunk;
    if (chunk != blk->n_chunks) return EQ_ERR_SHAPE;
    P.n_chunks = chunk;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned g = (chunk + kEncThreads - 1) / kEncThreads;
    if (blk->codec == EQ_CODEC_PAIR) {
        k_encode_pair<false, false><<<g, kEncThreads, 0, st>>>(P);
        k_scan<<<1, 1024, 0, st>>>(chunk_sizes, chunk, blk->chunk_off, P.total, d_err);
        k_encode_pair<true, false><<<g, kEncThreads, 0, st>>>(P);
    } else if (blk->codec == EQ_CODEC_PAIR_G) {
        k_encode_pair<false, true><<<g, kEncThreads, 0, st>>>(P);
        k_scan<<<1, 1024, 0, st>>>(chunk_sizes, chunk, blk->chunk_off, P.total, d_err);
        k_encode_pair<true, true><<<g, kEncThreads, 0, st>>>(P);
    } else if (blk->codec == EQ_CODEC_WORD) {
        k_encode<false, true><<<g, kEncThreads, 0, st>>>(P);
        k_scan<<<1, 1024, 0, st>>>(chunk_sizes, chunk, blk->chunk_off, P.total, d_err);
        k_encode<true, true><<<g, kEncThreads, 0, st>>>(P);
    } else {
        k_encode<false, false><<<g, kEncThreads, 0, st>>>(P);
        k_scan<<<1, 1024, 0, st>>>(chunk_sizes, chunk, blk->chunk_off, P.total, d_err);
        k_encode<true, false><<<g, kEncThreads, 0, st>>>(P);
    }
    EQ_CUDA_TRY(cudaGetLastError());
    return EQ_OK;
}
