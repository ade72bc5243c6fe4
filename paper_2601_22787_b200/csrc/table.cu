// table.cu — §8(a) row a5: normalise the block's 256-bin histogram to a 12-bit frequency
// table (metadata ℳ) with the integer-only largest-remainder rule of
// reading R8 (SPEC's literal "residual to the largest" rule can go negative):
//   1. f_s = c_s>0 ? max(1, ⌊4096 c_s/T⌋) : 0,  r_s = (4096 c_s) mod T
//   2. D = 4096 − Σf
//   3. D > 0: +1 to the D present symbols with the largest r_s (ties: larger c_s, lower code)
//   4. while D < 0: −1 from the largest f_s with f_s > 1 (ties: lower code)
// One CTA of 256 threads, one thread per symbol.
#include "common.cuh"

namespace eq {

__global__ void __launch_bounds__(256)
k_build_table(const unsigned long long* __restrict__ hist, uint16_t* __restrict__ freq, uint32_t* err) {
    __shared__ unsigned long long c[256], r[256];
    __shared__ unsigned long long red[8];
    __shared__ long long s_sum;
    __shared__ unsigned s_key;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const unsigned long long ct = hist[t];
    c[t] = ct;
    // T = Σ c
    unsigned long long v = ct;
    #pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    unsigned long long T = 0;
    for (int w = 0; w < 8; ++w) T += red[w];
    if (T == 0) {
        freq[t] = 0;
        if (t == 0) atomicOr(err, EQ_EF_EMPTY);
        return;
    }
    const unsigned long long num = (unsigned long long)kM * ct;     // ct < 2^52
    const unsigned long long q = num / T;
    r[t] = num % T;
    long long f = ct ? (q < 1 ? 1 : (long long)q) : 0;
    // D = 4096 − Σ f
    if (t == 0) s_sum = 0;
    __syncthreads();
    atomicAdd((unsigned long long*)&s_sum, (unsigned long long)f);
    __syncthreads();
    long long D = (long long)kM - s_sum;
    if (D > 0 && ct) {
        const unsigned long long rt = r[t];
        long long rank = 0;
        for (int u = 0; u < 256; ++u) {
            if (!c[u] || u == t) continue;
            const bool ahead = r[u] > rt || (r[u] == rt && (c[u] > ct || (c[u] == ct && u < t)));
            rank += ahead;
        }
        if (rank < D) f += 1;
    }
    while (D < 0) {                             // block-uniform loop
        if (t == 0) s_key = 0;
        __syncthreads();
        const unsigned key = f > 1 ? ((unsigned)f << 8) | (unsigned)(255 - t) : 0u;
        atomicMax(&s_key, key);
        __syncthreads();
        if (s_key != 0 && t == 255 - (int)(s_key & 255u)) f -= 1;
        ++D;
        __syncthreads();
    }
    freq[t] = (uint16_t)f;
}

}  // namespace eq

extern "C" eq_status eq_build_table(const uint64_t* hist, uint16_t* freq, uint32_t* d_err, eq_stream_t stream) {
    if (!hist || !freq || !d_err) return EQ_ERR_ARG;
    eq::k_build_table<<<1, 256, 0, (cudaStream_t)stream>>>((const unsigned long long*)hist, freq, d_err);
    EQ_CUDA_TRY(cudaGetLastError());
    return EQ_OK;
}

// ---------------------------------------------------------------------------------------------
// §8(a) row a5 for EQ_CODEC_PAIR (reading R15): the pair table of one block, built
// on the device from the block histogram so eq_quantize_encode never leaves the stream.
// Written from R15's statement, as a parallel construction over one CTA of 256 threads:
//  * ranks — a present code's rank is the number of present codes that precede it (larger
//    count, or equal count and lower code); ranks 0..K−1, K = min(15, #present), name the codes;
//  * pair weights — slot q = ra·15 + rb holds c(code_ra)·c(code_rb); a pair is kept iff its ideal
//    frequency is ≥ 1/32 slot, 32·M·w ≥ T²; the escape carries T² − Σ kept (entry 225);
//  * R8 over the 226-entry vector, total W = T²: floors max(1, ⌊M·w/W⌋) of the present entries;
//    D > 0 — an entry gets +1 iff fewer than D present entries beat its key (remainder, weight,
//    lower index); D < 0 — "take one from the current largest, ties to the lower index", |D|
//    times, equals water-filling: the smallest level v with Σ max(0, f − v) ≤ |D| (bisection),
//    every entry above v lands on v, and the R = |D| − Σ max(0, f − v) lowest-indexed entries
//    with f ≥ v go one lower.
// Output (include/entquant.h, EQ_CODEC_PAIR): tab[256 + q] pair frequency (0 = not kept or rank
// ≥ K), tab[481] escape frequency, tab[482] K, tab[484..492) the 16 rank codes as bytes (unused
// ranks 0), every other entry of tab[256..512) zero.  Counts of one block are < 2^50 (ABI limits:
// < 2^32 chunks of ≤ 2^18 symbols), so T² < 2^100 and M·w < 2^112 fit in 128 bits.
namespace eq {

typedef unsigned __int128 u128;

// 256-thread block sum of a u128 (two u64 halves with carry through a shared array)
__device__ __forceinline__ u128 block_sum_u128(u128 v, u128* sh) {
    const int t = threadIdx.x;
    sh[t] = v;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (t < s) sh[t] += sh[t + s];
        __syncthreads();
    }
    const u128 r = sh[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ long long block_sum_ll(long long v, long long* sh8) {
    #pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, d);
    if ((threadIdx.x & 31) == 0) sh8[threadIdx.x >> 5] = v;
    __syncthreads();
    long long s = 0;
    #pragma unroll
    for (int w = 0; w < 8; ++w) s += sh8[w];
    __syncthreads();
    return s;
}

__global__ void __launch_bounds__(256)
k_build_pair_table(const unsigned long long* __restrict__ hist, uint16_t* __restrict__ tab, uint32_t* err) {
    constexpr int kNP = 225, kNV = 226;              // pairs, pairs + escape
    __shared__ unsigned long long cnt[256];
    __shared__ uint32_t rank_code[16];
    __shared__ u128 wv[kNV], rv[kNV];
    __shared__ int fv[kNV];
    __shared__ u128 red[256];
    __shared__ long long red8[8];
    const int t = threadIdx.x;
    const unsigned long long ct = hist[t];
    cnt[t] = ct;
    if (t < 16) rank_code[t] = 0;
    __syncthreads();
    const u128 T = block_sum_u128((u128)ct, red);
    if (T == 0) {                                  // empty block: k_build_table reports it
        tab[256 + t] = 0;
        if (t == 0) atomicOr(err, EQ_EF_EMPTY);
        return;
    }
    // ---- ranks (present codes only)
    const long long n_present = block_sum_ll(ct ? 1 : 0, red8);
    if (ct) {
        int rank = 0;
        for (int u = 0; u < 256; ++u) {
            const unsigned long long cu = cnt[u];
            rank += (cu > ct || (cu == ct && u < t)) ? 1 : 0;     // absent codes (0) never precede
        }
        if (rank < 15) rank_code[rank] = (uint32_t)t;
    }
    const int K = n_present < 15 ? (int)n_present : 15;
    __syncthreads();
    // ---- pair weights and the keep rule
    const u128 W = T * T;
    u128 w = 0;
    if (t < kNP) {
        const int ra = t / 15, rb = t % 15;
        if (ra < K && rb < K) {
            const u128 x = (u128)cnt[rank_code[ra]] * (u128)cnt[rank_code[rb]];
            if ((u128)32 * kM * x >= W) w = x;   // ideal frequency ≥ 1/32 slot
        }
    }
    const u128 kept = block_sum_u128(w, red);
    if (t < kNP) wv[t] = w;
    if (t == kNP) wv[t] = W - kept;               // escape: every pair not kept
    __syncthreads();
    // ---- R8 floors and remainders over the 226 entries
    int f = 0;
    if (t < kNV && wv[t] != 0) {
        const u128 num = (u128)kM * wv[t];
        const u128 q = num / W;
        rv[t] = num - q * W;
        f = q < 1 ? 1 : (int)q;
    } else if (t < kNV) {
        rv[t] = 0;
    }
    const long long D = (long long)kM - block_sum_ll(f, red8);
    if (D > 0 && t < kNV && wv[t] != 0) {
        const u128 ri = rv[t], wi = wv[t];
        long long ahead = 0;
        for (int j = 0; j < kNV; ++j) {
            if (j == t || wv[j] == 0) continue;
            ahead += (rv[j] > ri || (rv[j] == ri && (wv[j] > wi || (wv[j] == wi && j < t)))) ? 1 : 0;
        }
        if (ahead < D) f += 1;
    }
    if (D < 0) {                                   // block-uniform: water-filling from the top
        const long long S = -D;
        int lo = 1, hi = (int)kM;                  // smallest v with cost(v) <= S (cost(kM) = 0)
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            const long long cost = block_sum_ll(f > mid ? f - mid : 0, red8);
            if (cost <= S) hi = mid; else lo = mid + 1;
        }
        const int v = lo;
        const long long R = S - block_sum_ll(f > v ? f - v : 0, red8);
        if (t < kNV) fv[t] = f;
        __syncthreads();
        if (t < kNV && f >= v) {
            long long before = 0;                  // entries with f ≥ v at lower indices
            for (int j = 0; j < t; ++j) before += fv[j] >= v ? 1 : 0;
            f = before < R ? v - 1 : v;
        }
    }
    // ---- output: tab[256 + t], t < 256
    uint32_t out = 0;
    if (t < kNP) out = (uint32_t)f;
    else if (t == kNP) out = (uint32_t)f;          // escape frequency (0 when every pair is kept)
    else if (t == 226) out = (uint32_t)K;
    else if (t >= 228 && t < 236) out = rank_code[2 * (t - 228)] | (rank_code[2 * (t - 228) + 1] << 8);
    tab[256 + t] = (uint16_t)out;
}

}  // namespace eq

extern "C" eq_status eq_build_pair_table(const uint64_t* hist, uint16_t* table, uint32_t* d_err, eq_stream_t stream) {
    if (!hist || !table || !d_err) return EQ_ERR_ARG;
    eq::k_build_pair_table<<<1, 256, 0, (cudaStream_t)stream>>>((const unsigned long long*)hist, table, d_err);
    EQ_CUDA_TRY(cudaGetLastError());
    return EQ_OK;
}
