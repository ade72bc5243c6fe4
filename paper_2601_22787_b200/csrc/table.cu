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
