// quant.cu — §8(a) rows a1-a4 on sm_100a:
//   a1 AbsMax init (Eq. 1; Alg. 1 l.1)
//   a2 per-row scale search minimising Eq. 4 over bf16 candidates (R4, R5)
//   a3 FP8-E4M3 quantisation (clamp before RNE, −0 → +0 per P:509)
//   a4 256-bin symbol histogram (metadata ℳ) fused into a3
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cmath>
#include <vector>

namespace eq {

constexpr int kRedThreads = 256;
constexpr int kSearchThreads = 256;
constexpr int kMaxLambda = 32;

// ---------------------------------------------------------------- a1: AbsMax
// |max| of a bf16 row is exact in f32; s0 = bf16(max/448): the f32 quotient is within
// 2^-24 of the exact one and m/448 (m with 8 significant bits) is never within 2^-12
// (relative) of a bf16 rounding midpoint unless exact, so bf16(fl32(max/448)) is the
// exact RNE.  All-zero row -> 1.0.
__device__ __forceinline__ uint16_t absmax_from_max(float m, float qmax) {
    return m == 0.f ? (uint16_t)0x3F80u : float_to_bf16_bits(__fdiv_rn(m, qmax));
}

__global__ void __launch_bounds__(kRedThreads)
k_absmax(const uint16_t* __restrict__ W, int64_t rows, int64_t cols, float qmax, uint16_t* __restrict__ s0) {
    const int64_t r = blockIdx.x;
    if (r >= rows) return;
    const uint16_t* row = W + r * cols;
    uint32_t m = 0;                      // max of |w| bit patterns (monotone for |bf16|)
    for (int64_t j = threadIdx.x; j < cols; j += kRedThreads) m = max(m, (uint32_t)(row[j] & 0x7FFFu));
    #pragma unroll
    for (int d = 16; d > 0; d >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, d));
    __shared__ uint32_t wm[kRedThreads / 32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kRedThreads / 32; ++w) m = max(m, wm[w]);
        s0[r] = absmax_from_max(bf16_bits_to_float(m), qmax);
    }
}

// ---------------------------------------------------------------- ‖W‖₁ (deterministic)
// Stage 1: each CTA sums a fixed range in a fixed tree order (f64); stage 2 sums the
// partials in index order.  Bitwise reproducible run to run.
__global__ void __launch_bounds__(kRedThreads)
k_l1_partial(const uint16_t* __restrict__ W, int64_t n, int64_t per_cta, double* __restrict__ part) {
    const int64_t a = (int64_t)blockIdx.x * per_cta, b = min(n, a + per_cta);
    double s = 0.0;
    for (int64_t j = a + threadIdx.x; j < b; j += kRedThreads) s += (double)fabsf(bf16_bits_to_float(W[j]));
    #pragma unroll
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, d);
    __shared__ double ws[kRedThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) t += ws[w];
        part[blockIdx.x] = t;
    }
}

__global__ void k_l1_final(const double* __restrict__ part, int n, double* __restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < n; ++i) t += part[i];
        *out = t;
    }
}

// ---------------------------------------------------------------- a2: scale search
struct SearchParams {
    const uint16_t* W;
    float qmax;
    int64_t rows, cols;
    const uint32_t* row_list;   // nullable
    uint32_t n_rows;
    int32_t oct_lo, oct_hi;
    uint32_t n_lambda;
    double lambda[kMaxLambda];
    const double* l1;           // device ‖W‖₁
    uint16_t* scales;           // [n_lambda][rows]
    double* obj;                // [n_lambda][rows] or null
};

// one exact term pair: |w − s·v| in f32 (exact: see DESIGN.md §6 K-SRCH), |v|·512 integer
template <uint32_t FMT>
__device__ __forceinline__ void term2(float w0, float w1, float s, double& D, uint32_t& R) {
    const uint32_t q = codes2<FMT>(__fdiv_rn(w0, s), __fdiv_rn(w1, s));
    const float2 v = values2<FMT>(q);
    D += (double)fabsf(__fsub_rn(w0, __fmul_rn(s, v.x)));
    D += (double)fabsf(__fsub_rn(w1, __fmul_rn(s, v.y)));
    R += (uint32_t)__fmul_rn(fabsf(v.x), 512.f) + (uint32_t)__fmul_rn(fabsf(v.y), 512.f);
}

#ifndef EQ_SEARCH_FAST
#define EQ_SEARCH_FAST 1
#endif
// Division-free E4M3 term pair (same codes as term2).  For bf16 w and s the
// exact quotient w/s is never within 2^-13 (relative) of an E4M3 rounding midpoint unless it
// equals one (§8c.3; pinned by the oracle tests).  q± = w·fl(fl(1/s)·(1 ± 2^-18)) lie within
// 2^-18 ± 3·2^-24 of w/s, strictly above / below it: off a midpoint both round like w/s; on a
// midpoint they round to the two neighbours and RNE takes the even one (the code with LSB 0).
// (The sign of a zero code does not matter here: ±0 give the same |w − s·v| and |v|.)
// R accumulates |v|·512 + 2^23 as f32 bits (exact integers < 2^23): the caller subtracts
// 0x4B000000 per term once.
__device__ __forceinline__ void term2_fast(float w0, float w1, float s, float rp, float rm, double& D, uint32_t& R) {
    const uint32_t cp = e4m3x2_sat(__fmul_rn(w0, rp), __fmul_rn(w1, rp));
    const uint32_t cm = e4m3x2_sat(__fmul_rn(w0, rm), __fmul_rn(w1, rm));
    const uint32_t odd = (cp & 0x0101u) * 0xFFu;                  // bytes of cp with LSB 1
    const uint32_t q = cp ^ ((cp ^ cm) & odd);                    // a tie byte takes the even code
    const float2 v = e4m3x2_to_float2(q);
    D += (double)fabsf(__fsub_rn(w0, __fmul_rn(s, v.x)));
    D += (double)fabsf(__fsub_rn(w1, __fmul_rn(s, v.y)));
    R += __float_as_uint(__fmaf_rn(fabsf(v.x), 512.f, 8388608.f)) + __float_as_uint(__fmaf_rn(fabsf(v.y), 512.f, 8388608.f));
}

__device__ __forceinline__ bool better(double f, uint32_t k, double bf, uint32_t bk) {
    return f < bf || (f == bf && k < bk);
}

// One CTA per searched row.  The row is staged in shared memory as f32 (exact bf16
// values); warps take candidates k = warp, warp+8, ...; lanes stride over the row; warp
// reduction in fixed order; per-λ best kept by lane 0, merged over warps at the end.
template <uint32_t FMT>
__global__ void __launch_bounds__(kSearchThreads)
k_search(const __grid_constant__ SearchParams P) {
    extern __shared__ float srow[];
    __shared__ double bestf[kSearchThreads / 32][kMaxLambda];
    __shared__ uint32_t bestk[kSearchThreads / 32][kMaxLambda];
    __shared__ uint32_t s_max;

    const uint32_t ri = blockIdx.x;
    if (ri >= P.n_rows) return;
    const int64_t r = P.row_list ? (int64_t)P.row_list[ri] : (int64_t)ri;
    const int64_t N = P.cols;
    const uint16_t* row = P.W + r * N;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;

    if (t == 0) s_max = 0;
    __syncthreads();
    uint32_t m = 0;
    for (int64_t j = t; j < N; j += kSearchThreads) {
        uint16_t b = row[j];
        srow[j] = bf16_bits_to_float(b);
        m = max(m, (uint32_t)(b & 0x7FFFu));
    }
    if (N & 1) if (t == 0) srow[N] = 0.f;          // pad for pairwise processing
    #pragma unroll
    for (int d = 16; d > 0; d >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, d));
    if (lane == 0) atomicMax(&s_max, m);
    __syncthreads();
    m = s_max;
    const uint16_t s0 = absmax_from_max(bf16_bits_to_float(m), P.qmax);
    if (m == 0) {                                   // all-zero row keeps s = 1
        if (t < (int)P.n_lambda) {
            P.scales[(int64_t)t * P.rows + r] = 0x3F80u;
            if (P.obj) P.obj[(int64_t)t * P.rows + r] = 0.0;
        }
        return;
    }
    // candidate bracket: bf16(s0·2^oct_lo) .. bf16(s0·2^oct_hi), clamped to finite > 0
    const float s0f = bf16_bits_to_float(s0);
    int lo = float_to_bf16_bits(ldexpf(s0f, P.oct_lo)), hi = float_to_bf16_bits(ldexpf(s0f, P.oct_hi));
    lo = max(lo, 1);
    hi = min(hi, 0x7F7F);
    if (hi < lo) hi = lo;
    {   // every candidate from the first s with max|w|/s ≤ the first rounding midpoint (2^-10 for
        // E4M3, ½ for Int8; a tie rounds to the even code 0) quantises the whole row to 0: equal
        // objectives, and the smallest of them wins ties, so the rest need no evaluation
        const float z = __fmul_rn(bf16_bits_to_float(m), FMT == EQ_FMT_INT8 ? 2.0f : 1024.0f);
        const uint32_t zb = __float_as_uint(z);
        const int hz = (int)((zb >> 16) + ((zb & 0xFFFFu) ? 1u : 0u));   // smallest bf16 ≥ z
        if (isfinite(z) && hz >= lo && hz < hi) hi = hz;
    }
    const uint32_t nc = (uint32_t)(hi - lo + 1);

    const double l1 = *P.l1;
    const double mn = (double)P.rows * (double)N;
    double my_bf[kMaxLambda];
    uint32_t my_bk[kMaxLambda];
    for (uint32_t q = 0; q < P.n_lambda; ++q) { my_bf[q] = INFINITY; my_bk[q] = 0xFFFFFFFFu; }

    const int64_t npair = (N + 1) >> 1;
    for (uint32_t k = warp; k < nc; k += kSearchThreads / 32) {
        const float s = bf16_bits_to_float((uint32_t)(lo + (int)k));
        double D = 0.0;
        uint32_t R = 0;
        // fast path: E4M3 and fl(1/s) normal with margin (uniform per warp: one candidate)
        if (EQ_SEARCH_FAST && FMT == EQ_FMT_E4M3 && s >= 0x1p-124f && s <= 0x1p124f) {
            const float r = __frcp_rn(s);
            const float rp = __fmul_rn(r, 1.0f + 0x1p-18f), rm = __fmul_rn(r, 1.0f - 0x1p-18f);
            uint32_t nt = 0;
            for (int64_t p = lane; p < npair; p += 32) {
                const float2 w = reinterpret_cast<const float2*>(srow)[p];
                term2_fast(w.x, w.y, s, rp, rm, D, R);
                nt += 2;
            }
            R -= nt * 0x4B000000u;                                // modulo 2^32: the exact Σ|v|·512
        } else {
            for (int64_t p = lane; p < npair; p += 32) {
                const float2 w = reinterpret_cast<const float2*>(srow)[p];
                term2<FMT>(w.x, w.y, s, D, R);
            }
        }
        unsigned long long R64 = R;                 // a 28672-wide row overflows u32
        #pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            D += __shfl_xor_sync(0xFFFFFFFFu, D, d);
            R64 += __shfl_xor_sync(0xFFFFFFFFu, R64, d);
        }
        // exact pad term: a zero pad quantises to 0 with zero error, adds nothing
        if (lane == 0) {
            // same operation order as Eq. 4 in the oracle: D/‖W‖₁ + (λ·R)/(M·N)
            const double Dd = l1 > 0.0 ? D / l1 : 0.0, Rd = (double)R64 * (1.0 / 512.0);
            for (uint32_t q = 0; q < P.n_lambda; ++q) {
                const double f = Dd + P.lambda[q] * Rd / mn;
                if (better(f, k, my_bf[q], my_bk[q])) { my_bf[q] = f; my_bk[q] = k; }
            }
        }
    }
    if (lane == 0)
        for (uint32_t q = 0; q < P.n_lambda; ++q) { bestf[warp][q] = my_bf[q]; bestk[warp][q] = my_bk[q]; }
    __syncthreads();
    if (t < (int)P.n_lambda) {
        double bf = bestf[0][t];
        uint32_t bk = bestk[0][t];
        for (int w = 1; w < kSearchThreads / 32; ++w)
            if (better(bestf[w][t], bestk[w][t], bf, bk)) { bf = bestf[w][t]; bk = bestk[w][t]; }
        P.scales[(int64_t)t * P.rows + r] = (uint16_t)(lo + (int)bk);
        if (P.obj) P.obj[(int64_t)t * P.rows + r] = bf;
    }
}

// ---------------------------------------------------------------- a3 + a4
// Quantise (exact-rounded f32 quotient -> cvt.rn.satfinite.e4m3) and histogram with
// per-warp shared sub-histograms; the dominant zero symbol is counted in a register.
constexpr int kQhThreads = 256;

template <uint32_t FMT>
__global__ void __launch_bounds__(kQhThreads)
k_quant_hist(const uint16_t* __restrict__ W, int64_t rows, int64_t cols, const uint16_t* __restrict__ S,
             const uint32_t* __restrict__ row_list, uint32_t n_rows, uint8_t* __restrict__ codes,
             unsigned long long* __restrict__ hist) {
    __shared__ uint32_t h[kQhThreads / 32][256];
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < (kQhThreads / 32) * 256; i += kQhThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t zeros = 0;
    // CTAs stride over rows (in row-list order); threads stride over column pairs
    const int64_t npair = (cols + 1) >> 1;
    for (int64_t ri = blockIdx.x; ri < (int64_t)n_rows; ri += gridDim.x) {
        const int64_t r = row_list ? (int64_t)row_list[ri] : ri;
        const float s = bf16_bits_to_float(S[r]);
        const uint16_t* wr = W + r * cols;
        uint8_t* cr = codes ? codes + r * cols : nullptr;
        for (int64_t p = t; p < npair; p += kQhThreads) {
            const int64_t j = 2 * p;
            const float w0 = bf16_bits_to_float(wr[j]);
            const bool two = (j + 1 < cols);
            const float w1 = two ? bf16_bits_to_float(wr[j + 1]) : 0.f;
            const uint32_t q = codes2<FMT>(__fdiv_rn(w0, s), __fdiv_rn(w1, s));
            const uint32_t c0 = q & 0xFFu, c1 = q >> 8;
            if (cr) {
                cr[j] = (uint8_t)c0;
                if (two) cr[j + 1] = (uint8_t)c1;
            }
            if (c0 == 0) ++zeros; else atomicAdd(&h[warp][c0], 1u);
            if (two) { if (c1 == 0) ++zeros; else atomicAdd(&h[warp][c1], 1u); }
        }
    }
    #pragma unroll
    for (int d = 16; d > 0; d >>= 1) zeros += __shfl_xor_sync(0xFFFFFFFFu, zeros, d);
    if ((t & 31) == 0) atomicAdd(&h[warp][0], zeros);
    __syncthreads();
    for (int c = t; c < 256; c += kQhThreads) {
        unsigned long long v = 0;
        for (int w = 0; w < kQhThreads / 32; ++w) v += h[w][c];
        if (v) atomicAdd(hist + c, v);
    }
}

}  // namespace eq

using namespace eq;

static eq_status check_tensor(const eq_tensor* w) {
    if (!w || !w->w) return EQ_ERR_ARG;
    if (w->rows < 1 || w->cols < 1 || w->rows > (1ll << 31) || w->cols > (1ll << 31)) return EQ_ERR_SHAPE;
    return EQ_OK;
}

static float qmax_of(uint32_t format) { return format == EQ_FMT_INT8 ? 127.f : 448.f; }

extern "C" eq_status eq_absmax(const eq_tensor* w, uint32_t format, uint16_t* s0, eq_stream_t stream) {
    EQ_TRY(check_tensor(w));
    if (!s0 || format > EQ_FMT_INT8) return EQ_ERR_ARG;
    k_absmax<<<(unsigned)w->rows, kRedThreads, 0, (cudaStream_t)stream>>>(
        (const uint16_t*)w->w, w->rows, w->cols, qmax_of(format), s0);
    EQ_CUDA_TRY(cudaGetLastError());
    return EQ_OK;
}

static int l1_ctas(int64_t n) { return (int)std::min<int64_t>(1184, (n + 4095) / 4096); }

namespace eq {
uint64_t l1_scratch_bytes(int64_t n) { return 8ull * (uint64_t)l1_ctas(n); }
eq_status l1_device(const uint16_t* W, int64_t n, double* out, void* part, cudaStream_t st) {
    const int nct = l1_ctas(n);
    const int64_t per = (n + nct - 1) / nct;
    k_l1_partial<<<nct, kRedThreads, 0, st>>>(W, n, per, (double*)part);
    k_l1_final<<<1, 32, 0, st>>>((const double*)part, nct, out);
    EQ_CUDA_TRY(cudaGetLastError());
    return EQ_OK;
}
}  // namespace eq

extern "C" uint64_t eq_search_scratch_bytes(const eq_tensor* w) {
    if (!w) return 0;
    return 256 + 8ull * (uint64_t)l1_ctas(w->rows * w->cols);
}

extern "C" eq_status eq_search_scales(const eq_tensor* w, uint32_t format, const double* lambdas_host, uint32_t n_lambda,
                                      int32_t oct_lo, int32_t oct_hi, const uint32_t* rows, uint32_t n_rows,
                                      uint16_t* scales, double* obj, void* scratch, uint64_t scratch_bytes,
                                      eq_stream_t stream) {
    EQ_TRY(check_tensor(w));
    if (!lambdas_host || n_lambda == 0 || n_lambda > (uint32_t)kMaxLambda || !scales || !scratch) return EQ_ERR_ARG;
    if (format > EQ_FMT_INT8) return EQ_ERR_ARG;
    if (oct_hi < oct_lo || oct_lo < -40 || oct_hi > 40) return EQ_ERR_ARG;
    for (uint32_t q = 0; q < n_lambda; ++q)
        if (!(lambdas_host[q] >= 0.0)) return EQ_ERR_ARG;
    if (scratch_bytes < eq_search_scratch_bytes(w)) return EQ_ERR_BUFFER;
    const int64_t n = w->rows * w->cols;
    const uint64_t smem = (uint64_t)((w->cols + 2) & ~1ll) * 4;
    if (smem > 200 * 1024) return EQ_ERR_SHAPE;            // rows up to 51200 columns
    cudaStream_t st = (cudaStream_t)stream;
    double* l1 = (double*)scratch;
    double* part = (double*)((char*)scratch + 256);
    const int nct = l1_ctas(n);
    const int64_t per = (n + nct - 1) / nct;
    k_l1_partial<<<nct, kRedThreads, 0, st>>>((const uint16_t*)w->w, n, per, part);
    k_l1_final<<<1, 32, 0, st>>>(part, nct, l1);
    SearchParams P;
    P.W = (const uint16_t*)w->w;
    P.qmax = qmax_of(format);
    P.rows = w->rows;
    P.cols = w->cols;
    P.row_list = rows;
    P.n_rows = rows ? n_rows : (uint32_t)w->rows;
    P.oct_lo = oct_lo;
    P.oct_hi = oct_hi;
    P.n_lambda = n_lambda;
    for (int q = 0; q < kMaxLambda; ++q) P.lambda[q] = q < (int)n_lambda ? lambdas_host[q] : 0.0;
    P.l1 = l1;
    P.scales = scales;
    P.obj = obj;
    if (P.n_rows == 0) return EQ_OK;
    if (format == EQ_FMT_INT8) {
        EQ_CUDA_TRY(cudaFuncSetAttribute(k_search<EQ_FMT_INT8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_search<EQ_FMT_INT8><<<P.n_rows, kSearchThreads, smem, st>>>(P);
    } else {
        EQ_CUDA_TRY(cudaFuncSetAttribute(k_search<EQ_FMT_E4M3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_search<EQ_FMT_E4M3><<<P.n_rows, kSearchThreads, smem, st>>>(P);
    }
    EQ_CUDA_TRY(cudaGetLastError());
    return EQ_OK;
}

extern "C" eq_status eq_quantize_hist(const eq_tensor* w, uint32_t format, const uint16_t* scales, const uint32_t* rows,
                                      uint32_t n_rows, uint8_t* codes, uint64_t* hist, eq_stream_t stream) {
    EQ_TRY(check_tensor(w));
    if (!scales || !hist || format > EQ_FMT_INT8) return EQ_ERR_ARG;
    const uint32_t nr = rows ? n_rows : (uint32_t)w->rows;
    if (nr == 0) return EQ_OK;
    const int ctas = (int)std::min<int64_t>(148 * 8, nr);
    if (format == EQ_FMT_INT8)
        k_quant_hist<EQ_FMT_INT8><<<ctas, kQhThreads, 0, (cudaStream_t)stream>>>(
            (const uint16_t*)w->w, w->rows, w->cols, scales, rows, nr, codes, (unsigned long long*)hist);
    else
        k_quant_hist<EQ_FMT_E4M3><<<ctas, kQhThreads, 0, (cudaStream_t)stream>>>(
            (const uint16_t*)w->w, w->rows, w->cols, scales, rows, nr, codes, (unsigned long long*)hist);
    EQ_CUDA_TRY(cudaGetLastError());
    return EQ_OK;
}
