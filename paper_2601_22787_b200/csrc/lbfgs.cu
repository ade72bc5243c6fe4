// lbfgs.cu — §8(f) NEXT row 3: the paper's solver for Eq. 4: per layer,
// L-BFGS over the per-channel scales only, straight-through gradients through Q_γ,
// initialised with AbsMax, learning rate 0.25 for λ > 30 and 1.0 otherwise.
// Reading R13: variables u = log2 s, evaluated scale s = RNE_bf16(2^u)
// (R7), objective = the true discrete Eq. 4 (R4), Armijo backtracking (c1 = 1e-4,
// α_t = α0·2^-t, ≤ max_backtracks), two-loop recursion with history m, H0 = γI.
//
// GPU structure (one call optimises up to EQ_MAX_LAYERS layers, each independently):
//   k_lb_eval    one CTA per weight row: the row is staged in shared memory once and the
//                objective sums and STE gradient are accumulated for `trials` step lengths
//                of the current direction in one pass (fp64 terms, fixed-order reduction);
//   k_lb_update  one CTA per layer: picks the first trial meeting Armijo, updates u, g, the
//                curvature history and the objective trace, then computes the next
//                direction by the two-loop recursion (block reductions in fixed order).
// All decisions stay on the device; the host only polls a done flag every few passes.
// Every term is the same exact or correctly rounded f64 operation as in the oracle
// (the CPU oracle under oracle/); only summation order differs.
#include "common.cuh"
#include "internal.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

namespace eq {

constexpr int kEvThreads = 256;
constexpr int kUpThreads = 1024;
constexpr int kMaxTrials = 8;
constexpr int kMaxHist = 32;
constexpr double kLn2 = 0.6931471805599453;   // fp64 ln 2 (= Python math.log(2.0))

struct LayerState {
    double F, gd, a0, l1, mn;
    double rho[kMaxHist + 1];            // by ring slot
    uint32_t tb;          // backtracks already evaluated this iteration
    uint32_t iter;        // accepted steps
    uint32_t hist_n, hist_head;
    uint32_t done, converged, passes, pad;
};

struct LbParams {
    const uint16_t* w[EQ_MAX_LAYERS];
    int64_t cols[EQ_MAX_LAYERS];
    uint32_t row0[EQ_MAX_LAYERS + 1];   // prefix of rows over layers
    uint32_t n_layers, R;
    double lambda, lr, c1, grad_tol, change_tol;
    uint32_t max_iters, history, trials, max_backtracks;
    double *u, *g, *d, *q;                // [R]
    double *S, *Y;                        // [history + 1][R] ring (one free staging slot)
    double *tD, *tR, *tG;                 // [trials][R]
    LayerState* st;                       // [n_layers]
    double* trace;                        // [n_layers][max_iters + 1]
    uint32_t* done_flags;                 // [n_layers]
};

__device__ __forceinline__ uint32_t layer_of_row(const LbParams& P, uint32_t r) {
    uint32_t l = 0;
    for (uint32_t q = 1; q < P.n_layers; ++q)
        if (r >= P.row0[q]) l = q;
    return l;
}

// s = RNE_bf16(2^u): bit pattern
__device__ __forceinline__ uint16_t bf16_of_exp2(double u) {
    __nv_bfloat16 h = __double2bfloat16(exp2(u));
    return *reinterpret_cast<uint16_t*>(&h);
}

// ---------------------------------------------------------------- block reductions
// fixed order: warp shuffle tree, then warp partials summed by warp 0 in a tree
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double r = 0.0;
    if (warp == 0) {
        r = lane < NT / 32 ? sh[lane] : 0.0;
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xFFFFFFFFu, r, o);
        if (lane == 0) sh[32] = r;
    }
    __syncthreads();
    return sh[32];
}

template <int NT>
__device__ __forceinline__ double block_max(double v, double* sh) {
    #pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
        double r = lane < NT / 32 ? sh[lane] : 0.0;
        #pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xFFFFFFFFu, r, o));
        if (lane == 0) sh[32] = r;
    }
    __syncthreads();
    return sh[32];
}

// ---------------------------------------------------------------- init: u = log2(s0)
__global__ void k_lb_init(const LbParams P, const uint16_t* __restrict__ s0, const double* __restrict__ l1) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < P.R) {
        P.u[r] = log2((double)bf16_bits_to_float(s0[r]));
        P.d[r] = 0.0;
    }
    if (r < P.n_layers) {
        LayerState& S = P.st[r];
        S.F = 0.0;
        S.gd = 0.0;
        S.a0 = 0.0;
        S.l1 = l1[r];
        S.mn = (double)(P.row0[r + 1] - P.row0[r]) * (double)P.cols[r];
        S.tb = 0;
        S.iter = 0;
        S.hist_n = 0;
        S.hist_head = 0;
        S.done = 0;
        S.converged = 0;
        S.passes = 0;
        P.done_flags[r] = 0;
    }
}

// ---------------------------------------------------------------- objective + STE gradient
// Row sums {D, R, A, B, Q} at ntrial scales s_t = bf16(2^(u + α_t·d)).
template <uint32_t FMT>
__global__ void __launch_bounds__(kEvThreads) k_lb_eval(const __grid_constant__ LbParams P, uint32_t ntrial,
                                                        int first) {
    extern __shared__ uint16_t srow[];
    __shared__ double sh[33];
    const uint32_t r = blockIdx.x;
    const uint32_t l = layer_of_row(P, r);
    const LayerState& S = P.st[l];
    if (S.done) return;
    const int64_t N = P.cols[l];
    const uint16_t* row = P.w[l] + (int64_t)(r - P.row0[l]) * N;
    for (int64_t j = threadIdx.x; j < N; j += kEvThreads) srow[j] = row[j];
    __syncthreads();
    const double qmax = FMT == EQ_FMT_INT8 ? 127.0 : 448.0;
    const double ur = P.u[r], dr = P.d[r];
    for (uint32_t t = 0; t < ntrial; ++t) {
        double un = ur;
        if (!first) un = ur + ldexp(S.a0, -(int)(S.tb + t)) * dr;       // x + a·d (oracle order)
        const uint16_t sb = bf16_of_exp2(un);
        const double s = (double)bf16_bits_to_float(sb);
        double D = 0.0, Rr = 0.0, A = 0.0, B = 0.0, Q = 0.0;
        for (int64_t j = threadIdx.x; j < N; j += kEvThreads) {
            const double w = (double)bf16_bits_to_float(srow[j]);
            const double q = w / s;
            // the code from fl32(q): the exact quotient is never within 2^-13 (E4M3) / 2^-9
            // (Int8) relative of a rounding midpoint unless exactly on it
            const double v = (double)values2<FMT>(codes2<FMT>((float)q, 0.f)).x;
            const double e = s * v - w;
            D += fabs(e);
            Rr += fabs(v);
            if (fabs(q) <= qmax) {
                A += fabs(v - q);
                if (v != 0.0) Q += fabs(q);
            } else {
                B += (e > 0.0 ? 1.0 : e < 0.0 ? -1.0 : 0.0) * v;
            }
        }
        D = block_sum<kEvThreads>(D, sh);
        Rr = block_sum<kEvThreads>(Rr, sh);
        A = block_sum<kEvThreads>(A, sh);
        B = block_sum<kEvThreads>(B, sh);
        Q = block_sum<kEvThreads>(Q, sh);
        if (threadIdx.x == 0) {
            const uint64_t o = (uint64_t)t * P.R + r;
            P.tD[o] = D;
            P.tR[o] = Rr;
            const double first_term = S.l1 > 0.0 ? s * (A + B) / S.l1 : 0.0 * s;
            P.tG[o] = kLn2 * (first_term - P.lambda * Q / S.mn);
        }
    }
}

// ---------------------------------------------------------------- L-BFGS state update
// ring of m + 1 slots: k = 0 oldest .. hist_n-1 newest; slot k = hist_n is always free
__device__ __forceinline__ uint32_t hist_slot(const LayerState& S, uint32_t k, uint32_t m) {
    return (S.hist_head + k) % (m + 1);
}

__global__ void __launch_bounds__(kUpThreads) k_lb_update(const __grid_constant__ LbParams P, uint32_t ntrial,
                                                          int first) {
    __shared__ double sh[33];
    __shared__ double sF[kMaxTrials];
    __shared__ double alpha[kMaxHist];
    __shared__ int s_acc;
    const uint32_t l = blockIdx.x;
    LayerState& S = P.st[l];
    if (S.done) return;
    const uint32_t r0 = P.row0[l], r1 = P.row0[l + 1], R = P.R, m = P.history;
    const int tid = threadIdx.x;
    double* trace = P.trace ? P.trace + (uint64_t)l * (P.max_iters + 1) : nullptr;
    if (tid == 0) S.passes += 1;

    // ---- Armijo selection over this pass's trials (or the initial evaluation)
    for (uint32_t t = 0; t < ntrial; ++t) {
        double d = 0.0, rr = 0.0;
        for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) {
            d += P.tD[(uint64_t)t * R + r];
            rr += P.tR[(uint64_t)t * R + r];
        }
        d = block_sum<kUpThreads>(d, sh);
        rr = block_sum<kUpThreads>(rr, sh);
        if (tid == 0) sF[t] = (S.l1 > 0.0 ? d / S.l1 : 0.0) + P.lambda * rr / S.mn;
    }
    __syncthreads();
    if (first) {
        for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) P.g[r] = P.tG[r];
        if (tid == 0) {
            S.F = sF[0];
            if (trace) trace[0] = S.F;
        }
    } else {
        if (tid == 0) {
            int acc = -1;
            for (uint32_t t = 0; t < ntrial && S.tb + t < P.max_backtracks; ++t) {
                const double a = ldexp(S.a0, -(int)(S.tb + t));
                if (sF[t] <= S.F + P.c1 * a * S.gd) { acc = (int)t; break; }
            }
            s_acc = acc;
        }
        __syncthreads();
        const int acc = s_acc;
        if (acc < 0) {
            if (tid == 0) {
                S.tb += ntrial;
                if (S.tb >= P.max_backtracks) {      // line search failed
                    S.done = 1;
                    S.converged = 0;
                    P.done_flags[l] = 1;
                }
            }
            return;
        }
        // accept: u <- u + a·d, curvature pair (s_k, y_k)
        const double a = ldexp(S.a0, -(int)(S.tb + (uint32_t)acc));
        const uint32_t slot = hist_slot(S, S.hist_n, m);       // free staging slot
        double ys = 0.0, smax = 0.0;
        for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) {
            const double un = P.u[r] + a * P.d[r];
            const double sk = un - P.u[r];
            const double gn = P.tG[(uint64_t)acc * R + r];
            const double yk = gn - P.g[r];
            ys += sk * yk;
            smax = fmax(smax, fabs(sk));
            P.S[(uint64_t)slot * R + r] = sk;         // staged; kept only if ys > 1e-10
            P.Y[(uint64_t)slot * R + r] = yk;
            P.u[r] = un;
            P.g[r] = gn;
        }
        ys = block_sum<kUpThreads>(ys, sh);
        smax = block_max<kUpThreads>(smax, sh);
        if (tid == 0) {
            if (ys > 1e-10) {                                  // keep the pair (torch rule)
                S.rho[slot] = 1.0 / ys;
                if (S.hist_n < m) {
                    S.hist_n += 1;
                } else {
                    S.hist_head = (S.hist_head + 1) % (m + 1);  // drop the oldest
                }
            }
            const double dF = S.F - sF[acc];
            S.F = sF[acc];
            S.iter += 1;
            if (trace) trace[S.iter] = S.F;
            if (fabs(dF) < P.change_tol || smax <= P.change_tol) {
                S.done = 1;
                S.converged = 1;
            } else if (S.iter >= P.max_iters) {
                S.done = 1;
                S.converged = 0;
            }
            if (S.done) P.done_flags[l] = 1;
        }
        __syncthreads();
        if (S.done) return;
    }
    // ---- next direction
    double gmax = 0.0;
    for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) gmax = fmax(gmax, fabs(P.g[r]));
    gmax = block_max<kUpThreads>(gmax, sh);
    if (gmax <= P.grad_tol) {
        if (tid == 0) {
            S.done = 1;
            S.converged = 1;
            P.done_flags[l] = 1;
        }
        return;
    }
    const uint32_t hn = S.hist_n;
    if (hn == 0) {
        for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) P.d[r] = -P.g[r];
    } else {
        for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) P.q[r] = -P.g[r];
        for (int k = (int)hn - 1; k >= 0; --k) {               // newest -> oldest
            const uint32_t sl = hist_slot(S, (uint32_t)k, m);
            double dot = 0.0;
            for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) dot += P.S[(uint64_t)sl * R + r] * P.q[r];
            dot = block_sum<kUpThreads>(dot, sh);
            const double al = S.rho[sl] * dot;
            if (tid == 0) alpha[k] = al;
            for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) P.q[r] = P.q[r] - al * P.Y[(uint64_t)sl * R + r];
        }
        // H0 = γ I, γ = sᵀy / yᵀy of the newest pair
        const uint32_t sn = hist_slot(S, hn - 1, m);
        double sy = 0.0, yy = 0.0;
        for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) {
            const double yv = P.Y[(uint64_t)sn * R + r];
            sy += P.S[(uint64_t)sn * R + r] * yv;
            yy += yv * yv;
        }
        sy = block_sum<kUpThreads>(sy, sh);
        yy = block_sum<kUpThreads>(yy, sh);
        const double gam = sy / yy;
        for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) P.d[r] = P.q[r] * gam;
        __syncthreads();
        for (uint32_t k = 0; k < hn; ++k) {                       // oldest -> newest
            const uint32_t sl = hist_slot(S, k, m);
            double dot = 0.0;
            for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) dot += P.Y[(uint64_t)sl * R + r] * P.d[r];
            dot = block_sum<kUpThreads>(dot, sh);
            const double b = S.rho[sl] * dot;
            const double ab = alpha[k] - b;
            for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) P.d[r] = P.d[r] + P.S[(uint64_t)sl * R + r] * ab;
        }
    }
    double gd = 0.0;
    for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) gd += P.g[r] * P.d[r];
    gd = block_sum<kUpThreads>(gd, sh);
    bool sd = hn == 0;
    if (gd >= 0.0) {                                            // not a descent direction
        sd = true;
        for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) P.d[r] = -P.g[r];
        gd = 0.0;
        for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) gd += P.g[r] * P.d[r];
        gd = block_sum<kUpThreads>(gd, sh);
    }
    double dmax = 0.0;
    if (sd) {
        for (uint32_t r = r0 + tid; r < r1; r += kUpThreads) dmax = fmax(dmax, fabs(P.d[r]));
        dmax = block_max<kUpThreads>(dmax, sh);
    }
    if (tid == 0) {
        if (sd) S.hist_n = 0;
        S.gd = gd;
        S.a0 = sd ? P.lr / dmax : P.lr;
        S.tb = 0;
    }
}

__global__ void k_lb_final(const LbParams P, uint16_t* __restrict__ scales, uint32_t* __restrict__ info) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < P.R) scales[r] = bf16_of_exp2(P.u[r]);
    if (info && r < P.n_layers) {
        info[4 * r + 0] = P.st[r].iter;
        info[4 * r + 1] = P.st[r].converged;
        info[4 * r + 2] = P.st[r].passes;
        info[4 * r + 3] = P.st[r].done;
    }
}

// ---------------------------------------------------------------- host side
struct LbLayout {
    uint64_t u, g, d, q, S, Y, tD, tR, tG, st, l1, part, s0, flags, total;
};

static uint64_t al256(uint64_t x) { return (x + 255) & ~255ull; }

static LbLayout lb_layout(const eq_tensor* layers, uint32_t n, uint32_t history, uint32_t trials) {
    LbLayout L;
    uint64_t R = 0, part = 0;
    for (uint32_t i = 0; i < n; ++i) {
        R += (uint64_t)layers[i].rows;
        part = std::max<uint64_t>(part, l1_scratch_bytes(layers[i].rows * layers[i].cols));
    }
    uint64_t o = 0;
    auto take = [&](uint64_t bytes) { const uint64_t a = o; o = al256(o + bytes); return a; };
    L.u = take(8 * R);
    L.g = take(8 * R);
    L.d = take(8 * R);
    L.q = take(8 * R);
    L.S = take(8 * R * (history + 1));
    L.Y = take(8 * R * (history + 1));
    L.tD = take(8 * R * trials);
    L.tR = take(8 * R * trials);
    L.tG = take(8 * R * trials);
    L.st = take(sizeof(LayerState) * EQ_MAX_LAYERS);
    L.l1 = take(8 * EQ_MAX_LAYERS);
    L.part = take(part);
    L.s0 = take(2 * R);
    L.flags = take(4 * EQ_MAX_LAYERS);
    L.total = o;
    return L;
}

static eq_status lb_check(const eq_tensor* layers, uint32_t n, uint32_t format, double lambda,
                          const eq_lbfgs_params* p) {
    if (!layers || n < 1 || n > EQ_MAX_LAYERS || format > EQ_FMT_INT8 || !(lambda >= 0.0)) return EQ_ERR_ARG;
    if (p) {
        if (p->history < 1 || p->history > (uint32_t)kMaxHist || p->trials < 1 || p->trials > (uint32_t)kMaxTrials ||
            p->max_backtracks < 1 || p->max_backtracks > 1000 || !(p->c1 > 0.0 && p->c1 < 1.0) ||
            !(p->grad_tol >= 0.0) || !(p->change_tol >= 0.0) || !(p->lr >= 0.0))
            return EQ_ERR_ARG;
    }
    uint64_t R = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (!layers[i].w) return EQ_ERR_ARG;
        if (layers[i].rows < 1 || layers[i].cols < 1 || layers[i].cols > 100000) return EQ_ERR_SHAPE;
        R += (uint64_t)layers[i].rows;
    }
    if (R > (1ull << 31)) return EQ_ERR_SHAPE;
    return EQ_OK;
}

static eq_lbfgs_params lb_defaults() {
    eq_lbfgs_params d;
    d.max_iters = 100;
    d.history = 10;
    d.trials = 4;
    d.max_backtracks = 32;
    d.lr = 0.0;
    d.c1 = 1e-4;
    d.grad_tol = 1e-7;
    d.change_tol = 1e-9;
    return d;
}

// run init + the first evaluation; then (if iterate) the L-BFGS passes
static eq_status lb_run(const eq_tensor* layers, uint32_t n, uint32_t format, double lambda, const eq_lbfgs_params& p,
                        const uint16_t* given_scales, bool iterate, LbParams& P, const LbLayout& L, char* base,
                        double* trace, cudaStream_t st) {
    memset(&P, 0, sizeof(P));
    uint32_t R = 0;
    int64_t max_cols = 0;
    for (uint32_t i = 0; i < n; ++i) {
        P.w[i] = (const uint16_t*)layers[i].w;
        P.cols[i] = layers[i].cols;
        P.row0[i] = R;
        R += (uint32_t)layers[i].rows;
        max_cols = std::max(max_cols, layers[i].cols);
    }
    P.row0[n] = R;
    P.n_layers = n;
    P.R = R;
    P.lambda = lambda;
    P.lr = p.lr > 0.0 ? p.lr : (lambda > 30.0 ? 0.25 : 1.0);
    P.c1 = p.c1;
    P.grad_tol = p.grad_tol;
    P.change_tol = p.change_tol;
    P.max_iters = p.max_iters;
    P.history = p.history;
    P.trials = p.trials;
    P.max_backtracks = p.max_backtracks;
    P.u = (double*)(base + L.u);
    P.g = (double*)(base + L.g);
    P.d = (double*)(base + L.d);
    P.q = (double*)(base + L.q);
    P.S = (double*)(base + L.S);
    P.Y = (double*)(base + L.Y);
    P.tD = (double*)(base + L.tD);
    P.tR = (double*)(base + L.tR);
    P.tG = (double*)(base + L.tG);
    P.st = (LayerState*)(base + L.st);
    P.trace = trace;
    P.done_flags = (uint32_t*)(base + L.flags);
    double* l1 = (double*)(base + L.l1);
    uint16_t* s0 = (uint16_t*)(base + L.s0);
    for (uint32_t i = 0; i < n; ++i) {
        EQ_TRY(l1_device(P.w[i], layers[i].rows * layers[i].cols, l1 + i, base + L.part, st));
        if (given_scales) {
            EQ_CUDA_TRY(cudaMemcpyAsync(s0 + P.row0[i], given_scales + P.row0[i], 2 * layers[i].rows,
                                        cudaMemcpyDeviceToDevice, st));
        } else {
            EQ_TRY(eq_absmax(&layers[i], format, s0 + P.row0[i], st));
        }
    }
    if (trace) EQ_CUDA_TRY(cudaMemsetAsync(trace, 0xFF, 8ull * n * (p.max_iters + 1), st));   // NaN
    k_lb_init<<<(R + 255) / 256, 256, 0, st>>>(P, s0, l1);
    const size_t smem = (size_t)max_cols * 2;
    auto eval = [&](uint32_t nt, int first) -> eq_status {
        if (format == EQ_FMT_INT8) {
            EQ_CUDA_TRY(cudaFuncSetAttribute(k_lb_eval<EQ_FMT_INT8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_lb_eval<EQ_FMT_INT8><<<R, kEvThreads, smem, st>>>(P, nt, first);
        } else {
            EQ_CUDA_TRY(cudaFuncSetAttribute(k_lb_eval<EQ_FMT_E4M3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            k_lb_eval<EQ_FMT_E4M3><<<R, kEvThreads, smem, st>>>(P, nt, first);
        }
        k_lb_update<<<n, kUpThreads, 0, st>>>(P, nt, first);
        EQ_CUDA_TRY(cudaGetLastError());
        return EQ_OK;
    };
    EQ_TRY(eval(1, 1));
    if (!iterate || p.max_iters == 0) return EQ_OK;
    const uint64_t max_passes =
        (uint64_t)p.max_iters * ((p.max_backtracks + p.trials - 1) / p.trials) + (uint64_t)p.max_iters + 1;
    uint32_t flags[EQ_MAX_LAYERS];
    for (uint64_t pass = 0; pass < max_passes; ++pass) {
        EQ_TRY(eval(p.trials, 0));
        if ((pass & 7) == 7 || pass + 1 == max_passes) {
            EQ_CUDA_TRY(cudaMemcpyAsync(flags, P.done_flags, 4 * n, cudaMemcpyDeviceToHost, st));
            EQ_CUDA_TRY(cudaStreamSynchronize(st));
            bool all = true;
            for (uint32_t i = 0; i < n; ++i) all = all && flags[i];
            if (all) break;
        }
    }
    return EQ_OK;
}

}  // namespace eq

using namespace eq;

extern "C" void eq_lbfgs_default_params(eq_lbfgs_params* p) {
    if (p) *p = lb_defaults();
}

extern "C" uint64_t eq_lbfgs_scratch_bytes(const eq_tensor* layers, uint32_t n_layers, const eq_lbfgs_params* p) {
    if (!layers || n_layers < 1 || n_layers > EQ_MAX_LAYERS) return 0;
    const eq_lbfgs_params q = p ? *p : lb_defaults();
    if (q.history < 1 || q.history > (uint32_t)kMaxHist || q.trials < 1 || q.trials > (uint32_t)kMaxTrials) return 0;
    return lb_layout(layers, n_layers, q.history, q.trials).total;
}

extern "C" eq_status eq_lbfgs_scales(const eq_tensor* layers, uint32_t n_layers, uint32_t format, double lambda,
                                     const eq_lbfgs_params* params, uint16_t* scales, double* trace, uint32_t* info,
                                     void* scratch, uint64_t scratch_bytes, eq_stream_t stream) {
    EQ_TRY(lb_check(layers, n_layers, format, lambda, params));
    if (!scales || !scratch) return EQ_ERR_ARG;
    const eq_lbfgs_params p = params ? *params : lb_defaults();
    const LbLayout L = lb_layout(layers, n_layers, p.history, p.trials);
    if (scratch_bytes < L.total) return EQ_ERR_BUFFER;
    cudaStream_t st = (cudaStream_t)stream;
    LbParams P;
    EQ_TRY(lb_run(layers, n_layers, format, lambda, p, nullptr, true, P, L, (char*)scratch, trace, st));
    k_lb_final<<<(P.R + 255) / 256, 256, 0, st>>>(P, scales, info);
    EQ_CUDA_TRY(cudaGetLastError());
    EQ_CUDA_TRY(cudaStreamSynchronize(st));
    return EQ_OK;
}

extern "C" eq_status eq_rd_eval(const eq_tensor* layer, uint32_t format, double lambda, const uint16_t* scales,
                                double* f_out, double* g_out, void* scratch, uint64_t scratch_bytes,
                                eq_stream_t stream) {
    EQ_TRY(lb_check(layer, 1, format, lambda, nullptr));
    if (!scales || !f_out || !g_out || !scratch) return EQ_ERR_ARG;
    eq_lbfgs_params p = lb_defaults();
    p.max_iters = 0;
    const LbLayout L = lb_layout(layer, 1, p.history, p.trials);
    if (scratch_bytes < L.total) return EQ_ERR_BUFFER;
    cudaStream_t st = (cudaStream_t)stream;
    LbParams P;
    EQ_TRY(lb_run(layer, 1, format, lambda, p, scales, false, P, L, (char*)scratch, f_out, st));
    EQ_CUDA_TRY(cudaMemcpyAsync(g_out, P.g, 8ull * P.R, cudaMemcpyDeviceToDevice, st));
    return EQ_OK;
}
