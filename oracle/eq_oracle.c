/*
 * eq_oracle.c — plain, slow, obviously-correct CPU ORACLE for the EntQuant hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2601_22787_b200/) never links, imports or calls it, and this file shares no
 * code, headers, tables or constants with the CUDA path.
 *
 * Paper: "Float8@2bits: Entropy Coding Enables Data-Free Model Compression"
 * (arXiv 2601.22787), cited as P:<line> of PAPER.md; SPEC.md lines as S:<line>;
 * readings of ambiguous passages follow SURVEY.md §8(c) and are listed in DESIGN.md §3.
 *
 * Arithmetic: fp64 throughout; integers are exact.  No blocking, fusion or
 * reordering beyond the definitions.  Every function names the passage it follows.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"): E4M3 grid vs the bit-layout closed form
 * and vs ml_dtypes/torch float8_e4m3fn; quantiser exhaustively vs ml_dtypes RNE of the
 * exact quotient; dequant vs ml_dtypes bf16 RNE of the exact f64 product; objective
 * special cases (λ=0, λ→∞, on-grid W) and brute-force scan on tiny tensors;
 * normalisation worked examples; rANS lossless round trip, Shannon
 * lower bound, cross-entropy upper bound, hand-derived stream (tests/golden/).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define EQO_PROB_BITS 12          /* M = 2^12                                 */
#define EQO_M        (1u << EQO_PROB_BITS)

/* ------------------------------------------------------------------------------------
 * §2.1 Float8-E4M3 grid, torch.float8_e4m3fn flavour:
 * sign | 4 exponent bits (bias 7) | 3 mantissa bits; e=0 subnormal m/8·2^-6;
 * normal (1+m/8)·2^(e-7); 0x7F / 0xFF are NaN (no infinities).
 * ---------------------------------------------------------------------------------- */
double eqo_e4m3_value(uint32_t code)
{
    code &= 0xFF;
    uint32_t sign = code >> 7, e = (code >> 3) & 0xF, m = code & 7;
    if ((code & 0x7F) == 0x7F) return NAN;
    double mag = (e == 0) ? ldexp((double)m / 8.0, -6) : ldexp(1.0 + (double)m / 8.0, (int)e - 7);
    return sign ? -mag : mag;
}

/* bf16 <-> f64.  bf16 = top 16 bits of an IEEE binary32; rounding f64 -> bf16 is
 * round-to-nearest-even on the exact value (scales are stored BF16). */
double eqo_bf16_to_double(uint16_t b)
{
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* Exact RNE of a double to bf16 by enumerating the two bf16 neighbours: plain and
 * slow on purpose.  IEEE overflow rule: beyond the last midpoint the result is inf. */
uint16_t eqo_bf16_from_double(double x)
{
    if (x != x) return 0x7FC0;
    uint16_t sign = (x < 0) ? 0x8000 : 0;
    double a = fabs(x);
    /* find largest non-negative bf16 pattern p with value(p) <= a by bisection over
     * the ordered positive patterns 0x0000..0x7F80 (values increase with the pattern). */
    uint32_t lo = 0, hi = 0x7F80; /* value(0x7F80) = +inf */
    if (a >= ldexp(1.0, 128)) return sign | 0x7F80;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) / 2;
        if (eqo_bf16_to_double((uint16_t)mid) <= a) lo = mid; else hi = mid;
    }
    double vlo = eqo_bf16_to_double((uint16_t)lo), vhi = eqo_bf16_to_double((uint16_t)hi);
    if (hi == 0x7F80) vhi = ldexp(1.0, 128);  /* IEEE overflow: the value 2^128 stands for inf */
    uint32_t p;
    if (a - vlo < vhi - a) p = lo;
    else if (a - vlo > vhi - a) p = hi;
    else p = (lo & 1) ? hi : lo;          /* tie -> even pattern */
    return (uint16_t)(sign | p);
}

/* ------------------------------------------------------------------------------------
 * §2.1 quantiser Q_γ: W_q = clamp(⌊W/s⌉, -Q_max, Q_max), ⌊·⌉ = nearest value
 * representable in γ = E4M3, Q_max = 448.
 * Readings: clamp before rounding; ties to the even code;
 * signed zero resolved to +0 (App. A.1).
 * The quotient is formed in f64.  For bf16 W and bf16 s an exact E4M3 midpoint quotient
 * is representable in f64 and the f64 division returns it exactly; any other quotient is
 * ≥ 2^-13 (relative) from every midpoint, far above f64 rounding, so the
 * nearest-value choice below equals the choice for the exact quotient.
 * Nearest value: textbook RNE to a 3-bit mantissa (cross-checked against a brute-force
 * scan of all 253 finite codes, eqo_quantize_value_scan, in the pins).
 * ---------------------------------------------------------------------------------- */
/* Code of a grid value (inverse of eqo_e4m3_value on the finite grid; -0 -> 0x00). */
static uint8_t eqo_e4m3_code(double v)
{
    uint8_t sign = (v < 0) ? 0x80 : 0;
    double a = fabs(v);
    if (a == 0.0) return 0x00;
    if (a < ldexp(1.0, -6))                       /* subnormal: m/8 * 2^-6 */
        return (uint8_t)(sign | (uint8_t)(a * 512.0));
    int k;
    double m = frexp(a, &k);                      /* a = m * 2^k, m in [0.5, 1) */
    int e = k - 1 + 7;                            /* a = (1+f) 2^(k-1)          */
    int mant = (int)((m * 2.0 - 1.0) * 8.0);
    return (uint8_t)(sign | (uint8_t)(e << 3) | (uint8_t)mant);
}

/* Nearest E4M3 value to r after clamping, the textbook way: 4 significant bits in the
 * normal range (|r| >= 2^-6), fixed spacing 2^-9 in the subnormal range; rint() is
 * round-half-even in the default rounding mode, so a tie goes to the even mantissa. */
uint8_t eqo_quantize_value(double r)
{
    if (r > 448.0) r = 448.0;
    if (r < -448.0) r = -448.0;
    double a = fabs(r), q;
    if (a < ldexp(1.0, -6)) {
        q = ldexp(rint(ldexp(a, 9)), -9);
    } else {
        int k;
        double m = frexp(a, &k);                  /* m in [0.5,1): 4 bits = m*16 */
        q = ldexp(rint(m * 16.0), k - 4);
    }
    if (q == 0.0) return 0x00;                    /* signed zero resolved */
    return eqo_e4m3_code(r < 0 ? -q : q);
}

/* Independent brute-force definition (pins only): scan all 253 finite codes for the
 * nearest value, ties to the even code. */
uint8_t eqo_quantize_value_scan(double r)
{
    if (r > 448.0) r = 448.0;
    if (r < -448.0) r = -448.0;
    int best = -1;
    double bestd = 0.0;
    for (int c = 0; c < 256; c++) {
        if ((c & 0x7F) == 0x7F || c == 0x80) continue;   /* NaN codes; -0 resolved */
        double d = fabs(r - eqo_e4m3_value((uint32_t)c));
        if (best < 0 || d < bestd || (d == bestd && (c & 1) == 0 && (best & 1) == 1)) {
            best = c;
            bestd = d;
        }
    }
    return (uint8_t)best;
}

uint8_t eqo_quantize_one(uint16_t w_bf16, uint16_t s_bf16)
{
    double w = eqo_bf16_to_double(w_bf16), s = eqo_bf16_to_double(s_bf16);
    return eqo_quantize_value(w / s);
}

/* ------------------------------------------------------------------------------------
 * Base formats γ (§2.1; P:392 Int8 vs Float8; SPEC quantgrid S:26-118):
 *   fmt 0 = Float8 E4M3 (above), Q_max 448;
 *   fmt 1 = symmetric Int8, codes −127..127 stored as the two's-complement byte, value =
 *           the integer ("value(c)=c"), Q_max 127; −128 (0x80) never produced.
 * Quantiser for Int8: clamp the quotient to ±127, then round half to even.
 * The f64 quotient is exact enough: for bf16 W and s a non-tie quotient is ≥ 2^-9
 * (relative) away from every half-integer.
 * ---------------------------------------------------------------------------------- */
double eqo_qmax(int fmt) { return fmt == 1 ? 127.0 : 448.0; }

double eqo_grid_value(int fmt, uint32_t code)
{
    if (fmt == 1) return (double)(int8_t)(uint8_t)code;
    return eqo_e4m3_value(code);
}

uint8_t eqo_grid_quantize(int fmt, double r)
{
    if (fmt != 1) return eqo_quantize_value(r);
    if (r > 127.0) r = 127.0;
    if (r < -127.0) r = -127.0;
    double q = rint(r);                           /* round half to even */
    if (q == 0.0) return 0x00;
    return (uint8_t)(int8_t)q;
}

/* Eq. (1), Alg. 1 l.1: s = max|W_row| / Q_max, per output channel
 * (P:148).  Stored as bf16 (RNE) since scales are BF16.  All-zero row -> 1. */
uint16_t eqo_absmax_scale_fmt(int fmt, const uint16_t* w_row, int64_t n)
{
    double m = 0.0;
    for (int64_t j = 0; j < n; j++) {
        double a = fabs(eqo_bf16_to_double(w_row[j]));
        if (a > m) m = a;
    }
    if (m == 0.0) return eqo_bf16_from_double(1.0);
    return eqo_bf16_from_double(m / eqo_qmax(fmt));
}

uint16_t eqo_absmax_scale(const uint16_t* w_row, int64_t n) { return eqo_absmax_scale_fmt(0, w_row, n); }

/* Alg. 1 l.3: W_q = Q_γ(W, S*) with one scale per row. */
void eqo_quantize_fmt(int fmt, const uint16_t* W, int64_t M, int64_t N, const uint16_t* S, uint8_t* codes)
{
    for (int64_t i = 0; i < M; i++) {
        double s = eqo_bf16_to_double(S[i]);
        for (int64_t j = 0; j < N; j++)
            codes[i * N + j] = eqo_grid_quantize(fmt, eqo_bf16_to_double(W[i * N + j]) / s);
    }
}

void eqo_quantize(const uint16_t* W, int64_t M, int64_t N, const uint16_t* S, uint8_t* codes)
{
    eqo_quantize_fmt(0, W, M, N, S, codes);
}

/* §2.1 dequantiser Q†: Ŵ = s·W_q, returned as bf16 (RNE of the exact f64
 * product; the product of a bf16 and an E4M3 value has ≤ 12 significant bits). */
void eqo_dequant_fmt(int fmt, const uint8_t* codes, int64_t M, int64_t N, const uint16_t* S, uint16_t* out)
{
    for (int64_t i = 0; i < M; i++) {
        double s = eqo_bf16_to_double(S[i]);
        for (int64_t j = 0; j < N; j++)
            out[i * N + j] = eqo_bf16_from_double(s * eqo_grid_value(fmt, codes[i * N + j]));
    }
}

void eqo_dequant(const uint8_t* codes, int64_t M, int64_t N, const uint16_t* S, uint16_t* out)
{
    eqo_dequant_fmt(0, codes, M, N, S, out);
}

/* ------------------------------------------------------------------------------------
 * Eq. (4): objective d(W,Ŵ) + λ R(W_q), d = ‖W-Ŵ‖₁/‖W‖₁, R = ‖W_q‖₁.
 * Reading: R in the code domain (grid values, pre-scale), normalised by
 * M·N.  The objective is separable over rows, so row i contributes
 *   f_i(s) = D_i(s)/‖W‖₁ + λ·R_i(s)/(M·N),
 *   D_i(s) = Σ_j |W_ij − s·v_ij|,  R_i(s) = Σ_j |v_ij|,  v_ij = value(Q_γ(W_ij, s)).
 * Each term is exact in f64; sums are sequential in j (f64).
 * ---------------------------------------------------------------------------------- */
void eqo_row_terms_fmt(int fmt, const uint16_t* w_row, int64_t n, uint16_t s_bf16, double* D, double* R)
{
    double s = eqo_bf16_to_double(s_bf16), d = 0.0, r = 0.0;
    for (int64_t j = 0; j < n; j++) {
        double w = eqo_bf16_to_double(w_row[j]);
        double v = eqo_grid_value(fmt, eqo_grid_quantize(fmt, w / s));
        d += fabs(w - s * v);
        r += fabs(v);
    }
    *D = d;
    *R = r;
}

void eqo_row_terms(const uint16_t* w_row, int64_t n, uint16_t s_bf16, double* D, double* R)
{
    eqo_row_terms_fmt(0, w_row, n, s_bf16, D, R);
}

/* ------------------------------------------------------------------------------------
 * Straight-through gradient of Eq. (4) w.r.t. a row's scale ("We use the
 * straight-through estimator for Q_γ"; SPEC ste_gradient S:231-239; reading R13).
 * Forward values are the true discrete ones (v = value(Q_γ(w/s))); for the derivative
 * Q_γ's rounding is the identity inside the clamp range |w/s| ≤ Q_max (inclusive, as
 * torch.clamp's backward) and its clamp has derivative 0 outside, so with q = w/s
 *   ∂(s·v)/∂s = v + s·∂v/∂s = v − q   (inside),   v   (clamped),
 *   ∂|w − s·v|/∂s = sign(s·v − w)·∂(s·v)/∂s,     ∂|v|/∂s = sign(v)·(−q/s)  (inside).
 * Inside the clamp sign(s·v − w) = sign(v − q) (s > 0), so that term is |v − q|; for v ≠ 0
 * sign(v) = sign(q), so the regulariser term is −|q|/s (torch: d|x|/dx = 0 at x = 0).
 * Returns the row sums  out = {D, R, A, B, Q}:
 *   D = Σ|w − s·v|,  R = Σ|v|,  A = Σ_inside |v − q|,  B = Σ_clamped sign(s·v − w)·v,
 *   Q = Σ_{inside, v≠0} |q|;
 * then ∂f_i/∂s = (A + B)/‖W‖₁ − λ·Q/(s·M·N).  All terms are exact or correctly rounded
 * f64 operations on exact inputs; sums are sequential in j. */
void eqo_rd_row_fmt(int fmt, const uint16_t* w_row, int64_t n, uint16_t s_bf16, double out[5])
{
    double s = eqo_bf16_to_double(s_bf16), qmax = eqo_qmax(fmt);
    double D = 0.0, R = 0.0, A = 0.0, B = 0.0, Q = 0.0;
    for (int64_t j = 0; j < n; j++) {
        double w = eqo_bf16_to_double(w_row[j]);
        double q = w / s;
        double v = eqo_grid_value(fmt, eqo_grid_quantize(fmt, q));
        double e = s * v - w;
        D += fabs(e);
        R += fabs(v);
        if (fabs(q) <= qmax) {
            A += fabs(v - q);
            if (v != 0.0) Q += fabs(q);
        } else {
            B += (e > 0.0 ? 1.0 : e < 0.0 ? -1.0 : 0.0) * v;
        }
    }
    out[0] = D;
    out[1] = R;
    out[2] = A;
    out[3] = B;
    out[4] = Q;
}

double eqo_l1(const uint16_t* W, int64_t n)
{
    double a = 0.0;
    for (int64_t j = 0; j < n; j++) a += fabs(eqo_bf16_to_double(W[j]));
    return a;
}

/* Full-matrix objective (Eq. 4) for given per-row scales. */
double eqo_objective_fmt(int fmt, const uint16_t* W, int64_t M, int64_t N, const uint16_t* S, double lambda)
{
    double l1 = eqo_l1(W, M * N), Dt = 0.0, Rt = 0.0;
    for (int64_t i = 0; i < M; i++) {
        double D, R;
        eqo_row_terms_fmt(fmt, W + i * N, N, S[i], &D, &R);
        Dt += D;
        Rt += R;
    }
    double d = (l1 > 0.0) ? Dt / l1 : 0.0;
    return d + lambda * Rt / ((double)M * (double)N);
}

double eqo_objective(const uint16_t* W, int64_t M, int64_t N, const uint16_t* S, double lambda)
{
    return eqo_objective_fmt(0, W, M, N, S, lambda);
}

/* Candidate set for row search (reading, DESIGN.md §3 / SURVEY §8c.5): the contiguous
 * positive bf16 patterns from bf16(s0·2^oct_lo) to bf16(s0·2^oct_hi) (positive bf16 values
 * are ordered by their bit patterns).  Returns the count, writes first pattern. */
int64_t eqo_candidates(uint16_t s0, int32_t oct_lo, int32_t oct_hi, uint16_t* first)
{
    double v0 = eqo_bf16_to_double(s0);
    uint16_t lo = eqo_bf16_from_double(ldexp(v0, oct_lo));
    uint16_t hi = eqo_bf16_from_double(ldexp(v0, oct_hi));
    if (lo < 0x0001) lo = 0x0001;
    if (hi > 0x7F7F) hi = 0x7F7F;
    if (hi < lo) hi = lo;
    *first = lo;
    return (int64_t)hi - (int64_t)lo + 1;
}

/* Alg. 1 l.1-2, solved per row by exhaustive minimisation over the
 * candidate set (reading replacing L-BFGS+STE).  Tie rule: the
 * smallest candidate attaining the minimum.  All-zero rows keep s = 1.
 * obj_rows (nullable) receives f_i(s*_i). */
void eqo_search_rows_fmt(int fmt, const uint16_t* W, int64_t M, int64_t N, double lambda,
                         int32_t oct_lo, int32_t oct_hi, int64_t row_begin, int64_t row_end,
                         uint16_t* S, double* obj_rows)
{
    double l1 = eqo_l1(W, M * N);
    double mn = (double)M * (double)N;
    for (int64_t i = row_begin; i < row_end; i++) {
        const uint16_t* row = W + i * N;
        uint16_t s0 = eqo_absmax_scale_fmt(fmt, row, N);
        int zero_row = 1;
        for (int64_t j = 0; j < N; j++)
            if ((row[j] & 0x7FFF) != 0) { zero_row = 0; break; }
        if (zero_row) {
            S[i] = s0;
            if (obj_rows) obj_rows[i] = 0.0;
            continue;
        }
        uint16_t first;
        int64_t nc = eqo_candidates(s0, oct_lo, oct_hi, &first);
        double best = INFINITY;
        uint16_t bests = first;
        for (int64_t k = 0; k < nc; k++) {
            uint16_t s = (uint16_t)(first + k);
            double D, R;
            eqo_row_terms_fmt(fmt, row, N, s, &D, &R);
            double f = (l1 > 0.0 ? D / l1 : 0.0) + lambda * R / mn;
            if (f < best) { best = f; bests = s; }
        }
        S[i] = bests;
        if (obj_rows) obj_rows[i] = best;
    }
}

void eqo_search_rows(const uint16_t* W, int64_t M, int64_t N, double lambda,
                     int32_t oct_lo, int32_t oct_hi, int64_t row_begin, int64_t row_end,
                     uint16_t* S, double* obj_rows)
{
    eqo_search_rows_fmt(0, W, M, N, lambda, oct_lo, oct_hi, row_begin, row_end, S, obj_rows);
}

/* Per-candidate objective table of one row (used by tests to check GPU choices
 * against every candidate).  f[k] for candidate first+k.  Returns the count. */
int64_t eqo_row_objectives_fmt(int fmt, const uint16_t* W, int64_t M, int64_t N, int64_t row, double lambda,
                               int32_t oct_lo, int32_t oct_hi, uint16_t* first_out, double* f,
                               int64_t cap)
{
    double l1 = eqo_l1(W, M * N);
    double mn = (double)M * (double)N;
    const uint16_t* r = W + row * N;
    uint16_t s0 = eqo_absmax_scale_fmt(fmt, r, N), first;
    int64_t nc = eqo_candidates(s0, oct_lo, oct_hi, &first);
    *first_out = first;
    for (int64_t k = 0; k < nc && k < cap; k++) {
        double D, R;
        eqo_row_terms_fmt(fmt, r, N, (uint16_t)(first + k), &D, &R);
        f[k] = (l1 > 0.0 ? D / l1 : 0.0) + lambda * R / mn;
    }
    return nc;
}

/* ------------------------------------------------------------------------------------
 * Metadata ℳ: symbol histogram of the block stream and the
 * frequency table normalised to 2^12.  Reading:
 * integer-only largest-remainder rule, because SPEC's literal rule can go negative.
 *   1. f_s = c_s>0 ? max(1, ⌊4096 c_s / T⌋) : 0 ;  r_s = (4096 c_s) mod T
 *   2. D = 4096 − Σ f
 *   3. D > 0: +1 to the D present symbols with largest r_s (ties: larger c_s, lower code)
 *   4. while D < 0: −1 from the current largest f_s with f_s > 1 (ties: lower code)
 * Returns 0, or -1 when T = 0 ("empty").
 * ---------------------------------------------------------------------------------- */
void eqo_histogram(const uint8_t* sym, int64_t n, uint64_t hist[256])
{
    for (int c = 0; c < 256; c++) hist[c] = 0;
    for (int64_t i = 0; i < n; i++) hist[sym[i]]++;
}

int eqo_normalize(const uint64_t hist[256], uint16_t freq[256])
{
    uint64_t T = 0;
    for (int c = 0; c < 256; c++) T += hist[c];
    if (T == 0) return -1;
    int64_t f[256], sum = 0;
    uint64_t r[256];
    for (int c = 0; c < 256; c++) {
        if (hist[c] == 0) { f[c] = 0; r[c] = 0; continue; }
        unsigned __int128 num = (unsigned __int128)EQO_M * hist[c];
        uint64_t q = (uint64_t)(num / T);
        r[c] = (uint64_t)(num % T);
        f[c] = q < 1 ? 1 : (int64_t)q;
        sum += f[c];
    }
    int64_t D = (int64_t)EQO_M - sum;
    if (D > 0) {
        /* pick D present symbols with largest (r, c, -code) by repeated selection */
        int taken[256] = {0};
        for (int64_t k = 0; k < D; k++) {
            int b = -1;
            for (int c = 0; c < 256; c++) {
                if (hist[c] == 0 || taken[c]) continue;
                if (b < 0 || r[c] > r[b] || (r[c] == r[b] && hist[c] > hist[b])) b = c;
            }
            taken[b] = 1;
            f[b] += 1;
        }
    }
    while (D < 0) {
        int b = -1;
        for (int c = 0; c < 256; c++)
            if (f[c] > 1 && (b < 0 || f[c] > f[b])) b = c;
        f[b] -= 1;
        D += 1;
    }
    for (int c = 0; c < 256; c++) freq[c] = (uint16_t)f[c];
    return 0;
}

/* Shannon empirical entropy Ĥ, Eq. (2), bits per symbol. */
double eqo_entropy(const uint64_t hist[256])
{
    uint64_t T = 0;
    for (int c = 0; c < 256; c++) T += hist[c];
    if (T == 0) return 0.0;
    double h = 0.0;
    for (int c = 0; c < 256; c++)
        if (hist[c]) {
            double p = (double)hist[c] / (double)T;
            h -= p * log2(p);
        }
    return h;
}

/* ------------------------------------------------------------------------------------
 * ANS (§2.1; Alg. 1 l.5 P:213; Alg. 2 l.1 P:229): rANS with a 32-bit state,
 * M = 2^12, cumulative frequencies in code order.  Two
 * renormalisation widths (the paper's coder, nvCOMP, does not document its own):
 *
 *   codec 0 (EQO_CODEC_BYTE, reading R9): L = 2^23, b = 2^8 — bytes;
 *   codec 1 (EQO_CODEC_WORD, reading R14):           L = 2^16, b = 2^16 — 16-bit words,
 *           each stored little-endian (low byte first).
 *
 * Encoder: reverse symbol order from x = L; before coding s, emit the low log2(b) bits
 * while x ≥ ((L>>12)·b)·f_s and shift them out; then x = ⌊x/f_s⌋·M + (x mod f_s) + c_s;
 * finally the 4-byte state, little-endian, precedes the renormalisation units in decode
 * order.  Decoder: x = LE32; per symbol slot = x mod M, s with c_s ≤ slot < c_s + f_s,
 * x = f_s·⌊x/M⌋ + slot − c_s, then while x < L: x = x·b + next unit.
 * ---------------------------------------------------------------------------------- */
#define EQO_CODEC_BYTE 0
#define EQO_CODEC_WORD 1

static void eqo_cum(const uint16_t freq[256], uint32_t cum[257])
{
    cum[0] = 0;
    for (int c = 0; c < 256; c++) cum[c + 1] = cum[c] + freq[c];
}

/* lower bound L and unit width (bits) of a codec; 0 width = unknown codec */
static void eqo_codec_params(int codec, uint64_t* L, int* unit_bits)
{
    if (codec == EQO_CODEC_BYTE) { *L = 1u << 23; *unit_bits = 8; }
    else if (codec == EQO_CODEC_WORD) { *L = 1u << 16; *unit_bits = 16; }
    else { *L = 0; *unit_bits = 0; }
}

/* Encodes n symbols; writes into out[0..cap).  Returns the byte count, -1 if cap is too
 * small, -2 if a symbol has zero frequency ("unknown-symbol"), -3 bad codec. */
int64_t eqo_encode_chunk_codec(int codec, const uint8_t* sym, int64_t n, const uint16_t freq[256],
                               uint8_t* out, int64_t cap)
{
    uint64_t L;
    int ub;
    eqo_codec_params(codec, &L, &ub);
    if (ub == 0) return -3;
    const int unit_bytes = ub / 8;
    uint32_t cum[257];
    eqo_cum(freq, cum);
    /* units are produced back-to-front into a temporary of worst-case size */
    int64_t tcap = 4 + 2 * n + 8;
    uint8_t* tmp = (uint8_t*)malloc((size_t)tcap);
    int64_t pos = tcap;
    uint64_t x = L;
    for (int64_t i = n - 1; i >= 0; i--) {
        uint32_t f = freq[sym[i]], c = cum[sym[i]];
        if (f == 0) { free(tmp); return -2; }
        uint64_t x_max = ((L >> EQO_PROB_BITS) << ub) * f;
        while (x >= x_max) {
            pos -= unit_bytes;
            for (int k = 0; k < unit_bytes; k++) tmp[pos + k] = (uint8_t)((x >> (8 * k)) & 0xFF);
            x >>= ub;
        }
        x = (x / f) * EQO_M + (x % f) + c;
    }
    pos -= 4;
    tmp[pos + 0] = (uint8_t)(x & 0xFF);
    tmp[pos + 1] = (uint8_t)((x >> 8) & 0xFF);
    tmp[pos + 2] = (uint8_t)((x >> 16) & 0xFF);
    tmp[pos + 3] = (uint8_t)((x >> 24) & 0xFF);
    int64_t len = tcap - pos;
    if (len > cap) { free(tmp); return -1; }
    memcpy(out, tmp + pos, (size_t)len);
    free(tmp);
    return len;
}

/* Decoder (Alg. 2 l.1): s found by a linear scan of the cumulative table.  Integrity
 * (SURVEY §5): at the end x must equal L and every byte must have been consumed.
 * Returns 0 ok, 1 corrupt, 2 truncated, 3 bad codec. */
int eqo_decode_chunk_codec(int codec, const uint8_t* in, int64_t nbytes, const uint16_t freq[256],
                           uint8_t* sym, int64_t n)
{
    uint64_t L;
    int ub;
    eqo_codec_params(codec, &L, &ub);
    if (ub == 0) return 3;
    const int unit_bytes = ub / 8;
    uint32_t cum[257];
    eqo_cum(freq, cum);
    if (nbytes < 4) return 2;
    uint64_t x = (uint64_t)in[0] | ((uint64_t)in[1] << 8) | ((uint64_t)in[2] << 16) |
                 ((uint64_t)in[3] << 24);
    int64_t p = 4;
    for (int64_t i = 0; i < n; i++) {
        uint32_t slot = (uint32_t)(x % EQO_M);
        int s = 0;
        while (!(cum[s] <= slot && slot < cum[s + 1])) s++;   /* cum[256] = M > slot */
        sym[i] = (uint8_t)s;
        x = (uint64_t)freq[s] * (x / EQO_M) + slot - cum[s];
        while (x < L) {
            if (p + unit_bytes > nbytes) return 2;
            uint64_t u = 0;
            for (int k = 0; k < unit_bytes; k++) u |= (uint64_t)in[p + k] << (8 * k);
            p += unit_bytes;
            x = (x << ub) | u;
        }
    }
    if (x != L || p != nbytes) return 1;
    return 0;
}

int64_t eqo_encode_chunk(const uint8_t* sym, int64_t n, const uint16_t freq[256], uint8_t* out, int64_t cap)
{
    return eqo_encode_chunk_codec(EQO_CODEC_BYTE, sym, n, freq, out, cap);
}

int eqo_decode_chunk(const uint8_t* in, int64_t nbytes, const uint16_t freq[256], uint8_t* sym, int64_t n)
{
    return eqo_decode_chunk_codec(EQO_CODEC_BYTE, in, nbytes, freq, sym, n);
}

/* ------------------------------------------------------------------------------------
 * Block stream (App. A.1): the vec'd code matrices of a block's
 * layers are concatenated in order; one table over the whole stream; the stream is
 * split into chunks of `cs` symbols that restart at each segment start:
 * `layer_sizes` lists the segments — one per layer (layer-restart chunking), or one per
 * row (EQ_CHUNK_ROW: a K-column row splits into ⌈K/cs⌉ chunks; the Python wrapper
 * expands the layers into rows);
 * payload = chunk streams back to back; chunk_off[k] = byte offset of chunk k,
 * chunk_off[n_chunks] = payload bytes.
 * ---------------------------------------------------------------------------------- */
int64_t eqo_block_chunks(const int64_t* layer_sizes, int32_t n_layers, int64_t cs)
{
    int64_t n = 0;
    for (int32_t l = 0; l < n_layers; l++) n += (layer_sizes[l] + cs - 1) / cs;
    return n;
}

/* Returns payload bytes, or a negative error. */
int64_t eqo_encode_block_codec(int codec, const uint8_t* codes, const int64_t* layer_sizes, int32_t n_layers,
                               int64_t cs, const uint16_t freq[256], uint8_t* payload, int64_t cap,
                               uint32_t* chunk_off)
{
    int64_t pos = 0, k = 0, sbase = 0;
    for (int32_t l = 0; l < n_layers; l++) {
        for (int64_t a = 0; a < layer_sizes[l]; a += cs) {
            int64_t n = layer_sizes[l] - a < cs ? layer_sizes[l] - a : cs;
            chunk_off[k++] = (uint32_t)pos;
            int64_t len = eqo_encode_chunk_codec(codec, codes + sbase + a, n, freq, payload + pos, cap - pos);
            if (len < 0) return len;
            pos += len;
        }
        sbase += layer_sizes[l];
    }
    chunk_off[k] = (uint32_t)pos;
    return pos;
}

int64_t eqo_encode_block(const uint8_t* codes, const int64_t* layer_sizes, int32_t n_layers,
                         int64_t cs, const uint16_t freq[256], uint8_t* payload, int64_t cap,
                         uint32_t* chunk_off)
{
    return eqo_encode_block_codec(EQO_CODEC_BYTE, codes, layer_sizes, n_layers, cs, freq, payload, cap, chunk_off);
}

/* Decodes a whole block stream into codes; returns 0 / first failing status. */
int eqo_decode_block_codec(int codec, const uint8_t* payload, const uint32_t* chunk_off, const int64_t* layer_sizes,
                           int32_t n_layers, int64_t cs, const uint16_t freq[256], uint8_t* codes)
{
    int64_t k = 0, sbase = 0;
    for (int32_t l = 0; l < n_layers; l++) {
        for (int64_t a = 0; a < layer_sizes[l]; a += cs) {
            int64_t n = layer_sizes[l] - a < cs ? layer_sizes[l] - a : cs;
            int st = eqo_decode_chunk_codec(codec, payload + chunk_off[k],
                                            (int64_t)chunk_off[k + 1] - chunk_off[k], freq, codes + sbase + a, n);
            if (st) return st;
            k++;
        }
        sbase += layer_sizes[l];
    }
    return 0;
}

int eqo_decode_block(const uint8_t* payload, const uint32_t* chunk_off, const int64_t* layer_sizes,
                     int32_t n_layers, int64_t cs, const uint16_t freq[256], uint8_t* codes)
{
    return eqo_decode_block_codec(EQO_CODEC_BYTE, payload, chunk_off, layer_sizes, n_layers, cs, freq, codes);
}

/* ------------------------------------------------------------------------------------
 * CPU baseline timing helper (bench.py cpu_baseline only): the same decoder as above,
 * chunks statically partitioned over `threads` POSIX threads.  No change to the
 * arithmetic; it only runs eqo_decode_chunk on disjoint chunks concurrently.
 * ---------------------------------------------------------------------------------- */
typedef struct {
    const uint8_t* payload; const uint32_t* chunk_off; const uint64_t* chunk_sym0;
    const uint32_t* chunk_n; const uint16_t* freq; uint8_t* codes;
    int64_t k0, k1; int status; int codec;
} eqo_job;

static void* eqo_worker(void* p)
{
    eqo_job* j = (eqo_job*)p;
    j->status = 0;
    for (int64_t k = j->k0; k < j->k1; k++) {
        int st = eqo_decode_chunk_codec(j->codec, j->payload + j->chunk_off[k],
                                        (int64_t)j->chunk_off[k + 1] - j->chunk_off[k], j->freq,
                                        j->codes + j->chunk_sym0[k], j->chunk_n[k]);
        if (st && !j->status) j->status = st;
    }
    return NULL;
}

int eqo_decode_chunks_mt_codec(int codec, const uint8_t* payload, const uint32_t* chunk_off,
                               const uint64_t* chunk_sym0, const uint32_t* chunk_n, int64_t n_chunks,
                               const uint16_t freq[256], uint8_t* codes, int threads)
{
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    eqo_job* jobs = (eqo_job*)malloc(sizeof(eqo_job) * (size_t)threads);
    for (int t = 0; t < threads; t++) {
        jobs[t] = (eqo_job){payload, chunk_off, chunk_sym0, chunk_n, freq, codes,
                            n_chunks * t / threads, n_chunks * (t + 1) / threads, 0, codec};
        pthread_create(&th[t], NULL, eqo_worker, &jobs[t]);
    }
    int st = 0;
    for (int t = 0; t < threads; t++) {
        pthread_join(th[t], NULL);
        if (jobs[t].status && !st) st = jobs[t].status;
    }
    free(th);
    free(jobs);
    return st;
}

/* CPU baseline (bench.py only): Alg. 2 l.1-2 for the chunks of ONE layer — each chunk is
 * decoded with eqo_decode_chunk and every symbol dequantised exactly as eqo_dequant does
 * (bf16 RNE of s_row·value(code)); chunks statically partitioned over POSIX threads. */
typedef struct {
    const uint8_t* payload; const uint32_t* chunk_off; int64_t cs, size, cols;
    const uint16_t* scales; const uint16_t* freq; uint16_t* out; int64_t k0, k1; int status; int codec; int64_t seg;
} eqo_ljob;

/* Chunk k of a layer whose chunking restarts every `seg` symbols (seg = the layer size:
 * layer-restart chunking; seg = cols: EQ_CHUNK_ROW, boundaries also at every
 * row start): its first symbol, and its length in *n. */
static int64_t eqo_chunk_start(int64_t k, int64_t cs, int64_t seg, int64_t* n)
{
    int64_t cps = (seg + cs - 1) / cs;          /* chunks per segment */
    int64_t s = k / cps, j = k % cps;
    *n = seg - j * cs < cs ? seg - j * cs : cs;
    return s * seg + j * cs;
}

static void* eqo_lworker(void* p)
{
    eqo_ljob* j = (eqo_ljob*)p;
    uint8_t* sym = (uint8_t*)malloc((size_t)j->cs);
    j->status = 0;
    for (int64_t k = j->k0; k < j->k1; k++) {
        int64_t n, a = eqo_chunk_start(k, j->cs, j->seg, &n);
        int st = eqo_decode_chunk_codec(j->codec, j->payload + j->chunk_off[k],
                                        (int64_t)j->chunk_off[k + 1] - j->chunk_off[k], j->freq, sym, n);
        if (st && !j->status) j->status = st;
        for (int64_t i = 0; i < n; i++) {
            int64_t row = (a + i) / j->cols;
            j->out[a + i] = eqo_bf16_from_double(eqo_bf16_to_double(j->scales[row]) * eqo_e4m3_value(sym[i]));
        }
    }
    free(sym);
    return NULL;
}

int eqo_decode_dequant_layer_mt_codec_seg(int codec, const uint8_t* payload, const uint32_t* chunk_off,
                                          int64_t n_chunks, int64_t cs, int64_t size, int64_t cols, int64_t seg,
                                          const uint16_t* scales, const uint16_t freq[256], uint16_t* out, int threads)
{
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    eqo_ljob* jobs = (eqo_ljob*)malloc(sizeof(eqo_ljob) * (size_t)threads);
    for (int t = 0; t < threads; t++) {
        jobs[t] = (eqo_ljob){payload, chunk_off, cs, size, cols, scales, freq, out,
                             n_chunks * t / threads, n_chunks * (t + 1) / threads, 0, codec, seg};
        pthread_create(&th[t], NULL, eqo_lworker, &jobs[t]);
    }
    int st = 0;
    for (int t = 0; t < threads; t++) {
        pthread_join(th[t], NULL);
        if (jobs[t].status && !st) st = jobs[t].status;
    }
    free(th);
    free(jobs);
    return st;
}

int eqo_decode_dequant_layer_mt_codec(int codec, const uint8_t* payload, const uint32_t* chunk_off, int64_t n_chunks,
                                      int64_t cs, int64_t size, int64_t cols, const uint16_t* scales,
                                      const uint16_t freq[256], uint16_t* out, int threads)
{
    return eqo_decode_dequant_layer_mt_codec_seg(codec, payload, chunk_off, n_chunks, cs, size, cols, size, scales,
                                                 freq, out, threads);
}

int64_t eqo_row_objectives(const uint16_t* W, int64_t M, int64_t N, int64_t row, double lambda,
                           int32_t oct_lo, int32_t oct_hi, uint16_t* first_out, double* f, int64_t cap)
{
    return eqo_row_objectives_fmt(0, W, M, N, row, lambda, oct_lo, oct_hi, first_out, f, cap);
}

int eqo_decode_chunks_mt(const uint8_t* payload, const uint32_t* chunk_off, const uint64_t* chunk_sym0,
                         const uint32_t* chunk_n, int64_t n_chunks, const uint16_t freq[256], uint8_t* codes,
                         int threads)
{
    return eqo_decode_chunks_mt_codec(EQO_CODEC_BYTE, payload, chunk_off, chunk_sym0, chunk_n, n_chunks, freq,
                                      codes, threads);
}

int eqo_decode_dequant_layer_mt(const uint8_t* payload, const uint32_t* chunk_off, int64_t n_chunks, int64_t cs,
                                int64_t size, int64_t cols, const uint16_t* scales, const uint16_t freq[256],
                                uint16_t* out, int threads)
{
    return eqo_decode_dequant_layer_mt_codec(EQO_CODEC_BYTE, payload, chunk_off, n_chunks, cs, size, cols, scales,
                                             freq, out, threads);
}

/* ------------------------------------------------------------------------------------
 * Pair codec (codec 2, EQO_CODEC_PAIR; reading R15): the word codec's rANS
 * (L = 2^16, 16-bit words, M = 2^12) over PAIRS of consecutive symbols of a chunk, for
 * the block's most frequent symbols, with an escape to single symbols.  The paper fixes no
 * wire format (nvCOMP's is undocumented); the symbols are modelled i.i.d. (the
 * factorisation of P:160-168), so a pair's probability is the product of its symbols'.
 *
 * Tables (from the block histogram, integers only):
 *  - ranks: present codes by count descending, ties by lower code; the first
 *    K = min(15, #present) get ranks 0..K-1 (rank_code[r] = code);
 *  - pair weights w(ra, rb) = c[code_ra]·c[code_rb] over the ranked codes (T = Σc, total T²);
 *    a pair is KEPT when its ideal frequency is at least 1/32 slot, 32·M·w ≥ T² (it then
 *    gets ≥ 1 slot: about as cheap as an escape followed by two singles, and escapes — the
 *    decoder's divergent path — become 5× rarer);
 *  - escape weight = T² − Σ kept w (all other pairs); the vector [kept pairs in (ra, rb)
 *    lexicographic order, escape] is normalised to M by the R8 rule (eqo_normalize's rule on
 *    128-bit numerators; escape present iff its weight is > 0); cum in that order, so the
 *    escape owns the top slots;
 *  - the single-symbol table is the R8 table of the histogram (eqo_normalize).
 * Chunk of n symbols: pairs (s[2i], s[2i+1]), i < ⌊n/2⌋, in order, then s[n−1] with the
 * single table if n is odd.  A pair whose two codes are ranked and whose (ra, rb) is kept is
 * one pair-table symbol; otherwise the escape (pair table) followed by the two codes
 * (single table).  The encoder works in reverse (for an escaped pair: b, a, then escape).
 * ---------------------------------------------------------------------------------- */
#define EQO_CODEC_PAIR 2
#define EQO_PAIR_K 15

/* R8 normalisation of n weights (total W) to M; pres[i] = weight > 0. */
static void eqo_normalize_w(const unsigned __int128* w, int n, unsigned __int128 W, int64_t* f)
{
    unsigned __int128 r[EQO_PAIR_K * EQO_PAIR_K + 1];
    int64_t sum = 0;
    for (int i = 0; i < n; i++) {
        if (w[i] == 0) { f[i] = 0; r[i] = 0; continue; }
        unsigned __int128 num = (unsigned __int128)EQO_M * w[i];
        unsigned __int128 q = num / W;
        r[i] = num % W;
        f[i] = q < 1 ? 1 : (int64_t)q;
        sum += f[i];
    }
    int64_t D = (int64_t)EQO_M - sum;
    if (D > 0) {
        int taken[EQO_PAIR_K * EQO_PAIR_K + 1] = {0};
        for (int64_t k = 0; k < D; k++) {
            int b = -1;
            for (int i = 0; i < n; i++) {
                if (w[i] == 0 || taken[i]) continue;
                if (b < 0 || r[i] > r[b] || (r[i] == r[b] && w[i] > w[b])) b = i;
            }
            taken[b] = 1;
            f[b] += 1;
        }
    }
    while (D < 0) {
        int b = -1;
        for (int i = 0; i < n; i++)
            if (f[i] > 1 && (b < 0 || f[i] > f[b])) b = i;
        f[b] -= 1;
        D += 1;
    }
}

/* Builds the pair tables.  rank_code[16] (unused ranks 0), *K, pf[15*15] = pair frequency
 * by (ra, rb) (0 = not kept), *fesc = escape frequency.  Returns 0, or -1 for an empty
 * histogram. */
int eqo_pair_table(const uint64_t hist[256], uint8_t rank_code[16], int32_t* K_out, uint16_t pf[225],
                   uint16_t* fesc)
{
    uint64_t T = 0;
    for (int c = 0; c < 256; c++) T += hist[c];
    if (T == 0) return -1;
    /* ranks: repeated selection of the largest count, lower code first on ties */
    int used[256] = {0}, K = 0;
    memset(rank_code, 0, 16);
    for (; K < EQO_PAIR_K; K++) {
        int b = -1;
        for (int c = 0; c < 256; c++)
            if (hist[c] && !used[c] && (b < 0 || hist[c] > hist[b])) b = c;
        if (b < 0) break;
        used[b] = 1;
        rank_code[K] = (uint8_t)b;
    }
    const unsigned __int128 W = (unsigned __int128)T * T;
    unsigned __int128 w[EQO_PAIR_K * EQO_PAIR_K + 1];
    int idx[EQO_PAIR_K * EQO_PAIR_K];
    int n = 0;
    unsigned __int128 kept = 0;
    for (int ra = 0; ra < K; ra++)
        for (int rb = 0; rb < K; rb++) {
            unsigned __int128 x = (unsigned __int128)hist[rank_code[ra]] * hist[rank_code[rb]];
            if ((unsigned __int128)32 * EQO_M * x >= W) {     /* ideal frequency ≥ 1/32 slot */
                w[n] = x;
                idx[n] = ra * EQO_PAIR_K + rb;
                kept += x;
                n++;
            }
        }
    w[n] = W - kept;                 /* escape: every other pair */
    int64_t f[EQO_PAIR_K * EQO_PAIR_K + 1];
    eqo_normalize_w(w, n + 1, W, f);
    for (int i = 0; i < 225; i++) pf[i] = 0;
    for (int i = 0; i < n; i++) pf[idx[i]] = (uint16_t)f[i];
    *fesc = (uint16_t)f[n];
    *K_out = K;
    return 0;
}

/* cumulative pair table in cum order: kept pairs lexicographic by (ra, rb), escape last */
static void eqo_pair_cum(const uint16_t pf[225], int K, uint32_t pcum[225], uint32_t* cesc)
{
    uint32_t run = 0;
    for (int ra = 0; ra < EQO_PAIR_K; ra++)
        for (int rb = 0; rb < EQO_PAIR_K; rb++) {
            int i = ra * EQO_PAIR_K + rb;
            pcum[i] = run;
            if (ra < K && rb < K) run += pf[i];
        }
    *cesc = run;
}

/* one rANS encode step with the word codec's renormalisation (units emitted back to front) */
static void eqo_w_put(uint64_t* x, uint32_t f, uint32_t c, uint8_t* tmp, int64_t* pos)
{
    const uint64_t L = 1u << 16;
    uint64_t x_max = ((L >> EQO_PROB_BITS) << 16) * f;
    while (*x >= x_max) {
        *pos -= 2;
        tmp[*pos] = (uint8_t)(*x & 0xFF);
        tmp[*pos + 1] = (uint8_t)((*x >> 8) & 0xFF);
        *x >>= 16;
    }
    *x = (*x / f) * EQO_M + (*x % f) + c;
}

int64_t eqo_encode_chunk_pair(const uint8_t* sym, int64_t n, const uint16_t freq[256], const uint8_t rank_code[16],
                              int32_t K, const uint16_t pf[225], uint16_t fesc, uint8_t* out, int64_t cap)
{
    uint32_t cum[257], pcum[225], cesc;
    eqo_cum(freq, cum);
    eqo_pair_cum(pf, K, pcum, &cesc);
    int rank[256];
    for (int c = 0; c < 256; c++) rank[c] = -1;
    for (int r = 0; r < K; r++) rank[rank_code[r]] = r;
    int64_t tcap = 4 + 4 * n + 8;
    uint8_t* tmp = (uint8_t*)malloc((size_t)tcap);
    int64_t pos = tcap;
    uint64_t x = 1u << 16;
    if (n & 1) {
        uint8_t s = sym[n - 1];
        if (freq[s] == 0) { free(tmp); return -2; }
        eqo_w_put(&x, freq[s], cum[s], tmp, &pos);
    }
    for (int64_t i = n / 2 - 1; i >= 0; i--) {
        uint8_t a = sym[2 * i], b = sym[2 * i + 1];
        if (freq[a] == 0 || freq[b] == 0) { free(tmp); return -2; }
        int ra = rank[a], rb = rank[b];
        if (ra >= 0 && rb >= 0 && pf[ra * EQO_PAIR_K + rb] > 0) {
            eqo_w_put(&x, pf[ra * EQO_PAIR_K + rb], pcum[ra * EQO_PAIR_K + rb], tmp, &pos);
        } else {
            if (fesc == 0) { free(tmp); return -2; }
            eqo_w_put(&x, freq[b], cum[b], tmp, &pos);
            eqo_w_put(&x, freq[a], cum[a], tmp, &pos);
            eqo_w_put(&x, fesc, cesc, tmp, &pos);
        }
    }
    pos -= 4;
    for (int k = 0; k < 4; k++) tmp[pos + k] = (uint8_t)((x >> (8 * k)) & 0xFF);
    int64_t len = tcap - pos;
    if (len > cap) { free(tmp); return -1; }
    memcpy(out, tmp + pos, (size_t)len);
    free(tmp);
    return len;
}

/* one rANS decode step: slot, then the caller's symbol lookup, state update, renormalise */
static int eqo_w_get(uint64_t* x, uint32_t f, uint32_t c, uint32_t slot, const uint8_t* in, int64_t nbytes,
                     int64_t* p)
{
    *x = (uint64_t)f * (*x / EQO_M) + slot - c;
    while (*x < (1u << 16)) {
        if (*p + 2 > nbytes) return 2;
        *x = (*x << 16) | (uint64_t)in[*p] | ((uint64_t)in[*p + 1] << 8);
        *p += 2;
    }
    return 0;
}

int eqo_decode_chunk_pair(const uint8_t* in, int64_t nbytes, const uint16_t freq[256], const uint8_t rank_code[16],
                          int32_t K, const uint16_t pf[225], uint16_t fesc, uint8_t* sym, int64_t n)
{
    uint32_t cum[257], pcum[225], cesc;
    eqo_cum(freq, cum);
    eqo_pair_cum(pf, K, pcum, &cesc);
    if (nbytes < 4) return 2;
    uint64_t x = (uint64_t)in[0] | ((uint64_t)in[1] << 8) | ((uint64_t)in[2] << 16) | ((uint64_t)in[3] << 24);
    int64_t p = 4;
    for (int64_t i = 0; i < n / 2; i++) {
        uint32_t slot = (uint32_t)(x % EQO_M);
        if (slot >= cesc) {                                   /* escape, then two singles */
            if (eqo_w_get(&x, fesc, cesc, slot, in, nbytes, &p)) return 2;
            for (int k = 0; k < 2; k++) {
                uint32_t sl = (uint32_t)(x % EQO_M);
                int s = 0;
                while (!(cum[s] <= sl && sl < cum[s + 1])) s++;
                sym[2 * i + k] = (uint8_t)s;
                if (eqo_w_get(&x, freq[s], cum[s], sl, in, nbytes, &p)) return 2;
            }
        } else {
            int j = -1;                                      /* the kept pair owning slot */
            for (int q = 0; q < 225 && j < 0; q++) {
                int ra = q / EQO_PAIR_K, rb = q % EQO_PAIR_K;
                if (ra < K && rb < K && pf[q] && pcum[q] <= slot && slot < pcum[q] + pf[q]) j = q;
            }
            if (j < 0) return 1;
            sym[2 * i] = rank_code[j / EQO_PAIR_K];
            sym[2 * i + 1] = rank_code[j % EQO_PAIR_K];
            if (eqo_w_get(&x, pf[j], pcum[j], slot, in, nbytes, &p)) return 2;
        }
    }
    if (n & 1) {
        uint32_t sl = (uint32_t)(x % EQO_M);
        int s = 0;
        while (!(cum[s] <= sl && sl < cum[s + 1])) s++;
        sym[n - 1] = (uint8_t)s;
        if (eqo_w_get(&x, freq[s], cum[s], sl, in, nbytes, &p)) return 2;
    }
    if (x != (1u << 16) || p != nbytes) return 1;
    return 0;
}

/* ------------------------------------------------------------------------------------
 * Pair codec with grouped escapes (codec 3, EQO_CODEC_PAIRG; reading R18).  The
 * same tables and the same coded symbols as codec 2 (R15) — only their ORDER in the rANS
 * stream differs, so the coded size is the same up to the state's end effects.  The chunk's
 * n symbols are cut into groups of 16 (the last one may be shorter, length g).  In decode
 * order, a group is:
 *   (1) its ⌊g/2⌋ pair positions in order, each a kept pair or the escape (pair table);
 *   (2) for every escaped position, in increasing order, its two codes a then b (single table);
 *   (3) if g is odd (the chunk's last group only), its last symbol (single table).
 * The encoder writes the group sequence (1)(2)(3) of every group, first group first, into a
 * list of (frequency, cumulative) steps and codes the list in reverse.
 * ---------------------------------------------------------------------------------- */
#define EQO_CODEC_PAIRG 3
#define EQO_GROUP 16

int64_t eqo_encode_chunk_pairg(const uint8_t* sym, int64_t n, const uint16_t freq[256], const uint8_t rank_code[16],
                               int32_t K, const uint16_t pf[225], uint16_t fesc, uint8_t* out, int64_t cap)
{
    uint32_t cum[257], pcum[225], cesc;
    eqo_cum(freq, cum);
    eqo_pair_cum(pf, K, pcum, &cesc);
    int rank[256];
    for (int c = 0; c < 256; c++) rank[c] = -1;
    for (int r = 0; r < K; r++) rank[rank_code[r]] = r;
    /* the decode-order list of steps: at most 3 per pair position + 1 */
    uint32_t* sf = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(3 * n / 2 + 2));
    uint32_t* sc = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(3 * n / 2 + 2));
    int64_t m = 0;
    for (int64_t g0 = 0; g0 < n; g0 += EQO_GROUP) {
        int64_t g = n - g0 < EQO_GROUP ? n - g0 : EQO_GROUP;
        int esc[EQO_GROUP / 2];
        for (int64_t i = 0; i < g / 2; i++) {                         /* (1) */
            uint8_t a = sym[g0 + 2 * i], b = sym[g0 + 2 * i + 1];
            if (freq[a] == 0 || freq[b] == 0) { free(sf); free(sc); return -2; }
            int ra = rank[a], rb = rank[b];
            esc[i] = !(ra >= 0 && rb >= 0 && pf[ra * EQO_PAIR_K + rb] > 0);
            if (esc[i]) {
                if (fesc == 0) { free(sf); free(sc); return -2; }
                sf[m] = fesc; sc[m] = cesc; m++;
            } else {
                sf[m] = pf[ra * EQO_PAIR_K + rb]; sc[m] = pcum[ra * EQO_PAIR_K + rb]; m++;
            }
        }
        for (int64_t i = 0; i < g / 2; i++) {                         /* (2) */
            if (!esc[i]) continue;
            uint8_t a = sym[g0 + 2 * i], b = sym[g0 + 2 * i + 1];
            sf[m] = freq[a]; sc[m] = cum[a]; m++;
            sf[m] = freq[b]; sc[m] = cum[b]; m++;
        }
        if (g & 1) {                                                  /* (3) */
            uint8_t s = sym[g0 + g - 1];
            if (freq[s] == 0) { free(sf); free(sc); return -2; }
            sf[m] = freq[s]; sc[m] = cum[s]; m++;
        }
    }
    int64_t tcap = 4 + 4 * n + 8;
    uint8_t* tmp = (uint8_t*)malloc((size_t)tcap);
    int64_t pos = tcap;
    uint64_t x = 1u << 16;
    for (int64_t k = m - 1; k >= 0; k--) eqo_w_put(&x, sf[k], sc[k], tmp, &pos);
    free(sf);
    free(sc);
    pos -= 4;
    for (int k = 0; k < 4; k++) tmp[pos + k] = (uint8_t)((x >> (8 * k)) & 0xFF);
    int64_t len = tcap - pos;
    if (len > cap) { free(tmp); return -1; }
    memcpy(out, tmp + pos, (size_t)len);
    free(tmp);
    return len;
}

/* the single-table symbol owning slot sl, then its decode step */
static int eqo_w_single(uint64_t* x, const uint16_t freq[256], const uint32_t cum[257], const uint8_t* in,
                        int64_t nbytes, int64_t* p, uint8_t* s_out)
{
    uint32_t sl = (uint32_t)(*x % EQO_M);
    int s = 0;
    while (!(cum[s] <= sl && sl < cum[s + 1])) s++;
    *s_out = (uint8_t)s;
    return eqo_w_get(x, freq[s], cum[s], sl, in, nbytes, p);
}

int eqo_decode_chunk_pairg(const uint8_t* in, int64_t nbytes, const uint16_t freq[256], const uint8_t rank_code[16],
                           int32_t K, const uint16_t pf[225], uint16_t fesc, uint8_t* sym, int64_t n)
{
    uint32_t cum[257], pcum[225], cesc;
    eqo_cum(freq, cum);
    eqo_pair_cum(pf, K, pcum, &cesc);
    if (nbytes < 4) return 2;
    uint64_t x = (uint64_t)in[0] | ((uint64_t)in[1] << 8) | ((uint64_t)in[2] << 16) | ((uint64_t)in[3] << 24);
    int64_t p = 4;
    for (int64_t g0 = 0; g0 < n; g0 += EQO_GROUP) {
        int64_t g = n - g0 < EQO_GROUP ? n - g0 : EQO_GROUP;
        int esc[EQO_GROUP / 2];
        for (int64_t i = 0; i < g / 2; i++) {                         /* (1) */
            uint32_t slot = (uint32_t)(x % EQO_M);
            esc[i] = slot >= cesc;
            if (esc[i]) {
                if (eqo_w_get(&x, fesc, cesc, slot, in, nbytes, &p)) return 2;
                continue;
            }
            int j = -1;                                              /* the kept pair owning slot */
            for (int q = 0; q < 225 && j < 0; q++) {
                int ra = q / EQO_PAIR_K, rb = q % EQO_PAIR_K;
                if (ra < K && rb < K && pf[q] && pcum[q] <= slot && slot < pcum[q] + pf[q]) j = q;
            }
            if (j < 0) return 1;
            sym[g0 + 2 * i] = rank_code[j / EQO_PAIR_K];
            sym[g0 + 2 * i + 1] = rank_code[j % EQO_PAIR_K];
            if (eqo_w_get(&x, pf[j], pcum[j], slot, in, nbytes, &p)) return 2;
        }
        for (int64_t i = 0; i < g / 2; i++) {                         /* (2) */
            if (!esc[i]) continue;
            if (eqo_w_single(&x, freq, cum, in, nbytes, &p, &sym[g0 + 2 * i])) return 2;
            if (eqo_w_single(&x, freq, cum, in, nbytes, &p, &sym[g0 + 2 * i + 1])) return 2;
        }
        if (g & 1)                                                    /* (3) */
            if (eqo_w_single(&x, freq, cum, in, nbytes, &p, &sym[g0 + g - 1])) return 2;
    }
    if (x != (1u << 16) || p != nbytes) return 1;
    return 0;
}

typedef int64_t (*eqo_penc_fn)(const uint8_t*, int64_t, const uint16_t*, const uint8_t*, int32_t, const uint16_t*,
                               uint16_t, uint8_t*, int64_t);
typedef int (*eqo_pdec_fn)(const uint8_t*, int64_t, const uint16_t*, const uint8_t*, int32_t, const uint16_t*,
                           uint16_t, uint8_t*, int64_t);
/* the chunk coder of a pair codec: grouped = 0 -> R15 (codec 2), 1 -> R18 (codec 3) */
static eqo_penc_fn eqo_penc(int32_t grouped) { return grouped ? eqo_encode_chunk_pairg : eqo_encode_chunk_pair; }
static eqo_pdec_fn eqo_pdec(int32_t grouped) { return grouped ? eqo_decode_chunk_pairg : eqo_decode_chunk_pair; }

/* block stream of the pair codec (same chunking as eqo_encode_block) */
int64_t eqo_encode_block_pairx(const uint8_t* codes, const int64_t* layer_sizes, int32_t n_layers, int64_t cs,
                               const uint16_t freq[256], const uint8_t rank_code[16], int32_t K, const uint16_t pf[225],
                               uint16_t fesc, uint8_t* payload, int64_t cap, uint32_t* chunk_off, int32_t grouped)
{
    int64_t pos = 0, k = 0, sbase = 0;
    for (int32_t l = 0; l < n_layers; l++) {
        for (int64_t a = 0; a < layer_sizes[l]; a += cs) {
            int64_t n = layer_sizes[l] - a < cs ? layer_sizes[l] - a : cs;
            chunk_off[k++] = (uint32_t)pos;
            int64_t len = eqo_penc(grouped)(codes + sbase + a, n, freq, rank_code, K, pf, fesc, payload + pos,
                                            cap - pos);
            if (len < 0) return len;
            pos += len;
        }
        sbase += layer_sizes[l];
    }
    chunk_off[k] = (uint32_t)pos;
    return pos;
}

int eqo_decode_block_pairx(const uint8_t* payload, const uint32_t* chunk_off, const int64_t* layer_sizes,
                           int32_t n_layers, int64_t cs, const uint16_t freq[256], const uint8_t rank_code[16], int32_t K,
                           const uint16_t pf[225], uint16_t fesc, uint8_t* codes, int32_t grouped)
{
    int64_t k = 0, sbase = 0;
    for (int32_t l = 0; l < n_layers; l++) {
        for (int64_t a = 0; a < layer_sizes[l]; a += cs) {
            int64_t n = layer_sizes[l] - a < cs ? layer_sizes[l] - a : cs;
            int st = eqo_pdec(grouped)(payload + chunk_off[k], (int64_t)chunk_off[k + 1] - chunk_off[k], freq,
                                       rank_code, K, pf, fesc, codes + sbase + a, n);
            if (st) return st;
            k++;
        }
        sbase += layer_sizes[l];
    }
    return 0;
}

/* CPU baseline (bench.py only) for the pair codec: as eqo_decode_dequant_layer_mt, with
 * eqo_decode_chunk_pair per chunk. */
typedef struct {
    const uint8_t* payload; const uint32_t* chunk_off; int64_t cs, size, cols;
    const uint16_t* scales; const uint16_t* freq; const uint8_t* rank_code; int32_t K; const uint16_t* pf;
    uint16_t fesc; uint16_t* out; int64_t k0, k1; int status; int64_t seg; int32_t grouped;
} eqo_pjob;

static void* eqo_pworker(void* p)
{
    eqo_pjob* j = (eqo_pjob*)p;
    uint8_t* sym = (uint8_t*)malloc((size_t)j->cs);
    j->status = 0;
    for (int64_t k = j->k0; k < j->k1; k++) {
        int64_t n, a = eqo_chunk_start(k, j->cs, j->seg, &n);
        int st = eqo_pdec(j->grouped)(j->payload + j->chunk_off[k], (int64_t)j->chunk_off[k + 1] - j->chunk_off[k],
                                       j->freq, j->rank_code, j->K, j->pf, j->fesc, sym, n);
        if (st && !j->status) j->status = st;
        for (int64_t i = 0; i < n; i++) {
            int64_t row = (a + i) / j->cols;
            j->out[a + i] = eqo_bf16_from_double(eqo_bf16_to_double(j->scales[row]) * eqo_e4m3_value(sym[i]));
        }
    }
    free(sym);
    return NULL;
}

int eqo_decode_dequant_layer_mt_pairx_seg(const uint8_t* payload, const uint32_t* chunk_off, int64_t n_chunks,
                                          int64_t cs, int64_t size, int64_t cols, int64_t seg, const uint16_t* scales,
                                          const uint16_t freq[256], const uint8_t rank_code[16], int32_t K,
                                          const uint16_t pf[225], uint16_t fesc, uint16_t* out, int threads,
                                          int32_t grouped)
{
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    eqo_pjob* jobs = (eqo_pjob*)malloc(sizeof(eqo_pjob) * (size_t)threads);
    for (int t = 0; t < threads; t++) {
        jobs[t] = (eqo_pjob){payload, chunk_off, cs, size, cols, scales, freq, rank_code, K, pf, fesc, out,
                             n_chunks * t / threads, n_chunks * (t + 1) / threads, 0, seg, grouped};
        pthread_create(&th[t], NULL, eqo_pworker, &jobs[t]);
    }
    int st = 0;
    for (int t = 0; t < threads; t++) {
        pthread_join(th[t], NULL);
        if (jobs[t].status && !st) st = jobs[t].status;
    }
    free(th);
    free(jobs);
    return st;
}

int eqo_decode_dequant_layer_mt_pair(const uint8_t* payload, const uint32_t* chunk_off, int64_t n_chunks, int64_t cs,
                                     int64_t size, int64_t cols, const uint16_t* scales, const uint16_t freq[256],
                                     const uint8_t rank_code[16], int32_t K, const uint16_t pf[225], uint16_t fesc,
                                     uint16_t* out, int threads)
{
    return eqo_decode_dequant_layer_mt_pairx_seg(payload, chunk_off, n_chunks, cs, size, cols, size, scales, freq,
                                                rank_code, K, pf, fesc, out, threads, 0);
}

/* codec 2 (R15) forms of the block and layer helpers */
int64_t eqo_encode_block_pair(const uint8_t* codes, const int64_t* layer_sizes, int32_t n_layers, int64_t cs,
                              const uint16_t freq[256], const uint8_t rank_code[16], int32_t K, const uint16_t pf[225],
                              uint16_t fesc, uint8_t* payload, int64_t cap, uint32_t* chunk_off)
{
    return eqo_encode_block_pairx(codes, layer_sizes, n_layers, cs, freq, rank_code, K, pf, fesc, payload, cap,
                                  chunk_off, 0);
}

int eqo_decode_block_pair(const uint8_t* payload, const uint32_t* chunk_off, const int64_t* layer_sizes,
                          int32_t n_layers, int64_t cs, const uint16_t freq[256], const uint8_t rank_code[16], int32_t K,
                          const uint16_t pf[225], uint16_t fesc, uint8_t* codes)
{
    return eqo_decode_block_pairx(payload, chunk_off, layer_sizes, n_layers, cs, freq, rank_code, K, pf, fesc, codes, 0);
}

int eqo_decode_dequant_layer_mt_pair_seg(const uint8_t* payload, const uint32_t* chunk_off, int64_t n_chunks,
                                         int64_t cs, int64_t size, int64_t cols, int64_t seg, const uint16_t* scales,
                                         const uint16_t freq[256], const uint8_t rank_code[16], int32_t K,
                                         const uint16_t pf[225], uint16_t fesc, uint16_t* out, int threads)
{
    return eqo_decode_dequant_layer_mt_pairx_seg(payload, chunk_off, n_chunks, cs, size, cols, seg, scales, freq,
                                                 rank_code, K, pf, fesc, out, threads, 0);
}
