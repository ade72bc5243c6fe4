// api.cu — composite C-ABI entry points of libentquant: Alg. 1 for one block
// (eq_quantize_encode), sizing, error mapping, the host-buffer end-to-end decode, and the
// global-λ calibration of P:192 / P:507 (reading R11).  All arithmetic of the method runs
// in the kernels of quant.cu / table.cu / rans_enc.cu / rans_dec.cu; this file is host
// control flow (validation, launch order, scratch carving, one λ bisection loop).
#include "common.cuh"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

using namespace eq;

namespace {

uint64_t align_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

eq_status check_layers(const eq_tensor* layers, uint32_t n_layers) {
    if (!layers || n_layers == 0 || n_layers > EQ_MAX_LAYERS) return EQ_ERR_ARG;
    for (uint32_t l = 0; l < n_layers; ++l) {
        if (!layers[l].w) return EQ_ERR_ARG;
        if (layers[l].rows < 1 || layers[l].cols < 1 || layers[l].rows > (1ll << 31) ||
            layers[l].cols > (1ll << 31))
            return EQ_ERR_SHAPE;
    }
    return EQ_OK;
}

eq_status check_params(const eq_params* p) {
    if (!p) return EQ_ERR_ARG;
    if (p->format > EQ_FMT_INT8 || p->prob_bits != EQ_PROB_BITS) return EQ_ERR_ARG;
    if (p->chunk_symbols == 0 || p->chunk_symbols > 262144u) return EQ_ERR_ARG;
    if (p->scale_mode > EQ_SCALES_GIVEN) return EQ_ERR_ARG;
    if (p->codec > EQ_CODEC_PAIR_G) return EQ_ERR_ARG;
    if (p->chunk_mode > EQ_CHUNK_INTERLEAVED) return EQ_ERR_ARG;
    if (p->chunk_mode == EQ_CHUNK_INTERLEAVED && (!is_pair_codec(p->codec) || p->chunk_symbols % 32 != 0))
        return EQ_ERR_ARG;
    if (p->scale_mode == EQ_SCALES_SEARCH && !(p->lambda >= 0.0)) return EQ_ERR_ARG;
    return EQ_OK;
}

struct EncodeScratch {
    uint8_t* codes;
    uint64_t* hist;
    uint32_t* sizes;
    uint64_t* total;
    uint32_t* err;
    void* search;
    uint64_t search_bytes;
    uint64_t bytes;
};

EncodeScratch carve(const eq_tensor* layers, uint32_t n_layers, uint32_t n_chunks, char* base) {
    EncodeScratch s{};
    uint64_t syms = 0, sb = 0;
    for (uint32_t l = 0; l < n_layers; ++l) {
        syms += (uint64_t)layers[l].rows * (uint64_t)layers[l].cols;
        sb = std::max<uint64_t>(sb, eq_search_scratch_bytes(&layers[l]));
    }
    uint64_t pos = 0;
    auto take = [&](uint64_t n) { uint64_t p = pos; pos = align_up(pos + n, 256); return p; };
    const uint64_t o_codes = take(syms), o_hist = take(256 * 8), o_sizes = take(4ull * n_chunks),
                   o_total = take(8), o_err = take(4), o_search = take(sb);
    s.bytes = pos;
    if (base) {
        s.codes = (uint8_t*)(base + o_codes);
        s.hist = (uint64_t*)(base + o_hist);
        s.sizes = (uint32_t*)(base + o_sizes);
        s.total = (uint64_t*)(base + o_total);
        s.err = (uint32_t*)(base + o_err);
        s.search = base + o_search;
    }
    s.search_bytes = sb;
    return s;
}

uint64_t count_chunks(const eq_tensor* layers, uint32_t n_layers, uint32_t cs, uint32_t mode) {
    uint64_t n = 0;
    for (uint32_t l = 0; l < n_layers; ++l) n += layer_chunks(mode, layers[l].rows, layers[l].cols, cs);
    return n;
}

eq_status err_to_status(uint32_t e) {
    if (e & EQ_EF_TRUNCATED) return EQ_ERR_TRUNCATED;
    if (e & EQ_EF_CORRUPT) return EQ_ERR_CORRUPT;
    if (e & EQ_EF_EMPTY) return EQ_ERR_EMPTY;
    if (e & EQ_EF_UNKNOWN_SYMBOL) return EQ_ERR_UNKNOWN_SYMBOL;
    if (e & EQ_EF_BUFFER) return EQ_ERR_BUFFER;
    return EQ_OK;
}

}  // namespace

extern "C" const char* eq_status_string(eq_status s) {
    switch (s) {
        case EQ_OK: return "ok";
        case EQ_ERR_ARG: return "arg";
        case EQ_ERR_SHAPE: return "shape";
        case EQ_ERR_EMPTY: return "empty";
        case EQ_ERR_BUFFER: return "buffer";
        case EQ_ERR_CORRUPT: return "corrupt";
        case EQ_ERR_TRUNCATED: return "truncated";
        case EQ_ERR_UNKNOWN_SYMBOL: return "unknown-symbol";
        case EQ_ERR_UNREACHABLE_TARGET: return "unreachable-target";
        case EQ_ERR_CUDA: return "cuda";
    }
    return "?";
}

extern "C" const char* eq_version(void) { return "entquant-b200 0.1 (sm_100a)"; }

extern "C" eq_status eq_encode_bounds(const eq_tensor* layers, uint32_t n_layers, const eq_params* p,
                                      uint64_t* payload_cap, uint32_t* n_chunks, uint64_t* scratch_bytes) {
    EQ_TRY(check_layers(layers, n_layers));
    EQ_TRY(check_params(p));
    if (p->chunk_mode == EQ_CHUNK_INTERLEAVED)        // R17: 16-symbol groups must not straddle rows
        for (uint32_t l = 0; l < n_layers; ++l)
            if (layers[l].cols % 16 != 0) return EQ_ERR_SHAPE;
    uint64_t syms = 0;
    for (uint32_t l = 0; l < n_layers; ++l) syms += (uint64_t)layers[l].rows * (uint64_t)layers[l].cols;
    const uint64_t nc = count_chunks(layers, n_layers, p->chunk_symbols, p->chunk_mode);
    // worst case per chunk: 4-byte state + at most 2 renormalisation bytes per symbol
    // (two bytes, EQ_CODEC_BYTE, or one 16-bit word, EQ_CODEC_WORD)
    // (EQ_CODEC_PAIR: an escaped pair is three words for two symbols)
    const uint64_t cap = align_up(4 * nc + (is_pair_codec(p->codec) ? 3 : 2) * syms + EQ_PAYLOAD_SLACK, 256);
    if (payload_cap) *payload_cap = cap;
    if (n_chunks) *n_chunks = (uint32_t)nc;
    if (scratch_bytes) *scratch_bytes = carve(layers, n_layers, (uint32_t)nc, nullptr).bytes;
    if (nc > 0xFFFFFFFFull) return EQ_ERR_SHAPE;
    return EQ_OK;
}

extern "C" eq_status eq_check(const uint32_t* d_err, eq_stream_t stream) {
    if (!d_err) return EQ_ERR_ARG;
    uint32_t e = 0;
    EQ_CUDA_TRY(cudaMemcpyAsync(&e, d_err, 4, cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    EQ_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    return err_to_status(e);
}

extern "C" eq_status eq_quantize_encode(const eq_tensor* layers, uint32_t n_layers, const eq_params* p,
                                        eq_block* out, void* scratch, uint64_t scratch_bytes,
                                        eq_stream_t stream) {
    EQ_TRY(check_layers(layers, n_layers));
    EQ_TRY(check_params(p));
    if (!out || !out->payload || !out->chunk_off || !out->freq || !out->scales || !scratch) return EQ_ERR_ARG;
    uint64_t cap_needed, need;
    uint32_t nc;
    EQ_TRY(eq_encode_bounds(layers, n_layers, p, &cap_needed, &nc, &need));
    if (scratch_bytes < need) return EQ_ERR_BUFFER;
    cudaStream_t st = (cudaStream_t)stream;
    EncodeScratch S = carve(layers, n_layers, nc, (char*)scratch);

    out->n_layers = n_layers;
    out->format = p->format;
    out->codec = p->codec;
    out->chunk_mode = p->chunk_mode;
    out->n_chunks = nc;
    out->chunk_symbols = p->chunk_symbols;
    for (uint32_t l = 0; l < EQ_MAX_LAYERS; ++l) {
        out->layer_rows[l] = l < n_layers ? layers[l].rows : 0;
        out->layer_cols[l] = l < n_layers ? layers[l].cols : 0;
    }
    EQ_CUDA_TRY(cudaMemsetAsync(S.hist, 0, 256 * 8, st));
    EQ_CUDA_TRY(cudaMemsetAsync(S.err, 0, 4, st));
    // Alg. 1 l.1-3 per layer: scales, then quantise + histogram into the block stream
    uint64_t sym = 0, row = 0;
    for (uint32_t l = 0; l < n_layers; ++l) {
        uint16_t* sl = out->scales + row;
        const bool excluded = (p->exclude_mask >> l) & 1u;        // λ = 0, still coded
        if (p->scale_mode == EQ_SCALES_SEARCH && !excluded) {
            EQ_TRY(eq_search_scales(&layers[l], p->format, &p->lambda, 1, p->oct_lo, p->oct_hi, nullptr, 0, sl,
                                    nullptr, S.search, S.search_bytes, stream));
        } else if (p->scale_mode == EQ_SCALES_ABSMAX || (p->scale_mode == EQ_SCALES_SEARCH && excluded)) {
            EQ_TRY(eq_absmax(&layers[l], p->format, sl, stream));
        }
        EQ_TRY(eq_quantize_hist(&layers[l], p->format, sl, nullptr, 0, S.codes + sym, S.hist, stream));
        sym += (uint64_t)layers[l].rows * (uint64_t)layers[l].cols;
        row += (uint64_t)layers[l].rows;
    }
    // metadata ℳ and Alg. 1 l.4-5
    EQ_TRY(eq_build_table(S.hist, out->freq, S.err, stream));
    if (is_pair_codec(p->codec)) EQ_TRY(eq_build_pair_table(S.hist, out->freq, S.err, stream));   // R15
    EQ_TRY(eq_rans_encode(S.codes, out, S.sizes, S.total, S.err, stream));
    uint64_t total = 0;
    uint32_t e = 0;
    EQ_CUDA_TRY(cudaMemcpyAsync(&total, S.total, 8, cudaMemcpyDeviceToHost, st));
    EQ_CUDA_TRY(cudaMemcpyAsync(&e, S.err, 4, cudaMemcpyDeviceToHost, st));
    EQ_CUDA_TRY(cudaStreamSynchronize(st));
    if (e) return err_to_status(e);
    out->payload_bytes = total;
    if (out->payload_cap < total + EQ_PAYLOAD_SLACK) return EQ_ERR_BUFFER;
    return EQ_OK;
}

// ---------------------------------------------------------------- e2e with host buffers
// bytes of a block's table buffer: 256 u16, or 512 for the pair codecs (include/entquant.h)
static uint64_t table_bytes(const eq_block& b) { return is_pair_codec(b.codec) ? 1024 : 512; }
extern "C" uint64_t eq_decode_host_workspace_bytes(const eq_block* blocks, uint32_t n_blocks, uint32_t out_dtype) {
    if (!blocks || n_blocks == 0) return 0;
    uint64_t total = 0, pos = 0;
    if (eq_arena_layout(blocks, n_blocks, out_dtype, nullptr, &total) != EQ_OK) return 0;
    for (uint32_t b = 0; b < n_blocks; ++b) {
        uint64_t rows = 0;
        for (uint32_t l = 0; l < blocks[b].n_layers; ++l) rows += (uint64_t)blocks[b].layer_rows[l];
        pos += align_up(blocks[b].payload_bytes + EQ_PAYLOAD_SLACK, 256);
        pos += align_up(4ull * (blocks[b].n_chunks + 1), 256);
        pos += table_bytes(blocks[b]) + align_up(2 * rows, 256);
    }
    return align_up(pos, 256) + total + 256;
}

extern "C" eq_status eq_decode_dequant_host(const eq_block* blocks, uint32_t n_blocks, uint32_t out_dtype,
                                            void* arena_host, uint64_t arena_bytes, void* workspace,
                                            uint64_t workspace_bytes, eq_stream_t stream) {
    if (!blocks || n_blocks == 0 || !arena_host || !workspace) return EQ_ERR_ARG;
    const uint64_t need = eq_decode_host_workspace_bytes(blocks, n_blocks, out_dtype);
    if (need == 0) return EQ_ERR_ARG;
    if (workspace_bytes < need) return EQ_ERR_BUFFER;
    uint64_t total = 0;
    std::vector<uint64_t> offs((size_t)n_blocks * EQ_MAX_LAYERS);
    EQ_TRY(eq_arena_layout(blocks, n_blocks, out_dtype, offs.data(), &total));
    if (arena_bytes < total) return EQ_ERR_BUFFER;
    cudaStream_t st = (cudaStream_t)stream;
    char* ws = (char*)workspace;
    uint64_t pos = 0;
    std::vector<eq_block> dev(blocks, blocks + n_blocks);
    for (uint32_t b = 0; b < n_blocks; ++b) {
        const eq_block& h = blocks[b];
        eq_block& d = dev[b];
        uint64_t rows = 0;
        for (uint32_t l = 0; l < h.n_layers; ++l) rows += (uint64_t)h.layer_rows[l];
        d.payload = (uint8_t*)(ws + pos);
        d.payload_cap = align_up(h.payload_bytes + EQ_PAYLOAD_SLACK, 256);
        pos += d.payload_cap;
        d.chunk_off = (uint32_t*)(ws + pos);
        pos += align_up(4ull * (h.n_chunks + 1), 256);
        d.freq = (uint16_t*)(ws + pos);
        pos += table_bytes(h);
        d.scales = (uint16_t*)(ws + pos);
        pos += align_up(2 * rows, 256);
    }
    pos = align_up(pos, 256);
    char* arena = ws + pos;
    uint32_t* err = (uint32_t*)(ws + pos + total);
    // Three-stage pipeline over groups of blocks: host→device copy of group g+1 (copy stream)
    // and device→host copy of group g−1 (second copy stream) overlap the decode of group g
    // (the caller's stream); PCIe is full duplex, so the step costs ≈ max(H2D, D2H) + one
    // group's decode.  Streams and events live for this call only (the library keeps no state).
    const uint32_t n_groups = std::min<uint32_t>(n_blocks, 8u);
    const uint32_t per = (n_blocks + n_groups - 1) / n_groups;
    cudaStream_t s_in = nullptr, s_out = nullptr;
    std::vector<cudaEvent_t> ev_in(n_groups, nullptr), ev_dec(n_groups, nullptr);
    cudaEvent_t ev_start = nullptr, ev_done = nullptr;
    eq_status rs = EQ_OK;
    auto ck = [&](cudaError_t e) { if (e != cudaSuccess && rs == EQ_OK) rs = EQ_ERR_CUDA; return e == cudaSuccess; };
    ck(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
    ck(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
    ck(cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming));
    ck(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
    for (uint32_t g = 0; g < n_groups; ++g) {
        ck(cudaEventCreateWithFlags(&ev_in[g], cudaEventDisableTiming));
        ck(cudaEventCreateWithFlags(&ev_dec[g], cudaEventDisableTiming));
    }
    if (rs == EQ_OK) {
        ck(cudaMemsetAsync(err, 0, 4, st));
        ck(cudaEventRecord(ev_start, st));                        // work queued before this call
        ck(cudaStreamWaitEvent(s_in, ev_start, 0));
        for (uint32_t g = 0; g < n_groups && rs == EQ_OK; ++g) {
            const uint32_t b0 = g * per, b1 = std::min(n_blocks, b0 + per);
            if (b0 >= b1) break;
            for (uint32_t b = b0; b < b1; ++b) {
                const eq_block& h = blocks[b];
                const eq_block& d = dev[b];
                uint64_t rows = 0;
                for (uint32_t l = 0; l < h.n_layers; ++l) rows += (uint64_t)h.layer_rows[l];
                ck(cudaMemcpyAsync(d.payload, h.payload, h.payload_bytes, cudaMemcpyHostToDevice, s_in));
                ck(cudaMemcpyAsync(d.chunk_off, h.chunk_off, 4ull * (h.n_chunks + 1), cudaMemcpyHostToDevice, s_in));
                ck(cudaMemcpyAsync(d.freq, h.freq, table_bytes(h), cudaMemcpyHostToDevice, s_in));
                ck(cudaMemcpyAsync(d.scales, h.scales, 2 * rows, cudaMemcpyHostToDevice, s_in));
            }
            ck(cudaEventRecord(ev_in[g], s_in));
            ck(cudaStreamWaitEvent(st, ev_in[g], 0));
            const uint64_t a0 = offs[(size_t)b0 * EQ_MAX_LAYERS];
            const uint64_t a1 = b1 < n_blocks ? offs[(size_t)b1 * EQ_MAX_LAYERS] : total;
            const eq_status ds = eq_decode_dequant(dev.data() + b0, b1 - b0, out_dtype, arena + a0, a1 - a0, err, stream);
            if (ds != EQ_OK && rs == EQ_OK) rs = ds;
            ck(cudaEventRecord(ev_dec[g], st));
            ck(cudaStreamWaitEvent(s_out, ev_dec[g], 0));
            ck(cudaMemcpyAsync((char*)arena_host + a0, arena + a0, a1 - a0, cudaMemcpyDeviceToHost, s_out));
        }
        ck(cudaEventRecord(ev_done, s_out));
        ck(cudaStreamWaitEvent(st, ev_done, 0));                  // the caller's stream sees the result
    }
    if (s_in) cudaStreamSynchronize(s_in);
    if (s_out) cudaStreamSynchronize(s_out);
    for (uint32_t g = 0; g < n_groups; ++g) {
        if (ev_in[g]) cudaEventDestroy(ev_in[g]);
        if (ev_dec[g]) cudaEventDestroy(ev_dec[g]);
    }
    if (ev_start) cudaEventDestroy(ev_start);
    if (ev_done) cudaEventDestroy(ev_done);
    if (s_in) cudaStreamDestroy(s_in);
    if (s_out) cudaStreamDestroy(s_out);
    if (rs != EQ_OK) return rs;
    return eq_check(err, stream);
}

// ---------------------------------------------------------------- λ calibration (R11)
namespace {
constexpr int kGrid = 32;

struct CalibScratch {
    uint32_t* rows;     // per layer sampled row lists, concatenated
    uint16_t* scales;   // [kGrid][rows] per layer, concatenated
    uint64_t* hist;     // [kGrid][256]
    void* search;
    uint64_t search_bytes;
    uint64_t bytes;
};

CalibScratch carve_calib(const eq_tensor* layers, uint32_t n, uint32_t stride, char* base) {
    uint64_t nrows = 0, srows = 0, sb = 0;
    for (uint32_t l = 0; l < n; ++l) {
        nrows += (uint64_t)(layers[l].rows + stride - 1) / stride;
        srows += (uint64_t)layers[l].rows;
        sb = std::max<uint64_t>(sb, eq_search_scratch_bytes(&layers[l]));
    }
    uint64_t pos = 0;
    auto take = [&](uint64_t b) { uint64_t p = pos; pos = align_up(pos + b, 256); return p; };
    const uint64_t o_rows = take(4 * nrows), o_sc = take(2ull * kGrid * srows), o_h = take(8ull * kGrid * 256),
                   o_s = take(sb);
    CalibScratch c{};
    c.bytes = pos;
    c.search_bytes = sb;
    if (base) {
        c.rows = (uint32_t*)(base + o_rows);
        c.scales = (uint16_t*)(base + o_sc);
        c.hist = (uint64_t*)(base + o_h);
        c.search = base + o_s;
    }
    return c;
}

double entropy_bits(const uint64_t* h) {
    double T = 0.0, H = 0.0;
    for (int c = 0; c < 256; ++c) T += (double)h[c];
    if (T <= 0) return 0.0;
    for (int c = 0; c < 256; ++c)
        if (h[c]) {
            const double p = (double)h[c] / T;
            H -= p * std::log2(p);
        }
    return H;
}
}  // namespace

extern "C" uint64_t eq_calibrate_scratch_bytes(const eq_tensor* layers, uint32_t n_layers, uint32_t row_stride) {
    if (!layers || n_layers == 0 || row_stride == 0) return 0;
    return carve_calib(layers, n_layers, row_stride, nullptr).bytes;
}

extern "C" eq_status eq_calibrate_lambda(const eq_tensor* layers, uint32_t n_layers, const eq_params* p,
                                         double target_bits, uint32_t row_stride, double* lambda_out,
                                         double* est_bits_out, void* scratch, uint64_t scratch_bytes,
                                         eq_stream_t stream) {
    if (!layers || n_layers == 0 || !p || !lambda_out || !scratch || row_stride == 0) return EQ_ERR_ARG;
    for (uint32_t l = 0; l < n_layers; ++l)
        if (!layers[l].w || layers[l].rows < 1 || layers[l].cols < 1) return EQ_ERR_SHAPE;
    {
        eq_params q = *p;                          // λ is the output here: validate everything else
        q.lambda = 0.0;
        EQ_TRY(check_params(&q));
    }
    if (!(target_bits > 0.0)) return EQ_ERR_ARG;
    if (scratch_bytes < eq_calibrate_scratch_bytes(layers, n_layers, row_stride)) return EQ_ERR_BUFFER;
    cudaStream_t st = (cudaStream_t)stream;
    CalibScratch C = carve_calib(layers, n_layers, row_stride, (char*)scratch);

    // side information per parameter of the full layer set: chunk offsets,
    // bf16 scales, one table per 7 layers (a block: 256 x u16, or 512 x u16 for the pair
    // codec), + 4-byte states.
    double params = 0, rows_total = 0, chunks = 0;
    for (uint32_t l = 0; l < n_layers; ++l) {
        const double sz = (double)layers[l].rows * (double)layers[l].cols;
        params += sz;
        rows_total += (double)layers[l].rows;
        chunks += (double)layer_chunks(p->chunk_mode, layers[l].rows, layers[l].cols, p->chunk_symbols);
    }
    const double side = (8.0 * (4.0 * chunks + 4.0 * chunks + 2.0 * rows_total) + (is_pair_codec(p->codec) ? 8192.0 : 4096.0) * std::ceil(n_layers / 7.0)) / params;

    // sampled row lists
    std::vector<uint32_t> rl;
    std::vector<uint64_t> rl_off(n_layers + 1, 0), sc_off(n_layers + 1, 0);
    for (uint32_t l = 0; l < n_layers; ++l) {
        rl_off[l] = rl.size();
        for (int64_t r = 0; r < layers[l].rows; r += row_stride) rl.push_back((uint32_t)r);
        sc_off[l + 1] = sc_off[l] + (uint64_t)layers[l].rows * kGrid;
    }
    rl_off[n_layers] = rl.size();
    EQ_CUDA_TRY(cudaMemcpyAsync(C.rows, rl.data(), 4 * rl.size(), cudaMemcpyHostToDevice, st));

    auto evaluate = [&](const std::vector<double>& lam, std::vector<double>& est) -> eq_status {
        EQ_CUDA_TRY(cudaMemsetAsync(C.hist, 0, 8ull * kGrid * 256, st));
        for (uint32_t l = 0; l < n_layers; ++l) {
            const uint32_t nr = (uint32_t)(rl_off[l + 1] - rl_off[l]);
            uint16_t* sc = C.scales + sc_off[l];
            EQ_TRY(eq_search_scales(&layers[l], p->format, lam.data(), (uint32_t)lam.size(), p->oct_lo, p->oct_hi,
                                    C.rows + rl_off[l], nr, sc, nullptr, C.search, C.search_bytes, stream));
            for (size_t k = 0; k < lam.size(); ++k)
                EQ_TRY(eq_quantize_hist(&layers[l], p->format, sc + k * layers[l].rows, C.rows + rl_off[l], nr, nullptr,
                                        C.hist + 256 * k, stream));
        }
        std::vector<uint64_t> h(256 * lam.size());
        EQ_CUDA_TRY(cudaMemcpyAsync(h.data(), C.hist, 8 * h.size(), cudaMemcpyDeviceToHost, st));
        EQ_CUDA_TRY(cudaStreamSynchronize(st));
        est.resize(lam.size());
        for (size_t k = 0; k < lam.size(); ++k) est[k] = entropy_bits(&h[256 * k]) * 1.002 + side;
        return EQ_OK;
    };

    double lo = 0.0, hi = 1e6;
    std::vector<double> lam(kGrid), est;
    double best_l = 0.0, best_e = 0.0;
    for (int pass = 0; pass < 3; ++pass) {
        for (int k = 0; k < kGrid; ++k) {
            if (pass == 0)
                lam[k] = k == 0 ? 0.0 : std::pow(10.0, -2.0 + 8.0 * (k - 1) / (kGrid - 2));
            else
                lam[k] = lo == 0.0 ? hi * k / (kGrid - 1) : lo * std::pow(hi / lo, (double)k / (kGrid - 1));
        }
        EQ_TRY(evaluate(lam, est));
        if (pass == 0 && (target_bits > est[0] + 1e-9 || target_bits < est[kGrid - 1] - 1e-9))
            return EQ_ERR_UNREACHABLE_TARGET;
        // est is (essentially) non-increasing in λ: bracket the target
        int k = 0;
        while (k + 1 < kGrid && est[k + 1] > target_bits) ++k;
        lo = lam[k];
        hi = lam[std::min(k + 1, kGrid - 1)];
        const int kb = (k + 1 < kGrid && std::fabs(est[k + 1] - target_bits) < std::fabs(est[k] - target_bits)) ? k + 1 : k;
        best_l = lam[kb];
        best_e = est[kb];
    }
    *lambda_out = best_l;
    if (est_bits_out) *est_bits_out = best_e;
    return EQ_OK;
}
