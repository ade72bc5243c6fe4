// crc.cu — the optional CRC verify mode (CRC-32 over the
// uncompressed block stream).  Not on the timed path: the rANS integrity check (final state L,
// every payload byte consumed) is the free per-chunk check; this is the end-to-end one.
//
// CRC-32 (IEEE 802.3, reflected polynomial 0xEDB88320, initial value and final XOR 0xFFFFFFFF).
// The "raw" register update c ← T[(c ⊕ byte) & 0xFF] ⊕ (c >> 8) is linear over GF(2), so
//   raw(A‖B, c0) = Z_{|B|}(raw(A, c0)) ⊕ raw(B, 0),
// with Z_n the operator of n zero bytes (a 32 × 32 bit matrix).  Pass 1: one thread per 4 KB
// piece computes raw(piece, 0); pass 2 (one CTA): each thread folds a contiguous run of pieces,
// then one thread folds the runs, both with Z matrices built by repeated squaring.
#include "common.cuh"
#include "internal.h"

#include <algorithm>

namespace eq {

constexpr uint32_t kCrcPiece = 4096;              // bytes per pass-1 piece
constexpr uint32_t kCrcPoly = 0xEDB88320u;
constexpr int kCrcThreads = 256;
constexpr int kCrcFold = 1024;                    // pass-2 threads

__device__ __forceinline__ uint32_t gf2_apply(const uint32_t* m, uint32_t v) {
    uint32_t r = 0;
    #pragma unroll 4
    for (int i = 0; i < 32; ++i)
        if (v >> i & 1u) r ^= m[i];
    return r;
}

// dst = src · src (the operator applied twice)
__device__ void gf2_square(uint32_t* dst, const uint32_t* src) {
    for (int i = 0; i < 32; ++i) dst[i] = gf2_apply(src, src[i]);
}

// z = Z_n (n zero bytes): the one-bit operator (column i = image of bit i), squared three times
// for one byte, then the powers of two of n multiplied in (all powers of one operator commute)
__device__ void zero_bytes_op(uint32_t* z, uint64_t n) {
    uint32_t a[32], b[32];
    a[0] = kCrcPoly;
    for (int i = 1; i < 32; ++i) a[i] = 1u << (i - 1);
    gf2_square(b, a);                              // 2 bits
    gf2_square(a, b);                              // 4 bits
    gf2_square(b, a);                              // 8 bits: one zero byte
    for (int i = 0; i < 32; ++i) z[i] = 1u << i;  // identity
    uint32_t* p = b;
    uint32_t* q = a;
    while (n) {
        if (n & 1) {
            uint32_t t[32];
            for (int i = 0; i < 32; ++i) t[i] = gf2_apply(p, z[i]);
            for (int i = 0; i < 32; ++i) z[i] = t[i];
        }
        n >>= 1;
        if (n) {
            gf2_square(q, p);
            uint32_t* s = p; p = q; q = s;
        }
    }
}

__global__ void __launch_bounds__(kCrcThreads) k_crc_pieces(const uint8_t* __restrict__ data, uint64_t n,
                                                            uint64_t n_pieces, uint32_t* __restrict__ raw) {
    __shared__ uint32_t tab[256];
    for (int i = threadIdx.x; i < 256; i += kCrcThreads) {
        uint32_t c = (uint32_t)i;
        for (int k = 0; k < 8; ++k) c = (c >> 1) ^ ((c & 1u) ? kCrcPoly : 0u);
        tab[i] = c;
    }
    __syncthreads();
    for (uint64_t p = blockIdx.x * (uint64_t)kCrcThreads + threadIdx.x; p < n_pieces;
         p += (uint64_t)gridDim.x * kCrcThreads) {
        const uint64_t a = p * kCrcPiece, e = min(n, a + kCrcPiece);
        uint32_t c = 0;
        uint64_t i = a;
        if (((reinterpret_cast<uintptr_t>(data) + a) & 15) == 0)
            for (; i + 16 <= e; i += 16) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(data + i));
                const uint32_t w[4] = {v.x, v.y, v.z, v.w};
                #pragma unroll
                for (int k = 0; k < 16; ++k) c = tab[(c ^ (w[k >> 2] >> (8 * (k & 3)))) & 0xFFu] ^ (c >> 8);
            }
        for (; i < e; ++i) c = tab[(c ^ data[i]) & 0xFFu] ^ (c >> 8);
        raw[p] = c;
    }
}

__global__ void __launch_bounds__(kCrcFold) k_crc_fold(const uint32_t* __restrict__ raw, uint64_t n, uint64_t n_pieces,
                                                       uint32_t* __restrict__ out) {
    __shared__ uint32_t zp[32], zr[32], zt[32];
    __shared__ uint32_t part[kCrcFold];
    const uint64_t per = (n_pieces + kCrcFold - 1) / kCrcFold;   // pieces per run
    if (threadIdx.x == 0) zero_bytes_op(zp, kCrcPiece);
    if (threadIdx.x == 32) zero_bytes_op(zr, per * kCrcPiece);   // a whole run
    __syncthreads();
    // run t: pieces [t·per, min((t+1)·per, n_pieces)); its raw CRC from register 0
    const uint64_t a = threadIdx.x * per, e = min(n_pieces, a + per);
    uint32_t c = 0;
    for (uint64_t p = a; p < e; ++p) {
        const uint64_t len = (p + 1 == n_pieces) ? n - p * kCrcPiece : kCrcPiece;
        if (len == kCrcPiece) {
            c = gf2_apply(zp, c) ^ raw[p];
        } else {                                   // the ragged last piece (one thread)
            uint32_t z[32];
            zero_bytes_op(z, len);
            c = gf2_apply(z, c) ^ raw[p];
        }
    }
    part[threadIdx.x] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        // register after the whole message from the initial 0xFFFFFFFF: Z_n(~0) ⊕ raw(msg, 0)
        uint32_t acc = 0;
        for (uint32_t t = 0; t < kCrcFold; ++t) {
            const uint64_t ta = t * per, te = min(n_pieces, ta + per);
            if (ta >= te) break;
            const uint64_t bytes = min(n, te * kCrcPiece) - ta * kCrcPiece;
            if (te - ta == per && bytes == per * kCrcPiece) {
                acc = gf2_apply(zr, acc) ^ part[t];
            } else {
                zero_bytes_op(zt, bytes);
                acc = gf2_apply(zt, acc) ^ part[t];
            }
        }
        zero_bytes_op(zt, n);
        *out = (gf2_apply(zt, 0xFFFFFFFFu) ^ acc) ^ 0xFFFFFFFFu;
    }
}

}  // namespace eq

using namespace eq;

extern "C" uint64_t eq_crc32_scratch_bytes(uint64_t n) {
    return 4 * ((n + kCrcPiece - 1) / kCrcPiece) + 16;
}

extern "C" eq_status eq_crc32(const void* data, uint64_t n, uint32_t* crc, void* scratch, uint64_t scratch_bytes,
                              eq_stream_t stream) {
    if (!crc || (n && (!data || !scratch))) return EQ_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {                                  // CRC-32 of the empty message
        EQ_CUDA_TRY(cudaMemsetAsync(crc, 0, 4, st));
        return EQ_OK;
    }
    if (scratch_bytes < eq_crc32_scratch_bytes(n)) return EQ_ERR_BUFFER;
    const uint64_t pieces = (n + kCrcPiece - 1) / kCrcPiece;
    const unsigned grid = (unsigned)std::min<uint64_t>((pieces + kCrcThreads - 1) / kCrcThreads, 148ull * 16);
    k_crc_pieces<<<grid, kCrcThreads, 0, st>>>(static_cast<const uint8_t*>(data), n, pieces,
                                               static_cast<uint32_t*>(scratch));
    EQ_CUDA_TRY(cudaGetLastError());
    k_crc_fold<<<1, kCrcFold, 0, st>>>(static_cast<const uint32_t*>(scratch), n, pieces, crc);
    EQ_CUDA_TRY(cudaGetLastError());
    return EQ_OK;
}
