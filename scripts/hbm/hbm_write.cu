// HBM write-bandwidth probes (context for the decoder roofline; not part of the library):
// grid-stride 256-bit stores (st.global.L1::no_allocate.L2::evict_first.v8, as the decoder's),
// 128-bit stores, and a 1 : 8 read : write mix (32 bytes read, 256 bytes written per thread step).
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_write256(uint8_t* p, uint64_t n32, uint32_t v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n32; i += (uint64_t)gridDim.x * blockDim.x)
        asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + i * 32),
                     "r"(v) : "memory");
}
__global__ void k_write128(uint4* p, uint64_t n16, uint32_t v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(v, v, v, v);
}
// each "item": read 32 B of src, write 8 × 32 B of dst (the decoder's ≈ 1 : 8 in : out)
__global__ void k_mix18(const uint4* src, uint8_t* dst, uint64_t items) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < items; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 a = __ldcs(src + 2 * i), b = __ldcs(src + 2 * i + 1);
        const uint32_t v = a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
        for (int k = 0; k < 8; ++k)
            asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(
                             dst + (i * 8 + k) * 32),
                         "r"(v + k) : "memory");
    }
}

extern "C" int hbm_write256(void* p, uint64_t bytes, int blocks, int threads, void* stream) {
    k_write256<<<blocks, threads, 0, (cudaStream_t)stream>>>((uint8_t*)p, bytes / 32, 1u);
    return (int)cudaGetLastError();
}
extern "C" int hbm_write128(void* p, uint64_t bytes, int blocks, int threads, void* stream) {
    k_write128<<<blocks, threads, 0, (cudaStream_t)stream>>>((uint4*)p, bytes / 16, 1u);
    return (int)cudaGetLastError();
}
extern "C" int hbm_mix18(const void* src, void* dst, uint64_t dst_bytes, int blocks, int threads, void* stream) {
    k_mix18<<<blocks, threads, 0, (cudaStream_t)stream>>>((const uint4*)src, (uint8_t*)dst, dst_bytes / 256);
    return (int)cudaGetLastError();
}

// the decoder's pattern: thread t owns a contiguous region of `region` bytes (its chunk's
// output) and writes it front to back, `burst` × 32 bytes per step; all threads concurrently
template <int BURST, bool EF>
__global__ void k_scatter(uint8_t* p, uint64_t region, uint64_t threads_total) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= threads_total) return;
    uint8_t* base = p + t * region;
    for (uint64_t off = 0; off < region; off += 32 * BURST) {
        #pragma unroll
        for (int b = 0; b < BURST; ++b) {
            if (EF)
                asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(
                                 base + off + 32 * b), "r"((uint32_t)off) : "memory");
            else
                asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(base + off + 32 * b),
                             "r"((uint32_t)off) : "memory");
        }
    }
}
extern "C" int hbm_scatter(void* p, uint64_t region, uint64_t threads_total, int burst, int ef, int tpb, void* stream) {
    const unsigned blocks = (unsigned)((threads_total + tpb - 1) / tpb);
    cudaStream_t s = (cudaStream_t)stream;
    if (burst == 1 && ef) k_scatter<1, true><<<blocks, tpb, 0, s>>>((uint8_t*)p, region, threads_total);
    else if (burst == 1) k_scatter<1, false><<<blocks, tpb, 0, s>>>((uint8_t*)p, region, threads_total);
    else if (burst == 4 && ef) k_scatter<4, true><<<blocks, tpb, 0, s>>>((uint8_t*)p, region, threads_total);
    else k_scatter<4, false><<<blocks, tpb, 0, s>>>((uint8_t*)p, region, threads_total);
    return (int)cudaGetLastError();
}
