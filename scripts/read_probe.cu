// read_probe.cu -- achievable HBM READ bandwidth on this B200 at the K1
// working-set sizes (the roofline's practical ceiling for a read-only
// streaming kernel; MEASURED_PEAKS.json's figure is a read+write copy).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/_bin/read_probe scripts/read_probe.cu
//   scripts/_bin/read_probe [MB ...]
//
// Variants (each: 148*k CTAs, every CTA streams a contiguous range):
//   bulk  : per-warp ring of S stages of cp.async.bulk (global -> smem, mbarrier),
//           the K1 structure without the math
//   ldg   : plain 128-bit ld.global.nc, grid-stride, many CTAs
// Prints one JSON line per (variant, size): best and median of 20 launches.
// Between launches the L2 is flushed by a 256 MB memset (FLUSH=write, the
// default), a 256 MB read (FLUSH=read: leaves clean lines, no write-back in the
// timed kernel) or not at all (NOFLUSH=1 or FLUSH=none).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));     \
            exit(1);                                                                       \
        }                                                                                  \
    } while (0)

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned n) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(b);
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(a),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            (unsigned)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
        : "memory");
}

template <int W, int S, int CHUNK>
__global__ void __launch_bounds__(W * 32) k_bulk(const uint8_t* src, size_t bytes, unsigned* sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bars[W][S];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t nchunks = bytes / CHUNK;
    const size_t c0 = nchunks * blockIdx.x / gridDim.x, c1 = nchunks * (blockIdx.x + 1) / gridDim.x;
    uint8_t* ring = smem + size_t(warp) * S * CHUNK;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(&bars[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const size_t mine = c1 > c0 + warp ? (c1 - c0 - warp + W - 1) / W : 0;
    if (lane == 0)
        for (int s = 0; s < S && s < (int)mine; ++s) {
            mbar_expect(&bars[warp][s], CHUNK);
            bulk(ring + s * CHUNK, src + (c0 + warp + size_t(s) * W) * CHUNK, CHUNK, &bars[warp][s]);
        }
    unsigned acc = 0;
    for (size_t k = 0; k < mine; ++k) {
        const int s = int(k % S);
        mbar_wait(&bars[warp][s], unsigned((k / S) & 1));
        acc += reinterpret_cast<const unsigned*>(ring + s * CHUNK)[lane];
        __syncwarp();
        if (lane == 0 && k + S < mine) {
            mbar_expect(&bars[warp][s], CHUNK);
            bulk(ring + s * CHUNK, src + (c0 + warp + (k + S) * W) * CHUNK, CHUNK, &bars[warp][s]);
        }
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

// The split kernel's fp32 stream: every stage is a K chunk and a V chunk at
// the same offset of two separate arrays (W warps x S stages, CHUNK bytes each).
template <int W, int S, int CHUNK>
__global__ void __launch_bounds__(W * 32) k_bulk_kv(const uint8_t* k, const uint8_t* v, size_t bytes, unsigned* sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t bars[W][S];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t nchunks = bytes / CHUNK;
    const size_t c0 = nchunks * blockIdx.x / gridDim.x, c1 = nchunks * (blockIdx.x + 1) / gridDim.x;
    uint8_t* ring = smem + size_t(warp) * S * 2 * CHUNK;
    if (lane == 0)
        for (int s = 0; s < S; ++s) mbar_init(&bars[warp][s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const size_t mine = c1 > c0 + warp ? (c1 - c0 - warp + W - 1) / W : 0;
    auto issue = [&](size_t kk, int s) {
        const size_t off = (c0 + warp + kk * W) * CHUNK;
        mbar_expect(&bars[warp][s], 2 * CHUNK);
        bulk(ring + s * 2 * CHUNK, k + off, CHUNK, &bars[warp][s]);
        bulk(ring + s * 2 * CHUNK + CHUNK, v + off, CHUNK, &bars[warp][s]);
    };
    if (lane == 0)
        for (int s = 0; s < S && s < (int)mine; ++s) issue(s, s);
    unsigned acc = 0;
    for (size_t kk = 0; kk < mine; ++kk) {
        const int s = int(kk % S);
        mbar_wait(&bars[warp][s], unsigned((kk / S) & 1));
        acc += reinterpret_cast<const unsigned*>(ring + s * 2 * CHUNK)[lane];
        __syncwarp();
        if (lane == 0 && kk + S < mine) issue(kk + S, s);
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

__global__ void k_ldg(const uint4* src, size_t n, unsigned* sink) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(src + i));
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) sink[0] = acc;
}

template <typename F>
void timeit(const char* name, size_t bytes, int ctas, F launch, uint8_t* flush, size_t flush_bytes) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    std::vector<float> ms;
    static const char* fm = getenv("FLUSH");
    static const bool no_flush = getenv("NOFLUSH") != nullptr || (fm && !strcmp(fm, "none"));
    static const bool read_flush = fm && !strcmp(fm, "read");
    for (int it = 0; it < 23; ++it) {
        if (!no_flush && read_flush)
            k_ldg<<<1184, 512>>>(reinterpret_cast<const uint4*>(flush), flush_bytes / 16, reinterpret_cast<unsigned*>(flush));
        else if (!no_flush)
            CK(cudaMemsetAsync(flush, it & 255, flush_bytes));
        CK(cudaEventRecord(a));
        launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float t;
        CK(cudaEventElapsedTime(&t, a, b));
        if (it >= 3) ms.push_back(t);
    }
    CK(cudaGetLastError());
    std::sort(ms.begin(), ms.end());
    printf("{\"flush\": \"%s\", \"variant\": \"%s\", \"ctas\": %d, \"mb\": %.1f, \"best_us\": %.2f, \"median_us\": %.2f, "
           "\"best_gbs\": %.1f, \"median_gbs\": %.1f}\n",
           no_flush ? "none" : (read_flush ? "read" : "write"), name, ctas, bytes / 1e6, ms[0] * 1e3, ms[ms.size() / 2] * 1e3, bytes / (ms[0] * 1e-3) / 1e9,
           bytes / (ms[ms.size() / 2] * 1e-3) / 1e9);
    fflush(stdout);
}

int main(int argc, char** argv) {
    std::vector<double> mbs;
    for (int i = 1; i < argc; ++i) mbs.push_back(atof(argv[i]));
    if (mbs.empty()) mbs = {134.2, 268.4, 536.9, 1073.7, 4295.0};
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t maxb = size_t(*std::max_element(mbs.begin(), mbs.end()) * 1e6) + (1 << 20);
    uint8_t* src;
    uint8_t* flush;
    unsigned* sink;
    const size_t flush_bytes = size_t(256) << 20;
    CK(cudaMalloc(&src, maxb));
    CK(cudaMalloc(&flush, flush_bytes));
    CK(cudaMalloc(&sink, 64));
    CK(cudaMemset(src, 1, maxb));
    constexpr int W = 4, S = 3, CH = 16384;
    const int smem = W * S * CH;
    CK(cudaFuncSetAttribute(k_bulk<W, S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    constexpr int W2 = 8, S2 = 3, CH2 = 8192;
    CK(cudaFuncSetAttribute(k_bulk<W2, S2, CH2>, cudaFuncAttributeMaxDynamicSharedMemorySize, W2 * S2 * CH2));
    constexpr int W3 = 3, S3 = 2, CH3 = 16384;
    CK(cudaFuncSetAttribute(k_bulk_kv<W3, S3, CH3>, cudaFuncAttributeMaxDynamicSharedMemorySize, W3 * S3 * 2 * CH3));
    CK(cudaFuncSetAttribute(k_bulk_kv<4, 3, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 3 * 2 * 8192));
    for (double mb : mbs) {
        const size_t bytes = size_t(mb * 1e6) / 16384 * 16384;
        // K and V halves of the same total bytes: the fp32 split kernel's two streams
        const size_t half = bytes / 2 / 16384 * 16384;
        const uint8_t* vsrc = src + (maxb / 2) / (size_t(2) << 20) * (size_t(2) << 20);  // a 2 MB-aligned second array
        if (vsrc + half <= src + maxb) {
            timeit("bulk_kv_w3_s2_16k", 2 * half, sms,
                   [&] { k_bulk_kv<W3, S3, CH3><<<sms, W3 * 32, W3 * S3 * 2 * CH3>>>(src, vsrc, half, sink); }, flush,
                   flush_bytes);
            timeit("bulk_kv_w4_s3_8k", 2 * half, sms,
                   [&] { k_bulk_kv<4, 3, 8192><<<sms, 4 * 32, 4 * 3 * 2 * 8192>>>(src, vsrc, half, sink); }, flush,
                   flush_bytes);
        }
        timeit("bulk_w4_s3_16k", bytes, sms, [&] { k_bulk<W, S, CH><<<sms, W * 32, smem>>>(src, bytes, sink); },
               flush, flush_bytes);
        timeit("bulk_w8_s3_8k", bytes, sms,
               [&] { k_bulk<W2, S2, CH2><<<sms, W2 * 32, W2 * S2 * CH2>>>(src, bytes, sink); }, flush, flush_bytes);
        timeit("bulk_w4_s3_16k_2cta", bytes, 2 * sms,
               [&] { k_bulk<W, S, CH><<<2 * sms, W * 32, smem>>>(src, bytes, sink); }, flush, flush_bytes);
        timeit("ldg_v4", bytes, sms * 8,
               [&] { k_ldg<<<sms * 8, 512>>>(reinterpret_cast<const uint4*>(src), bytes / 16, sink); }, flush,
               flush_bytes);
    }
    return 0;
}
