// How long after a kernel's last warp ends does its programmatic dependent get past
// griddepcontrol.wait, when that kernel stored into a peer GPU's memory (NVLink,
// cudaDeviceEnablePeerAccess), read from it, or touched only local memory?
// (the exchange kernel K2x -> next K1 gap of DESIGN.md §4).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/pdl_release_probe.cu -o scripts/_bin/pdl_release_probe
//   CUDA_VISIBLE_DEVICES=0,1 scripts/_bin/pdl_release_probe
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// mode 0: store into dst (local), 1: store into dst (peer), 2: load from src (peer)
__global__ void k_a(float* dst, const float* src, int n, int mode, unsigned long long* st) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float acc = 0.f;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (mode == 2)
            acc += *reinterpret_cast<const volatile float*>(src + i);
        else
            dst[i] = float(i);
    }
    if (acc == 12345.f) dst[0] = acc;
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(st, gt());
}

__global__ void k_b(unsigned long long* st) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) atomicMin(st + 1, gt());
}

int main() {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (ndev < 2) {
        printf("{\"error\": \"needs 2 GPUs\"}\n");
        return 0;
    }
    CK(cudaSetDevice(1));
    float* peer;
    const int n = 32 * 129 * 2;  // one rank's exchange payload (32 rows x 129 LL words)
    CK(cudaMalloc(&peer, n * sizeof(float)));
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    float* local;
    unsigned long long* st;
    CK(cudaMalloc(&local, n * sizeof(float)));
    CK(cudaMalloc(&st, 2 * sizeof(unsigned long long)));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    const char* names[3] = {"store_local", "store_peer", "load_peer"};
    for (int mode = 0; mode < 3; ++mode) {
        std::vector<double> gaps;
        for (int it = 0; it < 200; ++it) {
            unsigned long long init[2] = {0ull, ~0ull};
            CK(cudaMemcpyAsync(st, init, sizeof(init), cudaMemcpyHostToDevice, s));
            cudaLaunchConfig_t ca{};
            ca.gridDim = dim3(128);
            ca.blockDim = dim3(256);
            ca.stream = s;
            ca.attrs = attr;
            ca.numAttrs = 1;
            float* dst = mode == 1 ? peer : local;
            CK(cudaLaunchKernelEx(&ca, k_a, dst, (const float*)peer, n, mode, st));
            cudaLaunchConfig_t cb = ca;
            cb.gridDim = dim3(148);
            cb.blockDim = dim3(128);
            CK(cudaLaunchKernelEx(&cb, k_b, st));
            unsigned long long h[2];
            CK(cudaMemcpyAsync(h, st, sizeof(h), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (it >= 20) gaps.push_back((double(h[1]) - double(h[0])) * 1e-3);
        }
        std::sort(gaps.begin(), gaps.end());
        printf("{\"mode\": \"%s\", \"median_us\": %.2f, \"p10_us\": %.2f, \"p90_us\": %.2f}\n", names[mode],
               gaps[gaps.size() / 2], gaps[gaps.size() / 10], gaps[gaps.size() * 9 / 10]);
    }
    return 0;
}
