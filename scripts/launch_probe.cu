// Floors of an isolated call (the e2e shape: 8 KB query in from pinned host
// memory, two dependent kernels, 16 KB out to pinned host memory, the host
// waits for it), with tiny kernels so only launch / copy / notification
// latency is left. Each mode runs 200 calls after 20 warm-ups and prints the
// median and p10 host wall time per call as one JSON line:
//
//   empty_sync     one empty kernel + cudaStreamSynchronize
//   empty_spin     one kernel that writes a pinned completion word; the host spins on it
//   chain_stream   H2D q, k1 (148 CTAs x 128 threads), k2 (writes out to pinned memory
//                  + the completion word), spin; three stream operations per call
//   chain_pdl      the same with k2 a programmatic dependent of k1
//   chain_graph    the same three operations replayed as one CUDA graph (per-call
//                  kernel parameter update of the completion epoch)
//   chain_graph_pdl  graph captured from the PDL stream chain (programmatic edge)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o scripts/_bin/launch_probe scripts/launch_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                              \
        }                                                                              \
    } while (0)

__global__ void k_empty() {}

__global__ void k_flag(volatile unsigned* flag, unsigned epoch) {
    if (threadIdx.x == 0) {
        __threadfence_system();
        *flag = epoch;
    }
}

// k1: every CTA reads q (8 KB) and writes a partial per CTA
__global__ void k1(const float4* q, float4* part) {
    asm volatile("griddepcontrol.launch_dependents;");
    float4 a = q[threadIdx.x % 512];
    part[blockIdx.x * blockDim.x + threadIdx.x] = a;
}

// k2: one CTA sums a column of the partials into out (pinned host) and signals
__global__ void k2(const float4* part, float4* out, volatile unsigned* flag, unsigned epoch, int nparts) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    float4 s = make_float4(0, 0, 0, 0);
    for (int i = 0; i < nparts; i += 16) {
        float4 a = part[i * blockDim.x + threadIdx.x];
        s.x += a.x;
    }
    out[threadIdx.x] = s;  // 16 KB = 1024 float4: 4 per thread over 256 threads
    out[threadIdx.x + 256] = s;
    out[threadIdx.x + 512] = s;
    out[threadIdx.x + 768] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        *flag = epoch;
    }
}

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static void report(const char* name, std::vector<double>& t) {
    std::sort(t.begin(), t.end());
    std::printf("{\"mode\": \"%s\", \"median_us\": %.2f, \"p10_us\": %.2f, \"p90_us\": %.2f}\n", name, t[t.size() / 2],
                t[t.size() / 10], t[t.size() * 9 / 10]);
    std::fflush(stdout);
}

int main() {
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    unsigned* flag_h;
    CK(cudaHostAlloc(&flag_h, 64, cudaHostAllocMapped));
    unsigned* flag_d;
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&flag_d), flag_h, 0));
    float4 *q_h, *out_h, *out_d;
    CK(cudaHostAlloc(&q_h, 8192, cudaHostAllocDefault));
    CK(cudaHostAlloc(&out_h, 16384, cudaHostAllocMapped));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&out_d), out_h, 0));
    float4 *q_d, *part;
    CK(cudaMalloc(&q_d, 8192));
    const int ctas = 148, thr = 128;
    CK(cudaMalloc(&part, size_t(ctas) * thr * 16));
    const int N = 200, W = 20;
    unsigned epoch = 0;
    auto spin = [&](unsigned e) {
        while (*reinterpret_cast<volatile unsigned*>(flag_h) != e) {
        }
    };
    std::vector<double> t;

    t.clear();
    for (int i = 0; i < N + W; ++i) {
        double t0 = now_us();
        k_empty<<<1, 32, 0, st>>>();
        CK(cudaStreamSynchronize(st));
        if (i >= W) t.push_back(now_us() - t0);
    }
    report("empty_sync", t);

    t.clear();
    for (int i = 0; i < N + W; ++i) {
        double t0 = now_us();
        k_flag<<<1, 32, 0, st>>>(flag_d, ++epoch);
        spin(epoch);
        if (i >= W) t.push_back(now_us() - t0);
    }
    report("empty_spin", t);
    CK(cudaStreamSynchronize(st));

    auto chain = [&](bool pdl, unsigned e) {
        CK(cudaMemcpyAsync(q_d, q_h, 8192, cudaMemcpyHostToDevice, st));
        k1<<<ctas, thr, 0, st>>>(q_d, part);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = pdl ? 1 : 0;
        CK(cudaLaunchKernelEx(&cfg, k2, (const float4*)part, out_d, (volatile unsigned*)flag_d, e, ctas * thr / thr));
    };
    for (int pdl = 0; pdl < 2; ++pdl) {
        t.clear();
        for (int i = 0; i < N + W; ++i) {
            double t0 = now_us();
            chain(pdl, ++epoch);
            spin(epoch);
            if (i >= W) t.push_back(now_us() - t0);
        }
        report(pdl ? "chain_pdl" : "chain_stream", t);
        CK(cudaStreamSynchronize(st));
    }

    for (int pdl = 0; pdl < 2; ++pdl) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        chain(pdl, 0);
        CK(cudaStreamEndCapture(st, &g));
        cudaGraphExec_t ex;
        CK(cudaGraphInstantiate(&ex, g, 0));
        size_t n = 0;
        CK(cudaGraphGetNodes(g, nullptr, &n));
        std::vector<cudaGraphNode_t> nodes(n);
        CK(cudaGraphGetNodes(g, nodes.data(), &n));
        cudaGraphNode_t k2n = nullptr;
        cudaKernelNodeParams kp = {};
        for (auto nd : nodes) {
            cudaGraphNodeType ty;
            CK(cudaGraphNodeGetType(nd, &ty));
            if (ty != cudaGraphNodeTypeKernel) continue;
            cudaKernelNodeParams p;
            CK(cudaGraphKernelNodeGetParams(nd, &p));
            if (p.func == reinterpret_cast<void*>(k2)) {
                k2n = nd;
                kp = p;
            }
        }
        if (!k2n) {
            std::fprintf(stderr, "k2 node not found\n");
            return 1;
        }
        const float4* a0 = part;
        float4* a1 = out_d;
        volatile unsigned* a2 = flag_d;
        unsigned a3 = 0;
        int a4 = ctas;
        void* args[5] = {&a0, &a1, &a2, &a3, &a4};
        kp.kernelParams = args;
        t.clear();
        for (int i = 0; i < N + W; ++i) {
            double t0 = now_us();
            a3 = ++epoch;
            CK(cudaGraphExecKernelNodeSetParams(ex, k2n, &kp));
            CK(cudaGraphLaunch(ex, st));
            spin(epoch);
            if (i >= W) t.push_back(now_us() - t0);
        }
        report(pdl ? "chain_graph_pdl" : "chain_graph", t);
        CK(cudaStreamSynchronize(st));
        cudaGraphExecDestroy(ex);
        cudaGraphDestroy(g);
    }
    return 0;
}
