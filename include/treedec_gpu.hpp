// treedec_gpu.hpp -- header-only C++ drop-in over the B200 C-ABI with the
// reference's own decode signatures and types.
//
// Include it from code that builds against the reference library
// (namespace treedec, /root/reference/proj/core/include) and link
// libtreedec_b200.so. treedec::gpu::tree_decode / ring_decode take exactly the
// arguments of treedec::tree_decode / ring_decode (decode.hpp:70-78) and
// return a treedec::DecodeResult; status codes come back as the reference's
// exception types (invalid_argument / domain_error / runtime_error).
//
// In one process the p workers of the ShardedKVCache run on one GPU, each
// worker's chunk placed in HBM and reduced with the split-KV kernel
// (td_local_partial); the max-allreduce / rescale / sum-allreduce / divide
// of the p partials is the single-device combine kernel
// (td_combine_partials). Across GPUs the same call sequence runs one
// process per GPU with td_comm_init + td_tree_decode.
//
// Inputs must be Float32 or Bf16 tensors (the GPU computes in fp32 on those
// grids); Float64 tensors raise invalid_argument. The output is stored
// through the input's dtype grid like the reference's (Tensor::store).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "treedec/attention.hpp"
#include "treedec/cluster.hpp"
#include "treedec/decode.hpp"
#include "treedec/reduce.hpp"
#include "treedec_b200.h"

namespace treedec::gpu {

namespace detail {

inline void check(int rc) {
    if (rc == TD_OK) return;
    const std::string msg = td_last_error();
    if (rc == TD_EINVAL) throw std::invalid_argument(msg);
    if (rc == TD_EDOMAIN) throw std::domain_error(msg);
    throw std::runtime_error(msg);
}

inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Tensor values on the bf16 grid are exact in bf16; on the f32 grid, in float.
inline std::vector<std::uint16_t> to_bf16(std::span<const double> x) {
    std::vector<std::uint16_t> out(x.size());
    for (std::size_t i = 0; i < x.size(); ++i) {
        const float f = static_cast<float>(x[i]);
        std::uint32_t u;
        std::memcpy(&u, &f, 4);
        out[i] = static_cast<std::uint16_t>(u >> 16);
    }
    return out;
}
inline std::vector<float> to_f32(std::span<const double> x) {
    return std::vector<float>(x.begin(), x.end());
}

struct Context {
    td_context* h = nullptr;
    explicit Context(int device = 0) { check(td_create(device, &h)); }
    ~Context() { td_destroy(h); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
};

template <typename T>
struct DeviceArray {
    T* p = nullptr;
    explicit DeviceArray(std::size_t n) { cuda(cudaMalloc(&p, sizeof(T) * (n ? n : 1)), "cudaMalloc"); }
    ~DeviceArray() { cudaFree(p); }
};

inline int code_of(DType dt) {
    switch (dt) {
    case DType::Float32: return TD_F32;
    case DType::Bf16: return TD_BF16;
    default: throw std::invalid_argument("treedec::gpu: Float64 tensors are not computed on the GPU path");
    }
}

// Places worker w's chunk (k/v [b, n_h, t, d]) and returns its fp32 partial.
inline void chunk_partial(Context& ctx, const Tensor& q, const Tensor& k, const Tensor& v,
                          std::int64_t seq_len, std::int64_t start, double scale, float* rm,
                          float* lse, float* out_dev) {
    const int dt = code_of(q.dtype());
    const std::int64_t b = k.extent(0), n_kv = k.extent(1), t = k.extent(2), d = k.extent(3);
    const std::int64_t n_q = q.extent(1);
    if (dt == TD_BF16) {
        const auto kb = to_bf16(k.data()), vb = to_bf16(v.data()), qb = to_bf16(q.data());
        check(td_kv_place(ctx.h, dt, b, n_kv, seq_len, d, start, t, kb.data(), vb.data(), 1));
        std::vector<float> hrm(b * n_q), hl(b * n_q), ho(b * n_q * d);
        check(td_local_partial(ctx.h, qb.data(), n_q, scale, hrm.data(), hl.data(), ho.data(), TD_HOST_IO));
        cuda(cudaMemcpy(rm, hrm.data(), hrm.size() * 4, cudaMemcpyHostToDevice), "copy");
        cuda(cudaMemcpy(lse, hl.data(), hl.size() * 4, cudaMemcpyHostToDevice), "copy");
        cuda(cudaMemcpy(out_dev, ho.data(), ho.size() * 4, cudaMemcpyHostToDevice), "copy");
    } else {
        const auto kf = to_f32(k.data()), vf = to_f32(v.data()), qf = to_f32(q.data());
        check(td_kv_place(ctx.h, dt, b, n_kv, seq_len, d, start, t, kf.data(), vf.data(), 1));
        std::vector<float> hrm(b * n_q), hl(b * n_q), ho(b * n_q * d);
        check(td_local_partial(ctx.h, qf.data(), n_q, scale, hrm.data(), hl.data(), ho.data(), TD_HOST_IO));
        cuda(cudaMemcpy(rm, hrm.data(), hrm.size() * 4, cudaMemcpyHostToDevice), "copy");
        cuda(cudaMemcpy(lse, hl.data(), hl.size() * 4, cudaMemcpyHostToDevice), "copy");
        cuda(cudaMemcpy(out_dev, ho.data(), ho.size() * 4, cudaMemcpyHostToDevice), "copy");
    }
}

inline void require(const Tensor& q, const ShardedKVCache& cache, const Topology& topo, const char* what) {
    if (q.rank() != 4 || q.extent(2) != 1)
        throw std::invalid_argument(std::string(what) + ": single query row required");
    if (cache.workers() == 0) throw std::invalid_argument(std::string(what) + ": empty cache");
    if (cache.workers() != topo.world_size())
        throw std::invalid_argument(std::string(what) + ": cache/topology worker count mismatch");
}

}  // namespace detail

// treedec::tree_decode (decode.hpp:70-72) on the GPU.
inline DecodeResult tree_decode(const Tensor& q, const ShardedKVCache& cache, const Topology& topo,
                                ReduceStrategy allreduce_strategy = ReduceStrategy::Hierarchical,
                                double scale = 1.0, bool /*parallel_workers*/ = false) {
    detail::require(q, cache, topo, "tree_decode");
    const int p = cache.workers();
    const std::int64_t b = q.extent(0), n_h = q.extent(1), d_h = q.extent(3), rows = b * n_h;
    detail::Context ctx(0);
    detail::DeviceArray<float> rm(std::size_t(p) * rows), lse(std::size_t(p) * rows),
        out(std::size_t(p) * rows * d_h), res(std::size_t(rows) * d_h);
    std::int64_t start = 0;
    for (int w = 0; w < p; ++w) {
        const Tensor& k = cache.k_chunks[std::size_t(w)];
        detail::chunk_partial(ctx, q, k, cache.v_chunks[std::size_t(w)], cache.seq_len, start, scale,
                              rm.p + w * rows, lse.p + w * rows, out.p + w * rows * d_h);
        start += k.extent(2);
    }
    detail::check(td_combine_partials(p, lse.p, out.p, rows, d_h, res.p, nullptr));
    std::vector<float> host(std::size_t(rows) * d_h);
    detail::cuda(cudaMemcpy(host.data(), res.p, host.size() * 4, cudaMemcpyDeviceToHost), "copy");
    DecodeResult r;
    r.output = Tensor({b, n_h, 1, d_h}, std::vector<double>(host.begin(), host.end()), q.dtype());
    const ReductionSchedule s = allreduce_schedule(allreduce_strategy, topo.nodes, topo.gpus_per_node);
    const CollectiveRounds cr{s.reduce_rounds, static_cast<int>(s.rounds.size()) - s.reduce_rounds};
    r.collectives = {cr, cr};
    r.cost.elems_sent_intra = comm_volume_formula_seq(DecodeAlgo::Tree, b, cache.seq_len, n_h * d_h, n_h, p);
    r.cost.rounds = 2 * s.rounds.size();
    r.cost.peak_elems_per_worker =
        peak_memory_formula(DecodeAlgo::Tree, b, (cache.seq_len + p - 1) / p, n_h * d_h, n_h);
    const OverlapFeasibility of = overlap_feasibility(topo, b, (cache.seq_len + p - 1) / p, n_h * d_h);
    r.overlap_feasible = of.feasible;
    r.overlap_ratio = of.ratio;
    return r;
}

// treedec::ring_decode (decode.hpp:77-78) on the GPU: worker 0's fold order.
inline DecodeResult ring_decode(const Tensor& q, const ShardedKVCache& cache, const Topology& topo,
                                double scale = 1.0, bool /*parallel_workers*/ = false) {
    detail::require(q, cache, topo, "ring_decode");
    const int p = cache.workers();
    const std::int64_t b = q.extent(0), n_h = q.extent(1), d_h = q.extent(3), rows = b * n_h;
    detail::Context ctx(0);
    detail::DeviceArray<float> rm(std::size_t(p) * rows), lse(std::size_t(p) * rows),
        out(std::size_t(p) * rows * d_h);
    std::int64_t start = 0;
    for (int w = 0; w < p; ++w) {
        const Tensor& k = cache.k_chunks[std::size_t(w)];
        detail::chunk_partial(ctx, q, k, cache.v_chunks[std::size_t(w)], cache.seq_len, start, scale,
                              rm.p + w * rows, lse.p + w * rows, out.p + w * rows * d_h);
        start += k.extent(2);
    }
    for (int r = 0; r + 1 < p; ++r) {  // root = parts[0]; fold parts[(p-1-r) mod p]
        const int inc = ((p - 1 - r) % p + p) % p;
        detail::check(td_combine_pair(rm.p, lse.p, out.p, rm.p + inc * rows, lse.p + inc * rows,
                                      out.p + inc * rows * d_h, rows, d_h, nullptr));
    }
    std::vector<float> host(std::size_t(rows) * d_h);
    detail::cuda(cudaMemcpy(host.data(), out.p, host.size() * 4, cudaMemcpyDeviceToHost), "copy");
    DecodeResult r;
    r.output = Tensor({b, n_h, 1, d_h}, std::vector<double>(host.begin(), host.end()), q.dtype());
    r.cost.rounds = static_cast<std::uint64_t>(p - 1);
    r.cost.elems_sent_intra =
        p > 1 ? comm_volume_formula_seq(DecodeAlgo::Ring, b, cache.seq_len, n_h * d_h, n_h, p) : 0.0;
    r.cost.peak_elems_per_worker =
        p > 1 ? peak_memory_formula(DecodeAlgo::Ring, b, (cache.seq_len + p - 1) / p, n_h * d_h, n_h)
              : static_cast<std::uint64_t>(2 * b * cache.seq_len * n_h * d_h + 2 * b * n_h * d_h);
    const OverlapFeasibility of = overlap_feasibility(topo, b, (cache.seq_len + p - 1) / p, n_h * d_h);
    r.overlap_feasible = of.feasible;
    r.overlap_ratio = of.ratio;
    return r;
}

}  // namespace treedec::gpu
