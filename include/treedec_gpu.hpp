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
// tree_decode runs the p workers of the ShardedKVCache as a td_group: worker w
// is a context on GPU w * ndev / p of the visible GPUs (contiguous placement,
// cluster.hpp:18-24; several workers share a GPU when p exceeds the GPU
// count), its chunk placed in that GPU's HBM, and every worker runs the
// split-KV kernel and the one-shot exchange combine (allreduce(max) / rescale
// / allreduce(sum) / divide, decode.cpp:129-173) with its peers addressed as
// device pointers. The group is created once per worker count and reused
// (calls are serialised by a mutex, so the functions stay callable from any
// thread like the reference's). ring_decode folds the per-worker partials
// with combine_pair in the reference order on one cached context. Across
// processes the same kernels run one process per GPU with td_comm_init +
// td_tree_decode.
//
// Inputs must be Float32 or Bf16 tensors (the GPU computes in fp32 on those
// grids); Float64 tensors raise invalid_argument. The output is stored
// through the input's dtype grid like the reference's (Tensor::store).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "treedec/attention.hpp"
#include "treedec/cluster.hpp"
#include "treedec/decode.hpp"
#include "treedec/energy.hpp"
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
    DeviceArray(DeviceArray&& o) noexcept : p(o.p) { o.p = nullptr; }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
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
inline void chunk_partial(td_context* ctx, const Tensor& q, const Tensor& k, const Tensor& v,
                          std::int64_t seq_len, std::int64_t start, double scale, float* rm,
                          float* lse, float* out_dev) {
    const int dt = code_of(q.dtype());
    const std::int64_t b = k.extent(0), n_kv = k.extent(1), t = k.extent(2), d = k.extent(3);
    const std::int64_t n_q = q.extent(1);
    if (dt == TD_BF16) {
        const auto kb = to_bf16(k.data()), vb = to_bf16(v.data()), qb = to_bf16(q.data());
        check(td_kv_place(ctx, dt, b, n_kv, seq_len, d, start, t, kb.data(), vb.data(), 1));
        std::vector<float> hrm(b * n_q), hl(b * n_q), ho(b * n_q * d);
        check(td_local_partial(ctx, qb.data(), n_q, scale, hrm.data(), hl.data(), ho.data(), TD_HOST_IO));
        cuda(cudaMemcpy(rm, hrm.data(), hrm.size() * 4, cudaMemcpyHostToDevice), "copy");
        cuda(cudaMemcpy(lse, hl.data(), hl.size() * 4, cudaMemcpyHostToDevice), "copy");
        cuda(cudaMemcpy(out_dev, ho.data(), ho.size() * 4, cudaMemcpyHostToDevice), "copy");
    } else {
        const auto kf = to_f32(k.data()), vf = to_f32(v.data()), qf = to_f32(q.data());
        check(td_kv_place(ctx, dt, b, n_kv, seq_len, d, start, t, kf.data(), vf.data(), 1));
        std::vector<float> hrm(b * n_q), hl(b * n_q), ho(b * n_q * d);
        check(td_local_partial(ctx, qf.data(), n_q, scale, hrm.data(), hl.data(), ho.data(), TD_HOST_IO));
        cuda(cudaMemcpy(rm, hrm.data(), hrm.size() * 4, cudaMemcpyHostToDevice), "copy");
        cuda(cudaMemcpy(lse, hl.data(), hl.size() * 4, cudaMemcpyHostToDevice), "copy");
        cuda(cudaMemcpy(out_dev, ho.data(), ho.size() * 4, cudaMemcpyHostToDevice), "copy");
    }
}

// The process-wide worker group of tree_decode (re-created when the worker
// count changes) and the single context of ring_decode. Never destroyed: the
// CUDA runtime may already be torn down when static destructors run.
struct Cached {
    std::mutex mu;
    td_group* group = nullptr;
    int workers = 0;
    std::int64_t x_rows = 0, x_d = 0;
    td_context* ring = nullptr;
};
inline Cached& cached() {
    static Cached* c = new Cached;
    return *c;
}

inline td_group* group_for(Cached& c, int p) {
    if (c.group && c.workers == p) return c.group;
    if (c.group) td_group_destroy(c.group);
    c.group = nullptr;
    c.workers = 0;
    c.x_rows = c.x_d = 0;
    int n = 0;
    cuda(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    if (n < 1) throw std::runtime_error("treedec::gpu: no CUDA device");
    std::vector<int> devs(static_cast<std::size_t>(std::min(n, p)));
    for (std::size_t i = 0; i < devs.size(); ++i) devs[i] = static_cast<int>(i);
    check(td_group_create(static_cast<int>(devs.size()), devs.data(), p, &c.group));
    c.workers = p;
    return c.group;
}

// Worker w's chunk of the cache into its context's HBM (host upload).
inline void place_chunk(td_context* ctx, const Tensor& k, const Tensor& v, std::int64_t seq_len, std::int64_t start) {
    const int dt = code_of(k.dtype());
    const std::int64_t b = k.extent(0), n_kv = k.extent(1), t = k.extent(2), d = k.extent(3);
    if (dt == TD_BF16) {
        const auto kb = to_bf16(k.data()), vb = to_bf16(v.data());
        check(td_kv_place(ctx, dt, b, n_kv, seq_len, d, start, t, kb.data(), vb.data(), 1));
    } else {
        const auto kf = to_f32(k.data()), vf = to_f32(v.data());
        check(td_kv_place(ctx, dt, b, n_kv, seq_len, d, start, t, kf.data(), vf.data(), 1));
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
    const int dt = detail::code_of(q.dtype());
    std::vector<float> host(std::size_t(rows) * d_h);
    {
        detail::Cached& c = detail::cached();
        std::lock_guard<std::mutex> lock(c.mu);
        td_group* g = detail::group_for(c, p);
        std::int64_t start = 0;
        for (int w = 0; w < p; ++w) {
            td_context* ctx = nullptr;
            detail::check(td_group_context(g, w, &ctx));
            const Tensor& k = cache.k_chunks[std::size_t(w)];
            detail::place_chunk(ctx, k, cache.v_chunks[std::size_t(w)], cache.seq_len, start);
            start += k.extent(2);
        }
        if (c.x_rows < rows || c.x_d != d_h) {
            detail::check(td_group_p2p_open(g, rows, d_h));
            c.x_rows = rows;
            c.x_d = d_h;
        }
        const int strategy = static_cast<int>(allreduce_strategy);
        if (dt == TD_BF16) {
            const auto qb = detail::to_bf16(q.data());
            detail::check(td_group_tree_decode(g, qb.data(), n_h, scale, strategy, host.data(), TD_HOST_IO));
        } else {
            const auto qf = detail::to_f32(q.data());
            detail::check(td_group_tree_decode(g, qf.data(), n_h, scale, strategy, host.data(), TD_HOST_IO));
        }
    }
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
    std::vector<float> host(std::size_t(rows) * d_h);
    {
        detail::Cached& c = detail::cached();
        std::lock_guard<std::mutex> lock(c.mu);
        if (!c.ring) detail::check(td_create(0, &c.ring));
        detail::cuda(cudaSetDevice(0), "cudaSetDevice");
        detail::DeviceArray<float> rm(std::size_t(p) * rows), lse(std::size_t(p) * rows),
            out(std::size_t(p) * rows * d_h);
        std::int64_t start = 0;
        for (int w = 0; w < p; ++w) {
            const Tensor& k = cache.k_chunks[std::size_t(w)];
            detail::chunk_partial(c.ring, q, k, cache.v_chunks[std::size_t(w)], cache.seq_len, start, scale,
                                  rm.p + w * rows, lse.p + w * rows, out.p + w * rows * d_h);
            start += k.extent(2);
        }
        for (int r = 0; r + 1 < p; ++r) {  // root = parts[0]; fold parts[(p-1-r) mod p]
            const int inc = ((p - 1 - r) % p + p) % p;
            detail::check(td_combine_pair(rm.p, lse.p, out.p, rm.p + inc * rows, lse.p + inc * rows,
                                          out.p + inc * rows * d_h, rows, d_h, nullptr));
        }
        detail::cuda(cudaMemcpy(host.data(), out.p, host.size() * 4, cudaMemcpyDeviceToHost), "copy");
    }
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

namespace detail {

// A [b, h, n, d] tensor (or its key rows [k0, k1)) on the device, in its dtype.
inline DeviceArray<std::uint8_t> upload(const Tensor& t, std::int64_t k0 = 0, std::int64_t k1 = -1) {
    const int dt = code_of(t.dtype());
    const std::int64_t b = t.extent(0), h = t.extent(1), n = t.extent(2), d = t.extent(3);
    if (k1 < 0) k1 = n;
    const std::int64_t len = k1 - k0;
    std::vector<double> rows;
    rows.reserve(std::size_t(b * h * len * d));
    for (std::int64_t ib = 0; ib < b; ++ib)
        for (std::int64_t ih = 0; ih < h; ++ih) {
            const std::int64_t o = t.offset4(ib, ih, k0, 0);
            rows.insert(rows.end(), t.data().begin() + o, t.data().begin() + o + len * d);
        }
    const std::size_t esz = dt == TD_BF16 ? 2 : 4;
    DeviceArray<std::uint8_t> dev(rows.size() * esz);
    if (dt == TD_BF16) {
        const auto x = to_bf16(rows);
        cuda(cudaMemcpy(dev.p, x.data(), x.size() * 2, cudaMemcpyHostToDevice), "copy");
    } else {
        const auto x = to_f32(rows);
        cuda(cudaMemcpy(dev.p, x.data(), x.size() * 4, cudaMemcpyHostToDevice), "copy");
    }
    return dev;
}

inline void require_energy(const Tensor& q, const Tensor& k, const Tensor& v, const Tensor& source,
                           const char* what) {
    if (q.rank() != 4 || k.rank() != 4 || v.rank() != 4)
        throw std::invalid_argument(std::string(what) + ": rank-4 tensors required");
    if (k.extent(0) != q.extent(0) || k.extent(1) != q.extent(1) || k.extent(3) != q.extent(3))
        throw std::invalid_argument(std::string(what) + ": q/k shape mismatch");
    if (!v.same_shape(k)) throw std::invalid_argument(std::string(what) + ": k/v shape mismatch");
    if (!source.empty() && !source.same_shape(q))
        throw std::invalid_argument(std::string(what) + ": source must have the query shape");
}

// Per-chunk fp32 partials (row_max, lse, out) of q.k + source.v, keys split by chunk_extents.
inline void energy_chunks(const Tensor& q, const Tensor& k, const Tensor& v, const Tensor& source, int chunks,
                          DeviceArray<float>& rm, DeviceArray<float>& lse, DeviceArray<float>& out) {
    const int dt = code_of(q.dtype());
    const std::int64_t b = q.extent(0), h = q.extent(1), nq = q.extent(2), d = q.extent(3), n = k.extent(2);
    const std::int64_t rows = b * h * nq;
    const auto qd = upload(q);
    const bool with_source = !source.empty();
    DeviceArray<std::uint8_t> sdev = with_source ? upload(source) : DeviceArray<std::uint8_t>(1);
    const std::vector<std::int64_t> ext = chunk_extents(n, chunks);
    std::int64_t k0 = 0;
    for (int c = 0; c < chunks; ++c) {
        const std::int64_t t = ext[std::size_t(c)];
        const auto kd = upload(k, k0, k0 + t), vd = upload(v, k0, k0 + t);
        std::size_t ws = 0;
        check(td_energy_workspace_bytes(dt, b, h, nq, t, d, &ws));
        DeviceArray<std::uint8_t> work(ws);
        check(td_energy_partial(dt, qd.p, with_source ? sdev.p : nullptr, kd.p, vd.p, b, h, nq, t, d,
                                rm.p + c * rows, lse.p + c * rows, out.p + c * rows * d, work.p, ws, nullptr));
        k0 += t;
    }
    cuda(cudaDeviceSynchronize(), "energy");
}

inline Tensor download(const float* dev, std::vector<std::int64_t> shape, DType dt) {
    std::int64_t n = 1;
    for (auto e : shape) n *= e;
    std::vector<float> host(static_cast<std::size_t>(n));
    cuda(cudaMemcpy(host.data(), dev, host.size() * 4, cudaMemcpyDeviceToHost), "copy");
    return Tensor(std::move(shape), std::vector<double>(host.begin(), host.end()), dt);
}

}  // namespace detail

// treedec::energy_forward_parallel (energy.hpp:47-52, energy.cpp:152-203) on the GPU.
inline EnergyEval energy_forward_parallel(const Tensor& q, const Tensor& k, const Tensor& v, const Tensor& source,
                                          int chunks) {
    detail::require_energy(q, k, v, source, "energy_forward_parallel");
    if (chunks < 1 || chunks > k.extent(2))
        throw std::invalid_argument("energy_forward_parallel: need 1 <= chunks <= N");
    const std::int64_t b = q.extent(0), h = q.extent(1), nq = q.extent(2), d = q.extent(3), rows = b * h * nq;
    detail::DeviceArray<float> rm(std::size_t(chunks) * rows), lse(std::size_t(chunks) * rows),
        out(std::size_t(chunks) * rows * d), value(rows), rmax(rows), shifted(rows);
    detail::energy_chunks(q, k, v, source, chunks, rm, lse, out);
    detail::check(td_energy_combine(chunks, rm.p, lse.p, rows, value.p, rmax.p, shifted.p, nullptr));
    const DType sdt = stats_dtype(q.dtype());
    return EnergyEval{detail::download(value.p, {b, h, nq}, sdt), detail::download(rmax.p, {b, h, nq}, sdt),
                      detail::download(shifted.p, {b, h, nq}, sdt)};
}

// treedec::energy_grad_parallel (energy.hpp:54-58, energy.cpp:205-259) on the GPU.
inline Tensor energy_grad_parallel(const Tensor& q, const Tensor& k, const Tensor& v, const EnergyEval& saved,
                                   int chunks) {
    detail::require_energy(q, k, v, Tensor{}, "energy_grad_parallel");
    if (chunks < 1 || chunks > k.extent(2))
        throw std::invalid_argument("energy_grad_parallel: need 1 <= chunks <= N");
    const std::int64_t b = q.extent(0), h = q.extent(1), nq = q.extent(2), d = q.extent(3), rows = b * h * nq;
    const std::vector<std::int64_t> expected{b, h, nq};
    if (saved.value.shape() != expected || saved.row_max.shape() != expected ||
        saved.shifted_lse.shape() != expected)
        throw std::invalid_argument("energy_grad_parallel: saved evaluation does not match inputs");
    detail::DeviceArray<float> rm(std::size_t(chunks) * rows), lse(std::size_t(chunks) * rows),
        out(std::size_t(chunks) * rows * d), srm(rows), ssh(rows), grad(rows * d);
    detail::energy_chunks(q, k, v, Tensor{}, chunks, rm, lse, out);
    const std::vector<float> hrm(saved.row_max.data().begin(), saved.row_max.data().end());
    const std::vector<float> hsh(saved.shifted_lse.data().begin(), saved.shifted_lse.data().end());
    detail::cuda(cudaMemcpy(srm.p, hrm.data(), hrm.size() * 4, cudaMemcpyHostToDevice), "copy");
    detail::cuda(cudaMemcpy(ssh.p, hsh.data(), hsh.size() * 4, cudaMemcpyHostToDevice), "copy");
    detail::check(td_energy_grad_combine(chunks, lse.p, out.p, srm.p, ssh.p, rows, d, grad.p, nullptr));
    return detail::download(grad.p, {b, h, nq, d}, q.dtype());
}

}  // namespace treedec::gpu
