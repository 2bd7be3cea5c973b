// ref_shim.cpp -- C-ABI wrapper over the UNMODIFIED reference library
// (/root/reference/proj/core, compiled by path by oracle/Makefile into
// oracle/_ref/libtreedec_ref.so). TEST INFRASTRUCTURE ONLY: used by tests/ to
// pin the oracle restatement and by bench.py's cpu_baseline / --impl
// reference leg to time the reference's own tree_decode on host cores.
//
// The reference has no GQA (attention.cpp:22 demands equal q/k heads), so
// GQA inputs are run per (batch, q-head) with n_h = 1 against kv head
// h / group -- rows of tree_decode are independent, so this equals one call.
#include "treedec/attention.hpp"
#include "treedec/decode.hpp"
#include "treedec/energy.hpp"
#include "treedec/numerics.hpp"

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

using namespace treedec;

namespace {

thread_local std::string g_err;

DType to_dtype(int code) {
    switch (code) {
    case 1: return DType::Float32;
    case 2: return DType::Bf16;
    default: return DType::Float64;
    }
}

ReduceStrategy to_strategy(int code) {
    switch (code) {
    case 0: return ReduceStrategy::TreeBinary;
    case 1: return ReduceStrategy::Ring;
    default: return ReduceStrategy::Hierarchical;
    }
}

int fail(const std::exception& e, int code) {
    g_err = e.what();
    return code;
}

Tensor row_tensor(const double* base, std::int64_t rows, std::int64_t d, DType dt) {
    return Tensor({1, 1, rows, d}, std::vector<double>(base, base + rows * d), dt);
}

// A prepared per-(b, q-head) problem: tensors and shards built once, so the
// timed region holds only the decode call.
struct Prepared {
    std::vector<Tensor> q;
    std::vector<ShardedKVCache> caches; // one per (b, kv-head)
    std::vector<int> cache_of_row;
    Topology topo;
    int p = 1;
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

std::uint64_t ref_mix64(std::uint64_t seed, std::uint64_t counter) { return mix64(seed, counter); }

// Element `index` of seeded_random_tensor({index+1}, seed, scale, dtype).
int ref_seeded_values(std::uint64_t seed, double scale, int dtype, std::int64_t n, double* out) {
    try {
        const Tensor t = seeded_random_tensor({n}, seed, scale, to_dtype(dtype));
        std::memcpy(out, t.data().data(), sizeof(double) * static_cast<std::size_t>(n));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

double ref_round(double x, int dtype) { return round_to_dtype(x, to_dtype(dtype)); }

int ref_chunk_extents(std::int64_t n, int p, std::int64_t* out) {
    try {
        const auto ext = chunk_extents(n, p);
        for (int i = 0; i < p; ++i) out[i] = ext[static_cast<std::size_t>(i)];
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// attention_chunk_partial for MHA inputs q [b,h,1,d], k/v [b,h,t,d].
int ref_chunk_partial(const double* q, const double* k, const double* v, std::int64_t b,
                      std::int64_t h, std::int64_t t, std::int64_t d, double scale, int dtype,
                      double* row_max, double* lse, double* out) {
    try {
        const DType dt = to_dtype(dtype);
        const Tensor tq({b, h, 1, d}, std::vector<double>(q, q + b * h * d), dt);
        const Tensor tk({b, h, t, d}, std::vector<double>(k, k + b * h * t * d), dt);
        const Tensor tv({b, h, t, d}, std::vector<double>(v, v + b * h * t * d), dt);
        const SoftmaxPartial part = attention_chunk_partial(tq, tk, tv, scale);
        std::memcpy(row_max, part.row_max.data().data(), sizeof(double) * static_cast<std::size_t>(b * h));
        std::memcpy(lse, part.lse.data().data(), sizeof(double) * static_cast<std::size_t>(b * h));
        std::memcpy(out, part.out.data().data(), sizeof(double) * static_cast<std::size_t>(b * h * d));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// energy_forward_parallel (energy.cpp:152-203): q, src [b,h,nq,d] (src may be
// null: empty source), k, v [b,h,n,d]; value, row_max, shifted [b,h,nq].
int ref_energy_forward_parallel(const double* q, const double* k, const double* v, const double* src,
                                std::int64_t b, std::int64_t h, std::int64_t nq, std::int64_t n,
                                std::int64_t d, int chunks, int dtype, double* value, double* row_max,
                                double* shifted) {
    try {
        const DType dt = to_dtype(dtype);
        const Tensor tq({b, h, nq, d}, std::vector<double>(q, q + b * h * nq * d), dt);
        const Tensor tk({b, h, n, d}, std::vector<double>(k, k + b * h * n * d), dt);
        const Tensor tv({b, h, n, d}, std::vector<double>(v, v + b * h * n * d), dt);
        const Tensor ts = src ? Tensor({b, h, nq, d}, std::vector<double>(src, src + b * h * nq * d), dt) : Tensor{};
        const EnergyEval e = energy_forward_parallel(tq, tk, tv, ts, chunks);
        const std::size_t rows = static_cast<std::size_t>(b * h * nq);
        std::memcpy(value, e.value.data().data(), sizeof(double) * rows);
        std::memcpy(row_max, e.row_max.data().data(), sizeof(double) * rows);
        std::memcpy(shifted, e.shifted_lse.data().data(), sizeof(double) * rows);
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// energy_grad_parallel (energy.cpp:205-259) with saved (value, row_max, shifted).
int ref_energy_grad_parallel(const double* q, const double* k, const double* v, const double* value,
                             const double* row_max, const double* shifted, std::int64_t b, std::int64_t h,
                             std::int64_t nq, std::int64_t n, std::int64_t d, int chunks, int dtype,
                             double* grad) {
    try {
        const DType dt = to_dtype(dtype);
        const DType sdt = stats_dtype(dt);
        const Tensor tq({b, h, nq, d}, std::vector<double>(q, q + b * h * nq * d), dt);
        const Tensor tk({b, h, n, d}, std::vector<double>(k, k + b * h * n * d), dt);
        const Tensor tv({b, h, n, d}, std::vector<double>(v, v + b * h * n * d), dt);
        const std::size_t rows = static_cast<std::size_t>(b * h * nq);
        EnergyEval saved{Tensor::zeros({b, h, nq}, sdt), Tensor::zeros({b, h, nq}, sdt),
                         Tensor::zeros({b, h, nq}, sdt)};
        std::memcpy(saved.value.data().data(), value, sizeof(double) * rows);
        std::memcpy(saved.row_max.data().data(), row_max, sizeof(double) * rows);
        std::memcpy(saved.shifted_lse.data().data(), shifted, sizeof(double) * rows);
        const Tensor g = energy_grad_parallel(tq, tk, tv, saved, chunks);
        std::memcpy(grad, g.data().data(), sizeof(double) * rows * static_cast<std::size_t>(d));
        return 0;
    } catch (const std::exception& e) {
        return fail(e, -1);
    }
}

// combine_partials over P partials of shape rows x d (lse [P][rows], out [P][rows][d]).
int ref_combine_partials(int P, const double* lse, const double* out, std::int64_t rows,
                         std::int64_t d, int dtype, double* result) {
    try {
        const DType dt = to_dtype(dtype);
        const DType sdt = stats_dtype(dt);
        std::vector<SoftmaxPartial> parts;
        for (int p = 0; p < P; ++p) {
            const double* l = lse + p * rows;
            const double* o = out + p * rows * d;
            parts.push_back({Tensor({1, rows, 1}, std::vector<double>(l, l + rows), sdt),
                             Tensor({1, rows, 1}, std::vector<double>(l, l + rows), sdt),
                             Tensor({1, rows, 1, d}, std::vector<double>(o, o + rows * d), dt)});
        }
        const Tensor res = combine_partials(parts);
        std::memcpy(result, res.data().data(), sizeof(double) * static_cast<std::size_t>(rows * d));
        return 0;
    } catch (const std::invalid_argument& e) {
        return fail(e, -1);
    } catch (const std::exception& e) {
        return fail(e, -2);
    }
}

// Build the per-row problems. q [b, n_q, d], k/v [b, n_kv, seq, d].
void* ref_prepare(const double* q, const double* k, const double* v, std::int64_t b,
                  std::int64_t n_q, std::int64_t n_kv, std::int64_t seq, std::int64_t d, int p,
                  int dtype) {
    try {
        if (n_kv < 1 || n_q % n_kv != 0) throw std::invalid_argument("ref_prepare: bad GQA shape");
        const DType dt = to_dtype(dtype);
        auto* pr = new Prepared;
        pr->p = p;
        pr->topo = topology_for_workers(p);
        for (std::int64_t ib = 0; ib < b; ++ib)
            for (std::int64_t kh = 0; kh < n_kv; ++kh) {
                const double* kb = k + (ib * n_kv + kh) * seq * d;
                const double* vb = v + (ib * n_kv + kh) * seq * d;
                pr->caches.push_back(
                    shard_kv(row_tensor(kb, seq, d, dt), row_tensor(vb, seq, d, dt), p));
            }
        const std::int64_t group = n_q / n_kv;
        for (std::int64_t ib = 0; ib < b; ++ib)
            for (std::int64_t h = 0; h < n_q; ++h) {
                pr->q.push_back(row_tensor(q + (ib * n_q + h) * d, 1, d, dt));
                pr->cache_of_row.push_back(static_cast<int>(ib * n_kv + h / group));
            }
        return pr;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_release(void* handle) { delete static_cast<Prepared*>(handle); }

// Runs tree_decode (algo 0) or ring_decode (algo 1) over rows [row0, row1)
// of a prepared problem, writing out [rows][d]. Rows are spread over
// `nthreads` host threads (each row is an independent reference call; the
// reference functions are pure). *seconds = wall time of the decode calls
// alone. counters (optional, 4 doubles): elems_sent_total, wire_elems_total,
// peak_elems_per_worker, rounds -- of the first row's call.
int ref_decode(void* handle, int algo, int strategy, double scale, int parallel,
               std::int64_t row0, std::int64_t row1, int nthreads, double* out, double* seconds,
               double* counters) {
    auto* pr = static_cast<Prepared*>(handle);
    std::vector<std::string> errs(static_cast<std::size_t>(nthreads > 0 ? nthreads : 1));
    std::vector<int> codes(errs.size(), 0);
    auto work = [&](int tid, std::int64_t a, std::int64_t b) {
        try {
            for (std::int64_t r = a; r < b; ++r) {
                const Tensor& q = pr->q[static_cast<std::size_t>(r)];
                const ShardedKVCache& cache =
                    pr->caches[static_cast<std::size_t>(pr->cache_of_row[static_cast<std::size_t>(r)])];
                const DecodeResult res =
                    algo == 0 ? tree_decode(q, cache, pr->topo, to_strategy(strategy), scale, parallel != 0)
                              : ring_decode(q, cache, pr->topo, scale, parallel != 0);
                const std::int64_t d = q.extent(3);
                std::memcpy(out + (r - row0) * d, res.output.data().data(),
                            sizeof(double) * static_cast<std::size_t>(d));
                if (counters && r == row0) {
                    counters[0] = res.cost.elems_sent_total();
                    counters[1] = static_cast<double>(res.cost.wire_elems_total());
                    counters[2] = static_cast<double>(res.cost.peak_elems_per_worker);
                    counters[3] = static_cast<double>(res.cost.rounds);
                }
            }
        } catch (const std::invalid_argument& e) {
            errs[static_cast<std::size_t>(tid)] = e.what();
            codes[static_cast<std::size_t>(tid)] = -1;
        } catch (const std::exception& e) {
            errs[static_cast<std::size_t>(tid)] = e.what();
            codes[static_cast<std::size_t>(tid)] = -2;
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    const int nt = static_cast<int>(errs.size());
    if (nt == 1) {
        work(0, row0, row1);
    } else {
        std::vector<std::thread> pool;
        const std::int64_t n = row1 - row0;
        for (int i = 0; i < nt; ++i)
            pool.emplace_back(work, i, row0 + n * i / nt, row0 + n * (i + 1) / nt);
        for (auto& th : pool) th.join();
    }
    if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (std::size_t i = 0; i < errs.size(); ++i)
        if (codes[i] != 0) {
            g_err = errs[i];
            return codes[i];
        }
    return 0;
}

} // extern "C"
