// shim_parity.cpp -- the reference's decode test cases (test_decode.cpp:44-92,
// acceptance_main.cpp:154-187) replayed through treedec::gpu (include/
// treedec_gpu.hpp) against the reference's own treedec::tree_decode /
// ring_decode, using the reference's Tensor / ShardedKVCache / Topology types.
// Built by `make -C oracle shim` (links the reference library from oracle/_ref
// and libtreedec_b200.so); run by tests/test_gpu_shim.py on a GPU box.
#include "treedec_gpu.hpp"

#include "treedec/numerics.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

using namespace treedec;

namespace {

Tensor retag(const Tensor& t, DType dt) {
    return Tensor(t.shape(), std::vector<double>(t.data().begin(), t.data().end()), dt);
}

int failures = 0;
int checks = 0;

void expect(bool ok, const char* what, double err, double tol) {
    ++checks;
    if (!ok) {
        ++failures;
        std::printf("FAIL %s err=%.3e tol=%.3e\n", what, err, tol);
    }
}

}  // namespace

int main() {
    char what[256];
    const bool verbose = std::getenv("SHIM_VERBOSE") != nullptr;
    // exactness grid: f32 / bf16 grids, heads {1, 16}, d_h {8, 128}
    for (const DType dt : {DType::Float32, DType::Bf16})
        for (const std::int64_t n : {17LL, 64LL, 1024LL, 5000LL})
            for (const std::int64_t n_h : {1LL, 16LL})
                for (const std::int64_t d_h : {8LL, 128LL}) {
                    const std::uint64_t seed = 2 + static_cast<std::uint64_t>(n) + 131 * n_h + d_h;
                    const Tensor q = seeded_random_tensor({1, n_h, 1, d_h}, mix64(seed, 1), 1.0, dt);
                    const Tensor k = seeded_random_tensor({1, n_h, n, d_h}, mix64(seed, 2), 1.0, dt);
                    const Tensor v = seeded_random_tensor({1, n_h, n, d_h}, mix64(seed, 3), 1.0, dt);
                    for (const int p : {1, 2, 3, 4, 7, 8, 16}) {
                        if (p > n) continue;
                        const Topology topo = topology_for_workers(p);
                        const ShardedKVCache cache = shard_kv(k, v, p);
                        const ShardedKVCache cache64 = shard_kv(retag(k, DType::Float64), retag(v, DType::Float64), p);
                        const Tensor q64 = retag(q, DType::Float64);
                        for (const ReduceStrategy st :
                             {ReduceStrategy::TreeBinary, ReduceStrategy::Ring, ReduceStrategy::Hierarchical}) {
                            const DecodeResult want = tree_decode(q64, cache64, topo, st);
                            const DecodeResult ref = tree_decode(q, cache, topo, st);
                            if (verbose)
                                std::fprintf(stderr, "case tree dt=%s n=%lld h=%lld d=%lld p=%d st=%s\n", dtype_name(dt),
                                             (long long)n, (long long)n_h, (long long)d_h, p, strategy_name(st));
                            const DecodeResult got = gpu::tree_decode(q, cache, topo, st);
                            const double tol = decode_tolerance_abs(dt, max_abs(want.output));
                            const double err = max_abs_diff(got.output, want.output);
                            std::snprintf(what, sizeof what, "tree dt=%s n=%lld h=%lld d=%lld p=%d st=%s",
                                          dtype_name(dt), (long long)n, (long long)n_h, (long long)d_h, p,
                                          strategy_name(st));
                            expect(err <= tol, what, err, tol);
                            // same reporting counters as the reference
                            expect(got.collectives.size() == ref.collectives.size() &&
                                       got.collectives[0].reduce_rounds == ref.collectives[0].reduce_rounds &&
                                       got.collectives[0].broadcast_rounds == ref.collectives[0].broadcast_rounds,
                                   "collective rounds", 0, 0);
                            expect(got.cost.elems_sent_total() == ref.cost.elems_sent_total(), "elems_sent", 0, 0);
                            expect(got.cost.peak_elems_per_worker == ref.cost.peak_elems_per_worker, "peak", 0, 0);
                        }
                        const DecodeResult rw = ring_decode(q64, cache64, topo);
                        const DecodeResult rg = gpu::ring_decode(q, cache, topo);
                        const double tol = decode_tolerance_abs(dt, max_abs(rw.output));
                        const double err = max_abs_diff(rg.output, rw.output);
                        std::snprintf(what, sizeof what, "ring dt=%s n=%lld h=%lld d=%lld p=%d", dtype_name(dt),
                                      (long long)n, (long long)n_h, (long long)d_h, p);
                        expect(err <= tol, what, err, tol);
                    }
                }
    // validation throws like the reference (test_decode.cpp:239-251)
    {
        const Tensor q = seeded_random_tensor({1, 2, 1, 4}, 1, 1.0, DType::Float32);
        const Tensor k = seeded_random_tensor({1, 2, 16, 4}, 2, 1.0, DType::Float32);
        const ShardedKVCache cache = shard_kv(k, k, 4);
        bool threw = false;
        try {
            (void)gpu::tree_decode(q, cache, topology_for_workers(8));
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        expect(threw, "topology mismatch throws invalid_argument", 0, 0);
        threw = false;
        try {
            (void)gpu::tree_decode(seeded_random_tensor({1, 2, 3, 4}, 1, 1.0, DType::Float32), cache,
                                   topology_for_workers(4));
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        expect(threw, "multi-row query throws invalid_argument", 0, 0);
        threw = false;
        try {
            (void)gpu::tree_decode(retag(q, DType::Float64), shard_kv(retag(k, DType::Float64), retag(k, DType::Float64), 4),
                                   topology_for_workers(4));
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        expect(threw, "Float64 rejected with invalid_argument", 0, 0);
    }
    // energy formulation (energy.hpp:47-58) through treedec::gpu against the reference
    // at Float64 on the same grid values (test_energy.cpp:192-230)
    for (const DType dt : {DType::Float32, DType::Bf16})
        for (const std::int64_t n : {17LL, 300LL, 4096LL})
            for (const std::int64_t nq : {1LL, 3LL}) {
                const std::int64_t h = 2, d = 64;
                const std::uint64_t seed = 7 + static_cast<std::uint64_t>(n) + 11 * nq;
                const Tensor q = seeded_random_tensor({1, h, nq, d}, mix64(seed, 1), 1.0, dt);
                const Tensor k = seeded_random_tensor({1, h, n, d}, mix64(seed, 2), 1.0, dt);
                const Tensor v = seeded_random_tensor({1, h, n, d}, mix64(seed, 3), 1.0, dt);
                const Tensor src = seeded_random_tensor({1, h, nq, d}, mix64(seed, 4), 0.5, dt);
                const double tol = dt == DType::Bf16 ? 1e-3 : 1e-5;
                for (const int chunks : {1, 3, 8}) {
                    if (chunks > n) continue;
                    const EnergyEval want = energy_forward_parallel(retag(q, DType::Float64), retag(k, DType::Float64),
                                                                    retag(v, DType::Float64),
                                                                    retag(src, DType::Float64), chunks);
                    const EnergyEval got = gpu::energy_forward_parallel(q, k, v, src, chunks);
                    const double err = std::max({max_abs_diff(got.value, want.value),
                                                 max_abs_diff(got.row_max, want.row_max),
                                                 max_abs_diff(got.shifted_lse, want.shifted_lse)});
                    const double scale = std::max(1.0, max_abs(want.value));
                    std::snprintf(what, sizeof what, "energy fwd dt=%s n=%lld nq=%lld chunks=%d", dtype_name(dt),
                                  (long long)n, (long long)nq, chunks);
                    expect(err <= tol * scale, what, err, tol * scale);
                    const EnergyEval saved = energy_forward_parallel(retag(q, DType::Float64), retag(k, DType::Float64),
                                                                     retag(v, DType::Float64), Tensor{}, chunks);
                    const Tensor gw = energy_grad_parallel(retag(q, DType::Float64), retag(k, DType::Float64),
                                                           retag(v, DType::Float64), saved, chunks);
                    const Tensor gg = gpu::energy_grad_parallel(q, k, v, saved, chunks);
                    // the gradient is stored through the input grid like the reference's
                    // (Tensor::store): the reference's own bf16 decode tolerance applies
                    const double eg = max_abs_diff(gg, gw),
                                 tg = dt == DType::Bf16 ? decode_tolerance_abs(dt, max_abs(gw)) : tol * max_abs(gw);
                    std::snprintf(what, sizeof what, "energy grad dt=%s n=%lld nq=%lld chunks=%d", dtype_name(dt),
                                  (long long)n, (long long)nq, chunks);
                    expect(eg <= tg, what, eg, tg);
                }
            }
    std::printf("shim_parity: %d checks, %d failures\n", checks, failures);
    return failures == 0 ? 0 : 1;
}
