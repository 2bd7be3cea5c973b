/*
 * treedec_oracle.h -- CPU restatement of the reference's tree-decode path.
 *
 * TEST INFRASTRUCTURE ONLY. This library is the parity checker for the CUDA
 * product path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it. The product
 * (paper_2408_04093_b200) never links or calls it.
 *
 * Every function restates one reference function, in the same operation
 * order, in IEEE double, so that at DType Float64 the results are bitwise
 * equal to the reference's (checked against oracle/_ref in tests/).
 * Citations are relative to /root/reference/proj/core.
 *
 * Parity pinned: tests/test_oracle.py checks this restatement against the
 * reference library compiled by oracle/Makefile (oracle/_ref) and against the
 * committed fixtures in tests/golden/ (generated from oracle/_ref by
 * tests/golden/make_golden.py).
 *
 * Layouts (row-major, like Tensor::offset4, tensor.hpp:46-48):
 *   q    [b, n_q, d]          (the single query row of each head)
 *   k, v [b, n_kv, seq, d]    (full cache; shards are row ranges of seq)
 *   per-row stats [b, n_q]    out [b, n_q, d]
 * GQA: q head h reads kv head h / (n_q / n_kv). With n_q == n_kv this is
 * exactly the reference's MHA contract (attention.cpp:18-28).
 */
#ifndef TREEDEC_ORACLE_H
#define TREEDEC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* DType (dtype.hpp:13) and ReduceStrategy (reduce.hpp:10) codes. */
enum { ORC_F64 = 0, ORC_F32 = 1, ORC_BF16 = 2 };
enum { ORC_TREE_BINARY = 0, ORC_RING = 1, ORC_HIER = 2 };

/* numerics.cpp:30-39 */
uint64_t orc_mix64(uint64_t seed, uint64_t counter);
double orc_uniform01(uint64_t seed, uint64_t counter);

/* dtype.cpp:13-42 (round_bf16 / round_f32 / round_to_dtype), :53-55 */
double orc_round(double x, int dtype);
int orc_stats_dtype(int dtype);

/* Elements [offset, offset+n) of seeded_random_tensor(shape, seed, scale,
 * dtype) (numerics.cpp:41-50), rounded to dtype. Returns -1 if scale <= 0. */
int orc_seeded_fill(uint64_t seed, double scale, int dtype, int64_t offset, int64_t n,
                    double* out);

/* chunk_extents, attention.cpp:268-275. Returns -1 on bad arguments. */
int orc_chunk_extents(int64_t n, int p, int64_t* out);

/* attention_chunk_partial (attention.cpp:146-168) of q against rows
 * [start, start+len) of k/v (row_scores :32-46, row_softmax_stats :52-77).
 * Empty chunk -> (-inf, -inf, 0). nthreads > 1 splits rows over pthreads
 * (rows are independent; the result does not depend on nthreads). */
int orc_chunk_partial(const double* q, const double* k, const double* v, int64_t b,
                      int64_t n_q, int64_t n_kv, int64_t seq, int64_t start, int64_t len,
                      int64_t d, double scale, int dtype, int nthreads, double* row_max,
                      double* lse, double* out);

/* numerics.cpp:22-28. Returns NaN on NaN input (the reference throws). */
double orc_lse_combine(double a, double b);

/* combine_pair, attention.cpp:178-205, over `rows` rows of width d. */
int orc_combine_pair(const double* l_max, const double* l_lse, const double* l_out,
                     const double* r_max, const double* r_lse, const double* r_out, int64_t rows,
                     int64_t d, int dtype, double* o_max, double* o_lse, double* o_out);

/* combine_partials, attention.cpp:207-241. lse is [P][rows], out is
 * [P][rows][d]. Returns -1 if some row has no attended key (the reference
 * throws invalid_argument). */
int orc_combine_partials(int P, const double* lse, const double* out, int64_t rows, int64_t d,
                         int dtype, double* result);

/* partial_to_numerator, attention.cpp:243-266. */
int orc_partial_to_numerator(const double* lse, const double* out, const double* shift,
                             int64_t rows, int64_t d, int dtype, double* num, double* den);

/* Round counts of allreduce_schedule (reduce.cpp:60-139). */
int orc_schedule_rounds(int strategy, int nodes, int gpus_per_node, int* reduce_rounds,
                        int* total_rounds);

/* tree_decode (decode.cpp:100-184) with shard_kv (decode.cpp:68-85),
 * topology_for_workers (cluster.cpp:11-22) and execute_schedule
 * (reduce.hpp:62-92). Returns -1 on invalid arguments (reference:
 * invalid_argument), -2 on NaN (domain_error). */
int orc_tree_decode(const double* q, const double* k, const double* v, int64_t b, int64_t n_q,
                    int64_t n_kv, int64_t seq, int64_t d, int p, int strategy, double scale,
                    int dtype, int nthreads, double* out);

/* ring_decode (decode.cpp:186-251): root folds parts[0], parts[p-1], ... */
int orc_ring_decode(const double* q, const double* k, const double* v, int64_t b, int64_t n_q,
                    int64_t n_kv, int64_t seq, int64_t d, int p, double scale, int dtype,
                    int nthreads, double* out);

/* attention_naive (attention.cpp:87-106), non-causal, single query row. */
int orc_attention_naive(const double* q, const double* k, const double* v, int64_t b,
                        int64_t n_q, int64_t n_kv, int64_t seq, int64_t d, double scale,
                        int dtype, int nthreads, double* out);

/* energy_forward_parallel (energy.cpp:152-203): q, src [b][h][nq][d] (src may
 * be NULL: zero source), k, v [b][h][n][d]; value, row_max, shifted [b][h][nq].
 * Returns -1 unless 1 <= chunks <= n. */
int orc_energy_forward_parallel(const double* q, const double* k, const double* v, const double* src,
                                int64_t b, int64_t h, int64_t nq, int64_t n, int64_t d, int chunks,
                                int dtype, double* value, double* row_max, double* shifted);

/* energy_grad_parallel (energy.cpp:205-259) replaying a zero-source forward:
 * grad [b][h][nq][d] = the attention output. */
int orc_energy_grad_parallel(const double* q, const double* k, const double* v, const double* row_max,
                             const double* shifted, int64_t b, int64_t h, int64_t nq, int64_t n,
                             int64_t d, int chunks, int dtype, double* grad);

#ifdef __cplusplus
}
#endif
#endif
