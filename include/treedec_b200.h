/*
 * treedec_b200.h -- C-ABI of the B200 tree-decode library
 * (paper_2408_04093_b200/libtreedec_b200.so).
 *
 * Drop-in boundary for the reference's decode path (namespace treedec,
 * /root/reference/proj/core). Plain pointers and sizes, no C++ or torch
 * types; every call returns a td_status and td_last_error() describes the
 * last failure on the calling thread. Status codes map onto the reference's
 * exception types (decode.cpp:14-24, numerics.cpp:13-23):
 *   TD_EINVAL  -> std::invalid_argument    TD_EDOMAIN -> std::domain_error
 *   TD_ECUDA / TD_ENCCL / TD_ESTATE -> std::runtime_error
 *
 * Tensor layouts are the reference's row-major ones (tensor.hpp:16-19,46-48):
 *   q    [b, n_q, d]        the single query row of each head (N_q = 1)
 *   k, v [b, n_kv, t, d]    one worker's contiguous sequence shard
 *   out  [b, n_q, d]        fp32
 * GQA: q head h attends kv head h / (n_q / n_kv); n_q == n_kv is the
 * reference's MHA contract (attention.cpp:18-28).
 * dtype codes follow treedec::DType (dtype.hpp:13): 0 f64, 1 f32, 2 bf16.
 * The GPU path computes on f32 or bf16 inputs with fp32 accumulation.
 *
 * Threading: stateless calls are thread-safe. A td_context is used by one
 * host thread at a time (one context per GPU / rank), the analogue of one
 * reference worker (decode.cpp:28-46).
 */
#ifndef TREEDEC_B200_H
#define TREEDEC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TD_OK = 0,
    TD_EINVAL = 1,  /* invalid_argument: shapes, dtype, topology, p > N  */
    TD_EDOMAIN = 2, /* domain_error: NaN / no attended key            */
    TD_ECUDA = 3,
    TD_ENCCL = 4,
    TD_ESTATE = 5 /* call order (e.g. decode before td_kv_place)     */
} td_status;

typedef enum { TD_F64 = 0, TD_F32 = 1, TD_BF16 = 2 } td_dtype;

/* treedec::ReduceStrategy (reduce.hpp:10). It is validated and names the
 * reduction schedule whose round counts the host mirrors report
 * (DecodeResult::collectives, reduce.cpp:60-139). The GPU collective itself is
 * one NCCL allreduce per step (NCCL picks its algorithm; NCCL_ALGO steers it
 * process-wide) or the one-shot exchange (TD_P2P): the result is the same
 * exact combine whichever schedule is named. */
typedef enum { TD_TREE_BINARY = 0, TD_RING_ALLREDUCE = 1, TD_HIERARCHICAL = 2 } td_strategy;

/* flags for td_tree_decode / td_ring_decode */
enum {
    TD_HOST_IO = 1,      /* q and out are host pointers (copies inside the call) */
    TD_TIME_KERNELS = 2, /* record CUDA events around the split-KV kernel (K1) */
    TD_BF16_OUT = 4,     /* also write a bf16 copy of out (td_output_bf16)      */
    TD_TIME_PHASES = 8,  /* record CUDA events between the phases of the step   */
    TD_P2P = 16,         /* tree decode: one-shot NVLink exchange instead of the
                            two NCCL allreduces (needs td_p2p_open)              */
    TD_DEBUG_TS = 32,    /* kernels record %globaltimer stamps (td_debug_stamps) */
    TD_DETERMINISTIC = 64, /* static split (the default, see td_set_deterministic):
                              every CTA streams a fixed, calibrated range, so the
                              grouping of the sums and the result are bitwise
                              identical from call to call on a context */
    TD_PINNED_IO = 128,   /* with TD_HOST_IO: out is a pinned host buffer (cudaHostAlloc
                             / cudaHostRegister). The combine kernel writes it in place
                             and signals completion through pinned host memory; the
                             call returns when the host sees that signal (no stream
                             synchronisation). Ignored where it cannot apply (the
                             NCCL path, TD_BF16_OUT). */
    TD_DYNAMIC = 256,     /* this call: hand the last ~15% of each (batch, kv-head)
                             row out at run time to the SMs that stream fastest
                             (and let idle warps take other rows' chunks on long
                             shards). Up to ~2.5% faster on some shapes; results
                             then agree to ~1e-7, not bitwise, between calls. */
    TD_GRAPH = 512,       /* paper-literal NCCL path (nranks > 1 without TD_P2P), device
                             buffers: capture the step (K1, K2, allreduce(max), K3,
                             allreduce(sum), K4) as a CUDA graph once per shape and
                             replay it (TD_NCCL_GRAPH=1 sets it for every call) */
    TD_NCCL_DEVICE = 1024 /* tree decode, nranks > 1 (after td_comm_init): the same
                             two allreduces -- max of lse, then sum of [n|d] -- run
                             inside one combine kernel through NCCL's device API:
                             every rank stores into and polls the others' copies of
                             a symmetric NCCL window (NCCL >= 2.28, all ranks in one
                             NVLink domain). The window is registered on the first
                             such call of a size (collective: every rank makes the
                             call). TD_EINVAL when unavailable. */
};

typedef struct td_context td_context;

int td_version(void);
const char* td_last_error(void);

/* ---------------------------------------------------------------------
 * Stateless device primitives (device pointers; stream may be NULL).
 * ------------------------------------------------------------------- */

/* Elements [start, start+len) of every row of seeded_random_tensor(
 * [bh_count, seq, d], seed, scale, dtype), written as [bh_count, len, d].
 * Bit-exact with numerics.cpp:41-50 + dtype.cpp:13-42 (double -> dtype
 * directly). Replaces: seeded_random_tensor + slice_seq. */
int td_seeded_fill(int dtype, void* dst, uint64_t seed, double scale, int64_t bh_count,
                   int64_t seq, int64_t start, int64_t len, int64_t d, void* stream);

/* Process-wide default of every call (including the stateless
 * td_decode_partial): on (1, the default) = the static split, bitwise-
 * reproducible results like the reference's (test_decode.cpp:185-202);
 * off (0) = the dynamic pool of TD_DYNAMIC for every call. */
int td_set_deterministic(int on);

/* Workspace bytes td_decode_partial needs for this shard shape. */
int td_decode_workspace_bytes(int dtype, int64_t b, int64_t n_q, int64_t n_kv, int64_t t,
                              int64_t d, size_t* bytes);

/* attention_chunk_partial (attention.hpp:49-50, attention.cpp:146-168) of q
 * against one shard: fp32 row_max [b,n_q], lse [b,n_q], out [b,n_q,d].
 * Empty shard (t = 0) gives the identity (-inf, -inf, 0). */
int td_decode_partial(int dtype, const void* q, const void* k, const void* v, int64_t b,
                      int64_t n_q, int64_t n_kv, int64_t t, int64_t d, double scale,
                      float* row_max, float* lse, float* out, void* workspace,
                      size_t workspace_bytes, void* stream);

/* combine_partials (attention.hpp:65, attention.cpp:207-241): lse [P][rows],
 * out [P][rows][d] -> result [rows][d]. TD_EINVAL if a row attends no key. */
int td_combine_partials(int P, const float* lse, const float* out, int64_t rows, int64_t d,
                        float* result, void* stream);

/* partial_to_numerator (attention.hpp:70, attention.cpp:243-266):
 * nd = [num rows*d | den rows] against a common shift [rows]. */
int td_partial_to_numerator(const float* lse, const float* out, const float* shift,
                            int64_t rows, int64_t d, float* nd, void* stream);

/* combine_pair (attention.hpp:59, attention.cpp:178-205), in place into
 * left; left covers lower key indices. */
int td_combine_pair(float* l_max, float* l_lse, float* l_out, const float* r_max,
                    const float* r_lse, const float* r_out, int64_t rows, int64_t d,
                    void* stream);

/* out = num / den over nd = [num | den] (decode.cpp:165-173). */
int td_finalize(const float* nd, int64_t rows, int64_t d, float* out, void* out_bf16,
                void* stream);

/* ---------------------------------------------------------------------
 * Context: one per GPU / rank. Owns the stream, the KV shard placed in HBM,
 * workspaces and the NCCL communicator of the tree / ring collectives.
 * ------------------------------------------------------------------- */
int td_create(int device, td_context** ctx);
int td_destroy(td_context* ctx);
int td_stream(td_context* ctx, void** stream);

/* NCCL bootstrap (one process per GPU): rank 0 calls td_comm_unique_id and
 * ships the 128 bytes to the other ranks; every rank calls td_comm_init.
 * Without td_comm_init the context is a world of one (p = 1). */
int td_comm_unique_id(unsigned char id[128]);
int td_comm_init(td_context* ctx, int nranks, int rank, const unsigned char id[128]);
int td_comm_info(td_context* ctx, int* nranks, int* rank);

/* One-shot NVLink exchange (the single-collective exact combine, SURVEY.md
 * 8(f)1): each rank exports a CUDA-IPC handle of its exchange buffer sized
 * for max_rows = b * n_q rows of head_dim d, the handles are all-gathered by
 * the caller (rank order, nranks * 64 bytes) and every rank opens its peers'.
 * td_tree_decode with TD_P2P then pushes each rank's partial into every
 * peer's HBM and combines the p partials locally (one exchange, no NCCL).
 * A peer that never delivers within ~2 s makes the step fail: td_tree_decode
 * returns TD_ECUDA at its next synchronising point (TD_HOST_IO calls: the
 * same call; device calls: the next call, or td_p2p_status, which waits for
 * the stream and reports 1). The exchange must then be re-opened on every
 * rank (td_p2p_handle + td_p2p_open) before TD_P2P is used again. */
int td_p2p_handle(td_context* ctx, int64_t max_rows, int64_t d, unsigned char handle[64]);
int td_p2p_open(td_context* ctx, const unsigned char* handles);
int td_p2p_status(td_context* ctx, int* error);

/* shard_kv (decode.hpp:24, decode.cpp:68-85) for this rank: places rows
 * [start, start+len) of every (batch, kv-head) of a cache of seq_len tokens.
 * k/v are [b, n_kv, len, d] on the host (from_host = 1) or device. */
int td_kv_place(td_context* ctx, int dtype, int64_t b, int64_t n_kv, int64_t seq_len,
                int64_t d, int64_t start, int64_t len, const void* k, const void* v,
                int from_host);

/* Generates this rank's shard in place with the seeded generator: k, v =
 * seeded_random_tensor([b, n_kv, seq_len, d], seed_k / seed_v, scale, dtype)
 * restricted to chunk_extents(seq_len, nranks)[rank] (attention.cpp:268-275). */
int td_kv_generate(td_context* ctx, int dtype, int64_t b, int64_t n_kv, int64_t seq_len,
                   int64_t d, uint64_t seed_k, uint64_t seed_v, double scale);

/* KV append, the caller side of tree_decode in a generation loop (SURVEY.md
 * section 8(f)2): the cache grows by one token that lands at the end of the
 * last shard (rank p-1). Every rank calls it (seq_len += 1 everywhere); only
 * rank p-1 reads k/v, one [b, n_kv, 1, d] token in the cache dtype (host or
 * device). Capacity grows geometrically (or to td_kv_reserve's size).
 * A host token is copied in by the call. A device token on a bf16 cache is
 * fused: the next td_tree_decode's split kernel writes it into the cache while
 * it streams (no append kernel on the step); any other use of the cache first
 * writes it with an append kernel. The device buffers must therefore stay
 * unchanged until the next call on this context that reads the cache has run
 * on the context's stream (td_stream). TD_FUSED_APPEND=0 appends eagerly.
 * tree_decode is exact under any partition (safe-softmax invariance), so the
 * result equals the reference's decode over the grown cache. */
int td_kv_append(td_context* ctx, const void* k, const void* v, int from_host);
/* Reserves room for `tokens` more appended tokens on rank p-1 (no-op elsewhere). */
int td_kv_reserve(td_context* ctx, int64_t tokens);

/* ---- Energy formulation (energy.hpp:24-58) --------
 * The attention energy of a query row is F = log sum_a exp(q.k_a + src.v_a)
 * (no 1/sqrt(d) scale, like the reference); at src = 0 its gradient with
 * respect to src is the attention output. Layouts: q, src [b][h][nq][d] (nq
 * query rows per head), k, v [b][h][t][d] (MHA: the reference requires equal
 * q and kv heads, energy.cpp:15-25). Stats are fp32, natural log.
 *
 * td_energy_partial: one key chunk -> per row (row_max, lse, out), out the
 * softmax-weighted values. src may be NULL (zero source).
 * td_energy_combine: energy_forward_parallel's reductions (energy.cpp:181-198)
 * over P chunk partials ([P][rows]) -> value, row_max, shifted_lse.
 * td_energy_grad_combine: energy_grad_parallel (energy.cpp:205-259) from P
 * zero-source chunk partials and the saved forward: grad = sum_c
 * e^(lse_c - row_max - shifted) out_c. */
int td_energy_workspace_bytes(int dtype, int64_t b, int64_t h, int64_t nq, int64_t t, int64_t d,
                              size_t* bytes);
int td_energy_partial(int dtype, const void* q, const void* src, const void* k, const void* v,
                      int64_t b, int64_t h, int64_t nq, int64_t t, int64_t d, float* row_max,
                      float* lse, float* out, void* workspace, size_t workspace_bytes, void* stream);
int td_energy_combine(int P, const float* row_max, const float* lse, int64_t rows, float* value,
                      float* row_max_out, float* shifted, void* stream);
int td_energy_grad_combine(int P, const float* lse, const float* out, const float* row_max,
                           const float* shifted, int64_t rows, int64_t d, float* grad, void* stream);

/* The paper's Alg. 1 / Alg. 2 across the ranks of a context (device pointers):
 * td_energy_forward -- local (row_max, lse) of the placed shard, allreduce(max),
 * e^(lse - max), allreduce(sum) -> value, row_max, shifted [b][h][nq];
 * td_energy_grad -- with the saved forward, sum_a e^(s_a - F) v_a over the
 * shard, allreduce(sum) -> grad [b][h][nq][d] (= the attention output). */
int td_energy_forward(td_context* ctx, const void* q, const void* src, int64_t nq, float* value,
                      float* row_max, float* shifted, int flags);
int td_energy_grad(td_context* ctx, const void* q, int64_t nq, const float* row_max,
                   const float* shifted, float* grad, int flags);

/* The per-SM speed calibration of the split kernel's static partition (made on
 * the first long decode of a context): gain = measured K1 time saved over the
 * equal split (fraction); state -1 failed, 0 not run, 1 kept equal weights
 * (gain too small), 2 weights in use. */
int td_calibration_info(td_context* ctx, double* gain, int* state);

/* Shard geometry of the placed cache. */
int td_kv_info(td_context* ctx, int64_t* start, int64_t* len, size_t* bytes);
/* Device pointers of the placed shard (for tests). */
int td_kv_pointers(td_context* ctx, void** k, void** v);

/* tree_decode (decode.hpp:70-72, decode.cpp:100-184): local partial (K1+K2),
 * allreduce(max) of lse, rescale (K3), one fused sum-allreduce of [n|d],
 * out = n/d (K4). q [b, n_q, d] in the cache dtype; out [b, n_q, d] fp32,
 * identical on every rank. p = nranks must not exceed seq_len. */
int td_tree_decode(td_context* ctx, const void* q, int64_t n_q, double scale, int strategy,
                   float* out, int flags);

/* ring_decode (decode.hpp:77-78, decode.cpp:186-251): p-1 rotations of the
 * KV shards around the ring (NCCL send/recv over NVLink), each rank folding
 * the received chunk's partial with combine_pair in the reference order
 * (own chunk, then chunks rank-1, rank-2, ...). out is identical on all
 * ranks (the reference returns worker 0's). */
int td_ring_decode(td_context* ctx, const void* q, int64_t n_q, double scale, float* out,
                   int flags);

/* local_partials (decode.cpp:28-46) for this rank alone: the
 * attention_chunk_partial of q against the placed shard, fp32 row_max /
 * lse [b, n_q] and out [b, n_q, d]. TD_HOST_IO: q and the outputs are host
 * pointers. */
int td_local_partial(td_context* ctx, const void* q, int64_t n_q, double scale, float* row_max,
                     float* lse, float* out, int flags);

/* bf16 copy of the last output (TD_BF16_OUT), device pointer. */
int td_output_bf16(td_context* ctx, const void** out_bf16);

/* Mean duration (ms) of K1 over the calls made with TD_TIME_KERNELS since
 * the last td_reset_kernel_timer, and the number of timed calls. */
int td_kernel_time(td_context* ctx, double* mean_ms, int* calls);
int td_reset_kernel_timer(td_context* ctx);

/* Mean duration (ms) of each phase of the decode steps made with
 * TD_TIME_PHASES since the last td_reset_kernel_timer: phases[i] is the time
 * between mark i and mark i+1 (tree: K1, K2, allreduce(max), K3,
 * allreduce(sum), K4); *n = number of phases recorded. */
int td_phase_times(td_context* ctx, double* phases, int max_phases, int* n, int* calls);

/* Stamps of the last TD_DEBUG_TS call (ns, %globaltimer): [0] first K1 CTA
 * start, [1] last K1 CTA end, [8 + 8*blk + k] stages of K2 block blk
 * (0 entry, 1 merged + pushed, 2 fenced + flagged, 3 peers seen, 4 done),
 * [4096 + 2c], [4097 + 2c] start / end of K1 CTA c (n up to 6144). */
int td_debug_stamps(td_context* ctx, unsigned long long* out, int n);

/* Kernels of this library launched by the last decode call, and the
 * algorithmic HBM bytes of its K1 launch(es) (K + V of the shard). */
int td_last_launch_stats(td_context* ctx, int* kernels, double* kv_bytes, int* split_kernel);

/* Peak device bytes held by the context (KV shard, ring buffers, workspaces). */
int td_memory_bytes(td_context* ctx, size_t* bytes);

/* ---------------------------------------------------------------------
 * Worker group: the reference's p in-process workers (decode.hpp:70-72,
 * parallel_workers threads at decode.cpp:37-41) in ONE process. Worker w is a
 * td_context on device devs[w * ndev / workers] (contiguous placement,
 * cluster.hpp:18-24) with nranks = workers, rank = w; several workers may
 * share a GPU. Place each worker's shard through its context
 * (td_group_context + td_kv_place / td_kv_generate), open the exchange once
 * (td_group_p2p_open: every worker's exchange buffer, peers addressed as
 * device pointers over NVLink or in the same HBM -- no IPC, no NCCL), then
 * td_group_tree_decode runs K1 + K2x on every worker from one host thread:
 * the one-shot exact combine (allreduce(max) + rescale + allreduce(sum) +
 * divide, decode.cpp:129-173). Device q / out live on worker 0's device and
 * are ordered on worker 0's stream (td_stream of worker 0); TD_HOST_IO takes
 * host buffers and returns after every worker's step, reporting an exchange
 * timeout as TD_ECUDA. Workers sharing a GPU launch K1 without the
 * programmatic early launch (a waiting grid would hold the SMs a peer's K1
 * needs) and skip the per-SM calibration (the SMs are shared).
 * ------------------------------------------------------------------- */
typedef struct td_group td_group;
int td_group_create(int ndev, const int* devs, int workers, td_group** group);
int td_group_destroy(td_group* group);
int td_group_context(td_group* group, int worker, td_context** ctx);
int td_group_p2p_open(td_group* group, int64_t max_rows, int64_t d);
int td_group_tree_decode(td_group* group, const void* q, int64_t n_q, double scale, int strategy, float* out,
                         int flags);

#ifdef __cplusplus
}
#endif
#endif /* TREEDEC_B200_H */
