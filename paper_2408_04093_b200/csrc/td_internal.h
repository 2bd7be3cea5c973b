// td_internal.h -- host-side declarations shared by the kernel launchers
// (td_kernels.cu) and the C-ABI / context layer (td_capi.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace td {

enum DType { kF64 = 0, kF32 = 1, kBF16 = 2 };

// K1 tracks the (batch, head) rows a CTA's range touches in per-warp bit masks:
// a split plan (equal or speed-weighted) may span at most this many per CTA.
constexpr int kMaxSegments = 32;

inline int dtype_bytes(int dt) { return dt == kBF16 ? 2 : (dt == kF32 ? 4 : 8); }

// Split-KV work decomposition of one shard (K1). The shard holds bh_count
// = b * n_kv contiguous rows of t tokens ([bh][t][d], the reference's
// [b, h, seq, d] row-major layout restricted to this worker's seq range).
// Tiles of `tile` tokens are numbered bh-major; CTA c owns the contiguous
// range [c*total/ctas, (c+1)*total/ctas), so every SM gets the same number
// of tiles (+-1) whatever b, n_kv and t are.
struct SplitPlan {
    // tiles_per_bh / total_tiles describe the STATIC tile space (the first
    // tiles_per_bh tiles of every bh, bh-major); the remaining pool_tiles of
    // each bh (from tile pool_first on) form the dynamic pool.
    int64_t bh_count = 0, t = 0, tiles_per_bh = 0, total_tiles = 0;
    int64_t row_stride = 0;  // tokens per bh row in memory (0: t; > t with append capacity)
    int64_t full_tiles_per_bh = 0, pool_first = 0, pool_tiles = 0;
    int pool_chunk = 0, slot_warps = 0;
    int d = 0, n_q = 0, n_kv = 0, group = 0;
    int tile = 0, warps = 0, ctas = 0, maxseg = 0;
    int kernel = 0;  // 0 generic, 1 bf16 mma (TMA), 2 f32 (bulk)
    int dtype = kBF16;
    // run-time state of a launch (set by the caller): pool counters
    // [2 parities][bh_count] u32, zero at rest except the last launch's
    // parity, and the parity of this launch (alternate between launches)
    unsigned* counters = nullptr;
    int parity = 0;
    // cross-row stealing: warps whose own rows' pools are empty take chunks of
    // any row's pool and fold them into one of that row's fslots foreign states
    // ([bh_count][fslots]; 0 = off)
    int fslots = 0;
    // deterministic chunk pool (pool mode 2): every pool chunk k of row bh is its own
    // state, fslot (bh, k) with fslots = chunks per row; any warp of the grid claims
    // chunks from one queue (pool counter [0]), and since a chunk's state does not
    // depend on who computes it, results stay bitwise reproducible
    bool dpool = false;
    // tokens of every row that no kernel ahead of this launch on the stream may
    // still be writing (0: none). k1_bf16 loads its first tiles below it before
    // griddepcontrol.wait. Set only for the context's own cache (td_capi.cu
    // kv_safe): everything up to the last decode's length, or all of it after
    // a synchronising placement.
    int64_t t_safe = 0;
    // calibrated static partition (device tables, optional; see
    // build_partition): CTA c owns static tiles [x_table[c], x_table[c+1])
    const int64_t* x_table = nullptr;
    const int* bh_table = nullptr;
    // SM affinity of the calibrated partition (optional): the CTA on SM s takes
    // index sm_to_cta[s] (claimed with claims[c] = epoch; a CTA whose SM is
    // already taken in this launch takes the next free index), so CTA c runs
    // where its speed weight was measured whatever order the CTAs launch in
    const int* sm_to_cta = nullptr;
    unsigned* claims = nullptr;
    unsigned epoch = 0;
    // debug instrumentation of this launch (owned by the calling context, null = off):
    // TD_DEBUG_TS stamps [0] min K1 CTA start, [1] max K1 CTA end, [8 + 8*blk + k] K2
    // block stages, [2048 + c] / [4096 + 2c] per-CTA SM and times; TD_DEBUG_TIMELINE
    // per-step slot of 4 stamps (K1Args::tl) and per-CTA stamps (tl_cta)
    unsigned long long* dbg = nullptr;
    unsigned long long* tl = nullptr;
    unsigned long long* tl_cta = nullptr;
    // TD_PINNED_IO: the combine kernel's last warp stores done_epoch into the
    // mapped host word done_flag (done_ctr counts its warps), which the caller polls
    unsigned* done_ctr = nullptr;
    unsigned* done_flag = nullptr;
    unsigned done_epoch = 0;
    // fused KV append (bf16 kernel): the token appended since the last decode is
    // still only in the caller's buffers app_k / app_v ([bh][d]); the warp that
    // processes the tile holding position app_pos of a row patches that row's
    // token into its staged tile and writes it into the cache (no append kernel)
    const void* app_k = nullptr;
    const void* app_v = nullptr;
    int64_t app_pos = -1;
    // streamed combine (td_capi.cu stream_setup; stream_plan): K1 publishes each warp's
    // static state and each chunk state with a flag word = sepoch once written, and
    // the split K2 folds them as they arrive instead of after K1's grid completes.
    // Flags: [ctas * warps] static, then [bh_count][fslots] chunks; sepoch is new
    // for every launch of the buffer (graph replays patch it, graph_set_k*_epoch)
    unsigned* sflag = nullptr;
    unsigned sepoch = 0;
    int* serr = nullptr;  // mapped host word a streamed K2 sets when it gives up waiting (~1 s)
    size_t sflag_words() const { return size_t(ctas) * size_t(warps) + size_t(bh_count) * size_t(fslots); }
    // launch K1 as a programmatic dependent of the preceding kernel (off when several
    // contexts share one GPU and a peer's K1 must get SMs while this one's exchange waits)
    bool pdl = true;
    int64_t slots() const { return int64_t(ctas) * slot_warps * maxseg; }
    // workspace: slot_m, slot_l [slots][group]; slot_o [slots][group][d] (fp32),
    // then the per-CTA merged states [ctas * maxseg][group] (+ [..][d])
    size_t workspace_bytes() const {
        return sizeof(float) * ((size_t(slots()) + size_t(ctas) * maxseg) * size_t(group) * size_t(2 + d) +
                                size_t(bh_count) * size_t(fslots) * size_t(group) * size_t(2 + d));
    }
    // [2 parities][bh_count] pool chunk counters, then [2][bh_count] foreign-slot counters
    size_t counters_bytes() const { return sizeof(unsigned) * 4 * size_t(bh_count > 0 ? bh_count : 1); }
};

// Whether launches of the plan use the streamed combine (SplitPlan::sflag).
bool stream_plan(const SplitPlan& p);

// TD_DEBUG_TS: a one-thread kernel writing %globaltimer to *p (front-end gaps).
cudaError_t launch_stamp(unsigned long long* p, cudaStream_t stream);

// Chooses the kernel and grid for a shard. Returns false (with msg) when the
// shape is unsupported.
// pool_mode: 0 static split; 1 the dynamic home pool (+ stealing on long shards),
// results agree to ~1e-7 between calls; 2 the deterministic chunk pool (bitwise
// reproducible, see SplitPlan::dpool). generic_only forces k1_generic (needed for
// an energy source term).
bool plan_split(int dtype, int64_t b, int n_q, int n_kv, int64_t t, int d, int sm_count,
                SplitPlan& plan, std::string& msg, int pool_mode = 1, bool generic_only = false);

// Static partition proportional to per-CTA speeds (weights[c] > 0, size
// plan.ctas): x[c] = first static tile of CTA c (x has ctas + 1 entries),
// bh[3 bh + {0, 1, 2}] = (first covering CTA, last covering CTA, segment of
// bh in the first). Raises plan.maxseg when the uneven ranges need it.
void build_partition(SplitPlan& plan, const float* weights, int64_t* x, int* bh);

// K1 (+ merge tail): attention_chunk_partial of q against one shard, written as fp32
// (row_max, lse, out) rows [b][n_q] / [b][n_q][d]. tmk/tmv are the shard's
// tensor maps (bf16 mma kernel only; may be null otherwise).
cudaError_t launch_decode_partial(const SplitPlan& plan, const void* q, const void* k,
                                  const void* v, float scale, const CUtensorMap* tmk,
                                  const CUtensorMap* tmv, void* workspace, float* row_max,
                                  float* lse, float* out, cudaStream_t stream,
                                  cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr,
                                  const void* src = nullptr);

// K1 with the final-output tail (p = 1: the local partial is the answer).
cudaError_t launch_decode_final(const SplitPlan& plan, const void* q, const void* k, const void* v,
                                float scale, const CUtensorMap* tmk, const CUtensorMap* tmv,
                                void* workspace, float* out, cudaStream_t stream,
                                cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr);

// One-shot NVLink exchange buffers (td_p2p_*): every rank's exchange buffer
// holds [2 parities][p sources][max_rows][d out | lse] LL words (value, epoch).
struct XchgArgs {
    float* const* peers;       // device array [p]
    int p = 1, rank = 0;
    unsigned epoch = 0;
    int64_t max_rows = 0;
    int64_t max_blocks = 0;
    int* error = nullptr;
    int pull = 0;  // see k2_exchange
};
constexpr int kXchgBlocks = 1024;  // upper bound on K2x blocks

// K1 + exchange tail: split-KV partial, merge, one-shot exchange and exact combine;
// out [b, n_q, d] fp32 final (identical on every rank). parts: 1 = K1 only, 2 = K2x
// only (same arguments, e.g. after a cross-stream wait), 3 = both.
cudaError_t launch_decode_exchange(const SplitPlan& plan, const void* q, const void* k, const void* v,
                                   float scale, const CUtensorMap* tmk, const CUtensorMap* tmv,
                                   void* workspace, const XchgArgs& xa, float* out, cudaStream_t stream,
                                   cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr, int parts = 3);

// CUDA-graph replay of a captured step: the split kernel's entry point for `plan`
// (to find its node) and an update of that node's per-launch state -- the SM
// affinity claim epoch and the streamed-combine epoch -- in an instantiated graph;
// likewise the streamed split K2 (partial tail) and its epoch.
const void* k1_function(const SplitPlan& plan);
cudaError_t graph_set_k1_epoch(cudaGraphExec_t exec, cudaGraphNode_t node, const SplitPlan& plan);
const void* k2_stream_function();
cudaError_t graph_set_k2_epoch(cudaGraphExec_t exec, cudaGraphNode_t node, const SplitPlan& plan);

// Builds the 2-D tensor map used by the bf16 kernel over rows x d elements.
bool make_tensor_map(CUtensorMap* map, const void* base, int64_t rows, int d, int tile_rows,
                     std::string& msg);

// K2n: allreduce(max) + partial_to_numerator + allreduce(sum) + n/d of K2's
// per-row (lse, out) over the ranks' symmetric NCCL windows (xa.peers: every
// rank's window base, from launch_lsa_peers); programmatic dependent of K2.
// K1 + the streamed split K2x with the paper-literal two-round combine inside it
// (kTailLiteral: K2n's protocol over the NCCL window of xa, no extra kernel);
// cudaErrorInvalidValue when the plan has no streamed combine or too many rows.
cudaError_t launch_decode_literal(const SplitPlan& plan, const void* q, const void* k, const void* v, float scale,
                                  const CUtensorMap* tmk, const CUtensorMap* tmv, void* workspace,
                                  const XchgArgs& xa, float* out, cudaStream_t stream, cudaEvent_t ev0 = nullptr,
                                  cudaEvent_t ev1 = nullptr);
cudaError_t launch_literal_combine(const float* lse, const float* o, const XchgArgs& xa, int64_t rows, int d,
                                   float* out, cudaStream_t stream);
// Words of one rank's K2n window: A [2][p][max_rows] + B [2][p][max_rows][d + 1].
inline size_t literal_window_bytes(int p, int64_t max_rows, int64_t d) {
    return 2 * size_t(p) * size_t(max_rows) * size_t(d + 2) * 8;
}
// NCCL device API (td_nccl_dev.cu): ptrs[k] = ncclGetLsaPointer(win, 0, k) for
// k < p, the load/store address of rank k's copy of a symmetric window; *ok
// (device int) = 1 when this rank's LSA team index equals its world rank.
// Returns cudaErrorNotSupported when built without the NCCL device headers.
cudaError_t launch_lsa_peers(void* win, int p, void** ptrs, int* ok, cudaStream_t stream);

// K3: partial_to_numerator; nd = [num rows*d | den rows].
cudaError_t launch_to_numerator(const float* lse, const float* out, const float* shift,
                                int64_t rows, int d, float* nd, cudaStream_t stream);
// K4: out = num / den (+ optional bf16 copy).
cudaError_t launch_finalize(const float* nd, int64_t rows, int d, float* out, void* out_bf16,
                            cudaStream_t stream);
cudaError_t launch_to_bf16(const float* src, int64_t n, void* dst, cudaStream_t stream);
// K5: combine_pair (left covers lower key indices). In-place into left.
cudaError_t launch_combine_pair(float* l_max, float* l_lse, float* l_out, const float* r_max,
                                const float* r_lse, const float* r_out, int64_t rows, int d,
                                cudaStream_t stream);
// combine_partials over P partials ([P][rows], [P][rows][d]); *bad_row set
// to 1 (device int) when some row has no attended key.
cudaError_t launch_combine_partials(int P, const float* lse, const float* out, int64_t rows,
                                    int d, float* result, int* bad_row, cudaStream_t stream);
// K6: element (bh, start+i, j) of seeded_random_tensor([bh_count, seq, d]).
cudaError_t launch_seeded_fill(int dtype, void* dst, uint64_t seed, double scale,
                               int64_t bh_count, int64_t seq, int64_t start, int64_t len,
                               int64_t d, cudaStream_t stream);
// KV append from device memory: token rows kt/vt [rows][d] into position pos
// of the [rows][cap][d] shard (programmatic launch, see td_kernels.cu).
cudaError_t launch_kv_append(int dtype, void* k, void* v, const void* kt, const void* vt, int64_t rows,
                             int64_t cap, int64_t pos, int d, cudaStream_t stream);
// Energy formulation (energy.cpp:152-259), see td_kernels.cu.
cudaError_t launch_energy_combine(int P, const float* rmax, const float* lse, int64_t rows, float* value,
                                  float* rmax_out, float* shifted, cudaStream_t stream);
cudaError_t launch_energy_grad_combine(int P, const float* lse, const float* out, const float* rmax,
                                       const float* shifted, int64_t rows, int d, float* grad,
                                       cudaStream_t stream);
cudaError_t launch_energy_shift(const float* lse, const float* m, int64_t rows, float* x, cudaStream_t stream);
cudaError_t launch_energy_finish(const float* m, const float* s, int64_t rows, float* value, float* rmax_out,
                                 float* shifted, cudaStream_t stream);
cudaError_t launch_energy_logz(const float* rmax, const float* shifted, int64_t rows, float* f,
                               cudaStream_t stream);

}  // namespace td
