// td_kernels.cu -- sm_100a kernels of the tree-decode hot path.
//
//   K1  split-KV flash-decode partial over one KV shard
//         k1_bf16   bf16 K/V: per-warp TMA (SWIZZLE_128B) pipeline, q.K^T and
//                   P.V on mma.sync m16n8k16 with tokens on M and the GQA
//                   group on N; P is split hi+lo bf16 so the P.V product keeps
//                   fp32 accuracy.
//         k1_f32    fp32 K/V: per-warp bulk-copy pipeline, CUDA-core FMA,
//                   batched butterfly reduce-scatter for the scores.
//         k1_generic any head dim <= 256 (test shapes), plain loads.
//       contract: attention_chunk_partial, attention.cpp:146-168.
//   K2  logsumexp combine of the per-warp split states into the shard's
//       (row_max, lse, out)            -- combine_partials, attention.cpp:207-241
//   K3  rescale n = o*e^(lse-m), d = e^(lse-m) -- partial_to_numerator :243-266
//   K4  finalize out = n/d               -- decode.cpp:165-173
//   K5  pairwise merge                   -- combine_pair, attention.cpp:178-205
//   K6  seeded generator                 -- seeded_random_tensor, numerics.cpp:41-50
//
// Split state ("slot") format shared by all K1 variants: m = running max of
// the scaled scores in log2 units, l = sum 2^(s - m), o = sum 2^(s - m) v
// (unnormalised), fp32, one per (cta, warp, segment, head-of-group).
#include <math_constants.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

#include "td_device.cuh"
#include "td_internal.h"

namespace td {

// One-shot NVLink exchange (the single-collective exact combine, SURVEY.md
// 8(f)1): every rank's exchange buffer holds [2 parities][p sources]
// [max_rows][d out | lse] LL words (value bits, epoch) -- see k2_exchange.
struct Xchg {
    float* const* peers;  // [p] exchange buffers (own included), device array
    int p, rank;
    unsigned epoch;
    int64_t max_rows;
    int* error;           // set on timeout
    int pull;             // 0: push own rows into every peer's buffer; 1: write own buffer, read peers'
};

// What K2 does with the merged rows.
// kTailLiteral (streamed split K2x only): the paper-literal two collective rounds
// (allreduce(max) of lse, then allreduce(sum) of [n | d]) over an NCCL symmetric
// window, inside the combine kernel -- K2n's protocol without its kernel boundary.
enum TailMode { kTailPartial = 0, kTailFinal = 1, kTailExchange = 2, kTailLiteral = 3 };
struct Tail {
    int mode;
    float* row_max;      // [b][n_q]      (partial)
    float* lse;          // [b][n_q]      (partial)
    float* out;          // [b][n_q][d]   (partial / final)
    Xchg x;              // (exchange)
};

struct K1Args {
    const void* q;  // [b][n_q][d], kv dtype
    const void* src;  // optional energy source, q's layout: score += src . v (k1_generic)
    const void* k;  // [bh][t][d]
    const void* v;
    int64_t bh_count, t, tiles_per_bh, total_tiles;
    int64_t row_stride;  // tokens between consecutive bh rows in memory (>= t: append capacity)
    int64_t t_safe;      // tokens of every row no kernel ahead of this grid may still be writing
                         // (SplitPlan::t_safe): their tiles may be loaded before the PDL wait
    int d, n_q, n_kv, group, ctas, maxseg;
    float scale_log2;
    float* slot_m;  // [slots][group]
    float* slot_l;
    float* slot_o;  // [slots][group][d]
    float* cslot_m; // per-CTA merged states [ctas * maxseg][group]
    float* cslot_l;
    float* cslot_o; // [ctas * maxseg][group][d]
    unsigned long long* dbg;  // optional globaltimer stamps (TD_DEBUG_TS)
    unsigned long long* tl;   // optional per-step timeline (TD_DEBUG_TIMELINE): [K1 first start,
                              // first CTA past the PDL wait, K1 last end, K2 last done]
    unsigned long long* tl_cta;  // TD_DEBUG_TIMELINE: per CTA index c, [2048 + c] smid,
                                 // [4096 + 2c] past the PDL wait, [4097 + 2c] end (last step)
    int reverse;              // debug: CTA c takes range ctas-1-c (TD_DEBUG_REVERSE)
    // dynamic "home" pool (k1_bf16): tiles [pool_first, pool_first + pool_tiles)
    // of every bh are handed out at run time in chunks of pool_chunk tiles to
    // the CTAs whose static range covers that bh; a warp folds them into its
    // own slot (phase 1) of that segment, so K2 merges the same states.
    int64_t pool_first, pool_tiles;
    int pool_chunk;
    int slot_warps;           // state slots per CTA and segment (warps * 2 with a pool)
    unsigned* pool_ctr;       // [bh_count] chunks taken (this launch's parity)
    unsigned* pool_next;      // [bh_count] the other parity's counters (zeroed by K2)
    // cross-row stealing (SplitPlan::fslots): foreign states [bh][fslots][group]
    // (+ [..][d]); fcnt[bh] counts the claimed ones (this parity), fcnt_next is zeroed by K2
    int fslots;
    int dpool;                   // SplitPlan::dpool: fslots are the pool's chunk states
    int steal_scans, steal_min;  // scans per warp; least chunks left worth a visit
    unsigned* fcnt;
    unsigned* fcnt_next;
    float* fslot_m;
    float* fslot_l;
    float* fslot_o;
    // calibrated static partition (optional): CTA c owns static tiles
    // [x_table[c], x_table[c+1]); bh_table[3 bh + {0,1,2}] = the first and last
    // CTA covering bh and bh's segment index in the first one
    const int64_t* x_table;
    const int* bh_table;
    const int* sm_to_cta;     // SM affinity of the calibrated partition (SplitPlan)
    unsigned* claims;
    unsigned epoch;
    int early_trigger;        // debug: PDL trigger at K1 entry instead of after the main loop
    const void* app_k;        // fused KV append (SplitPlan::app_*)
    const void* app_v;
    int64_t app_pos;
    // TD_PINNED_IO (SplitPlan): completion signalled to the host by K2's last warp
    unsigned* done_ctr;
    unsigned* done_flag;
    unsigned done_epoch;
    // streamed combine (SplitPlan::sflag): k1_bf16 publishes every warp's static
    // state (flag c * W + warp) and every chunk state (flag ctas * W + bh * fslots + k)
    // by storing sepoch once it is written; the split K2 folds them as they arrive
    unsigned* sflag;
    unsigned sepoch;
    int sspin;  // ns between polls of a streamed K2 warp (TD_K2_STREAM_SLEEP)
    int* serr;  // set when a streamed K2 gave up waiting for a state (mapped host memory)
    int solo;   // the context has its GPU to itself (SplitPlan::pdl): the exchange may launch wide
    Tail tail;
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}


// n / d for non-negative operands; 32-bit division (a short sequence) when both
// fit, the 64-bit software division (~100 dependent instructions) otherwise.
__device__ __forceinline__ int64_t div_nn(int64_t n, int64_t d) {
    if (((n | d) >> 32) == 0) return static_cast<int64_t>(static_cast<uint32_t>(n) / static_cast<uint32_t>(d));
    return n / d;
}

// TD_PINNED_IO: after a K2 warp's last output store (to mapped host memory),
// count the warp; the grid's last warp stores the step's epoch into the mapped
// host word the caller polls. Each warp releases its stores at gpu scope before
// it counts (the threadfence-reduction pattern); the last warp, having
// observed every count, fences at system scope once before the flag, which by
// cumulativity orders every warp's output before the flag for the host.
__device__ __forceinline__ void signal_done(const K1Args& a) {
    if (!a.done_flag) return;
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        __threadfence();
        const unsigned warps = gridDim.x * (blockDim.x >> 5);
        if (atomicAdd(a.done_ctr, 1u) == warps - 1) {
            *a.done_ctr = 0u;  // the next launch is stream-ordered after this one
            __threadfence_system();
            st_release_sys(a.done_flag, a.done_epoch);
        }
    }
}

__device__ __forceinline__ int64_t cta_begin(int64_t total, int c, int ctas) {
    return div_nn(total * c, ctas);
}

// End of K1: merges the W warp states of each of CTA c's segments into one
// CTA state (cslot_*), so K2 merges ctas, not ctas * W, states per row. All
// loads of a phase are independent (one L2 round trip each). sm must hold
// 3 * W * maxseg * group floats; every thread of the CTA calls this after a
// __syncthreads() that follows the warps' final flushes.
template <int W>
__device__ void cta_merge(const K1Args& a, int c, float* sm) {
    const int g = a.group, D = a.d, ms = a.maxseg;
    const int nsh = ms * g;
    const int nml = W * nsh;
    float* sm_m = sm;
    float* sm_l = sm + nml;
    float* sm_e = sm + 2 * nml;
    const int64_t base = int64_t(c) * nml;
    for (int i = threadIdx.x; i < nml; i += blockDim.x) {
        sm_m[i] = a.slot_m[base + i];
        sm_l[i] = a.slot_l[base + i];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nsh; i += blockDim.x) {
        float M = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < W; ++w) M = fmaxf(M, sm_m[w * nsh + i]);
        float L = 0.f;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const float m = sm_m[w * nsh + i];
            const float e = (m == -CUDART_INF_F) ? 0.f : fast_exp2(m - M);
            sm_e[w * nsh + i] = e;
            L += e * sm_l[w * nsh + i];
        }
        a.cslot_m[int64_t(c) * nsh + i] = M;
        a.cslot_l[int64_t(c) * nsh + i] = L;
    }
    __syncthreads();
    const int64_t n = int64_t(nsh) * D;
#pragma unroll 4
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
        const int i = static_cast<int>(e / D), j = static_cast<int>(e % D);
        float O = 0.f;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const float ew = sm_e[w * nsh + i];
            if (ew != 0.f) O += ew * a.slot_o[(base + int64_t(w) * nsh + i) * D + j];
        }
        a.cslot_o[(int64_t(c) * nsh + i) * D + j] = O;
    }
}

// cta_merge with the loads of the merge batched: every thread loads its o
// elements of all W states (EPT per thread per chunk) together with the
// (m, l) pairs, before the weights are known, so the first chunk costs one
// L2 round trip -- this is the epilogue of the grid's last CTA, on the step's
// critical path. Needs W * maxseg * group <= blockDim.x (else cta_merge).
template <int W, int D, int EPT>
__device__ void cta_merge_batched(const K1Args& a, int c, float* sm) {
    const int g = a.group, nsh = a.maxseg * g, nml = W * nsh, nt = blockDim.x;
    if (nml > nt) {
        cta_merge<W>(a, c, sm);
        return;
    }
    float* sm_m = sm;
    float* sm_l = sm + nml;
    float* sm_e = sm + 2 * nml;
    const int64_t base = int64_t(c) * nml;
    const int n = nsh * D;
    float ov[EPT][W];
    auto load_chunk = [&](int e0) {
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const int e = e0 + static_cast<int>(threadIdx.x) + k * nt;
            if (e < n) {
                const int i = e / D, j = e % D;
#pragma unroll
                for (int w = 0; w < W; ++w) ov[k][w] = a.slot_o[(base + int64_t(w) * nsh + i) * D + j];
            }
        }
    };
    auto use_chunk = [&](int e0) {
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
            const int e = e0 + static_cast<int>(threadIdx.x) + k * nt;
            if (e < n) {
                const int i = e / D, j = e % D;
                float O = 0.f;
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    const float ew = sm_e[w * nsh + i];
                    O += ew != 0.f ? ew * ov[k][w] : 0.f;  // never-flushed o may hold anything
                }
                a.cslot_o[(int64_t(c) * nsh + i) * D + j] = O;
            }
        }
    };
    float mv = -CUDART_INF_F, lv = 0.f;
    if (static_cast<int>(threadIdx.x) < nml) {
        mv = a.slot_m[base + threadIdx.x];
        lv = a.slot_l[base + threadIdx.x];
    }
    load_chunk(0);
    if (static_cast<int>(threadIdx.x) < nml) {
        sm_m[threadIdx.x] = mv;
        sm_l[threadIdx.x] = lv;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nsh; i += nt) {
        float M = -CUDART_INF_F;
#pragma unroll
        for (int w = 0; w < W; ++w) M = fmaxf(M, sm_m[w * nsh + i]);
        float L = 0.f;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const float m = sm_m[w * nsh + i];
            const float e = (m == -CUDART_INF_F) ? 0.f : fast_exp2(m - M);
            sm_e[w * nsh + i] = e;
            L += e * sm_l[w * nsh + i];
        }
        a.cslot_m[int64_t(c) * nsh + i] = M;
        a.cslot_l[int64_t(c) * nsh + i] = L;
    }
    __syncthreads();
    use_chunk(0);
    for (int e0 = EPT * nt; e0 < n; e0 += EPT * nt) {
        load_chunk(e0);
        use_chunk(e0);
    }
}

// Logical CTA index: blockIdx, or -- with a calibrated partition -- the index
// calibrated on this SM (SplitPlan::sm_to_cta), claimed for this launch; a CTA
// whose SM already hosts one of this grid's CTAs takes the next free index.
__device__ __forceinline__ int cta_index(const K1Args& a) {
    if (!a.sm_to_cta) return (a.reverse & 1) ? a.ctas - 1 - static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x);
    __shared__ int s_c;
    if (threadIdx.x == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        int c0 = smid < 1024 ? a.sm_to_cta[smid] : -1;
        if (c0 < 0 || c0 >= a.ctas) c0 = static_cast<int>(blockIdx.x);
        int cc = c0;
        for (int k = 0; k < a.ctas; ++k) {
            cc = c0 + k < a.ctas ? c0 + k : c0 + k - a.ctas;
            if (atomicExch(a.claims + cc, a.epoch) != a.epoch) break;
        }
        s_c = cc;
    }
    __syncthreads();
    return s_c;
}

// =========================================================================
// K1, bf16: tokens on M (16 per m-tile), heads on N (8), d on K.
// S^T[tok][head] = K[tok][:] . Q[head][:]   (A = K via ldmatrix, B = Q^T regs)
// O^T[d][head]  += V^T[d][tok] . P^T[tok][head] (A = V^T via ldmatrix.trans)
// Each warp owns S stages of (K tile, V tile) in shared memory, filled by
// its lane 0 with 128-B-swizzled TMA boxes; no block-wide sync in the loop.
// =========================================================================
template <int D, int T, int W, int S>
__global__ void __launch_bounds__(W * 32, 1)
    k1_bf16(const K1Args a, const __grid_constant__ CUtensorMap tmk,
            const __grid_constant__ CUtensorMap tmv) {
    constexpr int BOXES = D / 64;           // 128-byte boxes per row
    constexpr int BOX_BYTES = T * 128;
    constexpr int TILE_BYTES = BOXES * BOX_BYTES;
    constexpr int STAGE_BYTES = 2 * TILE_BYTES;
    constexpr int MT = T / 16;   // m-tiles (tokens) per tile
    constexpr int KS = D / 16;   // k-steps of q.K
    constexpr int MD = D / 16;   // m-tiles (d) of P.V

    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bars[W][S];
    __shared__ int64_t st_bh[W][S], st_tb[W][S];  // tile of each stage (bh, tile-in-bh)
    __shared__ int st_rec[W][S];                   // -1: static tile, else pool record
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);

    const unsigned long long t_start = (a.dbg || a.tl) ? gtimer() : 0ull;
    // PDL: K2 may be scheduled once every CTA of this grid has triggered (or
    // exited); it waits (griddepcontrol.wait) for this grid's completion before
    // reading. The trigger comes after the main loop: K2's warps, parked in
    // their wait, would otherwise sit on the SMs for the whole of K1, unevenly
    // when they land while the previous step drains, and slow the SMs they share.
    if (a.early_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = cta_index(a);
    const int64_t A = a.tiles_per_bh;  // static tiles per bh (the pool holds the rest)
    const int64_t x0 = a.x_table ? a.x_table[c] : cta_begin(a.total_tiles, c, a.ctas);
    const int64_t x1 = a.x_table ? a.x_table[c + 1] : cta_begin(a.total_tiles, c + 1, a.ctas);
    const int64_t bh_first = x0 / (A > 0 ? A : 1);
    uint8_t* wsm = smem + size_t(warp) * S * STAGE_BYTES;

    if (lane == 0) {
        if (warp == 0) {
            prefetch_tmap(&tmk);
            prefetch_tmap(&tmv);
        }
        for (int s = 0; s < S; ++s) mbar_init(&bars[warp][s], 1);
        mbar_fence_init();
    }
    __syncwarp();
    const uint64_t pol = policy_evict_first();

    // ---- tile stream (warp-uniform): this CTA's static tiles x0 + warp + kW,
    // then chunks of the pools of the bhs its range covers (dynamic: CTAs on
    // SMs that stream faster take more of them). rec = slot phase (0 static,
    // 1 pool), so pool tiles land in this CTA's own segment slots.
    int64_t s_next = x0 + warp;
    const int64_t nch = a.pool_tiles > 0 ? (a.pool_tiles + a.pool_chunk - 1) / a.pool_chunk : 0;
    const int64_t cb_lo = x1 > x0 ? x0 / A : 0, cb_hi = x1 > x0 ? (x1 - 1) / A : -1;
    const int64_t ncb = cb_hi - cb_lo + 1;
    const int64_t last_static = x1 > x0 + warp ? x0 + warp + ((x1 - 1 - x0 - warp) / W) * W : -1;
    const int64_t cb_start = last_static >= 0 ? last_static / A : cb_hi;  // stay on the current bh first
    int64_t p_bh = -1, p_pos = 0, p_end = 0, p_tries = 0;
    bool p_done = nch == 0 || ncb <= 0 || a.dpool;
    // deterministic chunk pool: after its static tiles a warp takes whole chunks
    // from one grid-wide queue (chunk-major over the rows); a chunk is its own
    // state (fslot (bh, k)), so who computes it does not change the result
    int64_t d_bh = -1, d_pos = 0, d_end = 0;
    int d_k = 0;
    bool d_on = a.dpool && nch > 0;
    // cross-row stealing, once the own rows' pools are empty: the row whose pool
    // has the most chunks left (one coalesced read of the counters), one claimed
    // foreign state per visit; a claimed state that gets no chunk is written empty
    int64_t f_bh = -1, f_pos = 0, f_end = 0;
    int f_slot = 0, f_scans = 0;
    bool f_got = false, f_on = a.fslots > 0 && nch > 0 && !a.dpool;
    uint64_t f_full = 0;  // rows whose foreign states ran out (first 64 rows)
    auto empty_foreign = [&](int64_t bh, int slot) {
        const int64_t fs = (bh * a.fslots + slot) * a.group;
        for (int h = lane; h < a.group; h += 32) {
            a.fslot_m[fs + h] = -CUDART_INF_F;
            a.fslot_l[fs + h] = 0.f;
        }
    };
    auto next_tile = [&](int64_t& bh, int64_t& tb, int& rec) -> bool {
        if (s_next < x1) {
            bh = s_next / A;
            tb = s_next - bh * A;
            rec = 0;
            s_next += W;
            return true;
        }
        while (!p_done) {
            if (p_pos < p_end) {
                bh = p_bh;
                tb = p_pos++;
                rec = 1;
                return true;
            }
            if (p_bh >= 0) {  // next chunk of the bh being helped
                unsigned k = 0;
                if (lane == 0) k = atomicAdd(a.pool_ctr + p_bh, 1u);
                k = __shfl_sync(0xffffffffu, k, 0);
                if (k < nch) {
                    p_pos = a.pool_first + int64_t(k) * a.pool_chunk;
                    p_end = min(p_pos + a.pool_chunk, a.pool_first + a.pool_tiles);
                    continue;
                }
                p_bh = -1;  // exhausted
            }
            if (p_tries == ncb) {
                p_done = true;
                break;
            }
            p_bh = cb_lo + (cb_start - cb_lo + p_tries) % ncb;
            ++p_tries;
        }
        while (f_on) {
            if (f_pos < f_end) {
                bh = f_bh;
                tb = f_pos++;
                rec = 2 + f_slot;
                f_got = true;
                return true;
            }
            if (f_bh >= 0) {  // next chunk of the row being helped
                unsigned k = 0;
                if (lane == 0) k = atomicAdd(a.pool_ctr + f_bh, 1u);
                k = __shfl_sync(0xffffffffu, k, 0);
                if (k < nch) {
                    f_pos = a.pool_first + int64_t(k) * a.pool_chunk;
                    f_end = min(f_pos + a.pool_chunk, a.pool_first + a.pool_tiles);
                    continue;
                }
                if (!f_got) empty_foreign(f_bh, f_slot);
                f_bh = -1;
            }
            if (++f_scans > a.steal_scans) {
                f_on = false;
                break;
            }
            unsigned best_left = 0;
            int64_t best = -1;
            for (int64_t j0 = 0; j0 < a.bh_count; j0 += 32) {
                const int64_t j = j0 + lane;
                unsigned left = 0;
                if (j < a.bh_count && !(j < 64 && ((f_full >> j) & 1ull))) {
                    const unsigned used = *reinterpret_cast<volatile const unsigned*>(a.pool_ctr + j);
                    left = used < unsigned(nch) ? unsigned(nch) - used : 0u;
                }
                unsigned bl = left;
                int64_t bj = j;
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    const unsigned ol = __shfl_xor_sync(0xffffffffu, bl, off);
                    const int64_t oj = __shfl_xor_sync(0xffffffffu, bj, off);
                    if (ol > bl || (ol == bl && oj < bj)) {
                        bl = ol;
                        bj = oj;
                    }
                }
                if (bl > best_left) {
                    best_left = bl;
                    best = bj;
                }
            }
            if (best < 0 || best_left < unsigned(a.steal_min)) {  // the owners drain small remainders
                f_on = false;
                break;
            }
            unsigned fidx = 0;
            if (lane == 0) fidx = atomicAdd(a.fcnt + best, 1u);
            fidx = __shfl_sync(0xffffffffu, fidx, 0);
            if (fidx >= unsigned(a.fslots)) {
                if (best < 64) f_full |= 1ull << best;
                continue;
            }
            f_bh = best;
            f_slot = static_cast<int>(fidx);
            f_got = false;
        }
        while (d_on) {
            if (d_pos < d_end) {
                bh = d_bh;
                tb = d_pos++;
                rec = 2 + d_k;
                return true;
            }
            unsigned j = 0;
            if (lane == 0) j = atomicAdd(a.pool_ctr, 1u);
            j = __shfl_sync(0xffffffffu, j, 0);
            if (int64_t(j) >= nch * a.bh_count) {
                d_on = false;
                break;
            }
            d_k = static_cast<int>(div_nn(j, a.bh_count));
            d_bh = int64_t(j) - int64_t(d_k) * a.bh_count;
            d_pos = a.pool_first + int64_t(d_k) * a.pool_chunk;
            d_end = min(d_pos + a.pool_chunk, a.pool_first + a.pool_tiles);
        }
        return false;
    };
    auto issue = [&](int s, int64_t bh, int64_t tb) {
        if (lane != 0) return;
        const int row = static_cast<int>(bh * a.row_stride + tb * T);
        uint8_t* kd = wsm + size_t(s) * STAGE_BYTES;
        uint8_t* vd = kd + TILE_BYTES;
        mbar_expect_tx(&bars[warp][s], STAGE_BYTES);
#pragma unroll
        for (int bx = 0; bx < BOXES; ++bx) {
            tma_load_2d(kd + bx * BOX_BYTES, &tmk, &bars[warp][s], bx * 64, row, pol);
            tma_load_2d(vd + bx * BOX_BYTES, &tmv, &bars[warp][s], bx * 64, row, pol);
        }
    };
    auto refill = [&](int s) {
        int64_t bh, tb;
        int rec;
        if (next_tile(bh, tb, rec)) {
            if (lane == 0) {
                st_bh[warp][s] = bh;
                st_tb[warp][s] = tb;
                st_rec[warp][s] = rec;
            }
            issue(s, bh, tb);
        } else if (lane == 0) {
            st_bh[warp][s] = -1;
        }
        __syncwarp();
    };
    // this grid is itself a programmatic dependent (launch_pdl): q, the
    // workspace and the pool counters only after the preceding kernel is done.
    // The first static tiles, when they lie wholly inside t_safe tokens (no
    // kernel ahead may be writing them: an append only writes past the last
    // decode's length), are requested before the wait, so HBM streams while
    // the previous step's combine finishes.
    int pre = 0;
    for (; pre < S && a.t_safe > 0 && !a.early_trigger && s_next < x1; ++pre) {
        const int64_t tb = s_next - (s_next / A) * A;
        if ((tb + 1) * T > a.t_safe) break;
        refill(pre);
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    unsigned long long t_go = 0;
    if (a.tl && threadIdx.x == 0) {
        t_go = gtimer();
        atomicMin(a.tl + 0, t_start);
        atomicMin(a.tl + 1, t_go);
    }

    const int hA = 2 * (lane & 3), hB = hA + 1;  // this lane's heads (N columns)
    const int eta = lane >> 2;                   // B-fragment head / C-fragment row
    const int srcA = ((lane & 3) << 3) + (eta >> 1), srcB = srcA + 4;
    const uint32_t sel = (eta & 1) ? 0x7632u : 0x5410u;
    const int r8 = lane & 7, i4 = lane >> 3;

    float o[MD][4];
    float m0 = -CUDART_INF_F, m1 = -CUDART_INF_F, l0 = 0.f, l1 = 0.f;
    uint32_t qf[KS][2];
    int64_t cur_bh = -1, q_bh = -1;
    int cur_rec = -1;
    uint64_t flushed = 0;

    auto load_q = [&](int64_t bh) {
        q_bh = bh;
        const int64_t b = bh / a.n_kv, kvh = bh % a.n_kv;
        const bool ok = eta < a.group;
        const uint16_t* qrow = static_cast<const uint16_t*>(a.q) +
                               ((b * a.n_q) + kvh * a.group + (ok ? eta : 0)) * int64_t(D);
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int col = ks * 16 + 2 * (lane & 3);
            qf[ks][0] = ok ? __ldcg(reinterpret_cast<const unsigned*>(qrow + col)) : 0u;
            qf[ks][1] = ok ? __ldcg(reinterpret_cast<const unsigned*>(qrow + col + 8)) : 0u;
        }
    };
    auto reset = [&]() {
#pragma unroll
        for (int md = 0; md < MD; ++md) o[md][0] = o[md][1] = o[md][2] = o[md][3] = 0.f;
        m0 = m1 = -CUDART_INF_F;
        l0 = l1 = 0.f;
    };
    // every lane's state stores, then the flag (release at gpu scope)
    auto publish = [&](unsigned* f) {
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release_gpu(f, a.sepoch);
    };
    // state -> this warp's slot (c, warp, phase, seg); phase 1 holds pool tiles
    auto flush = [&](int64_t bh, int rec) {
        float la = l0, lb = l1;
        la += __shfl_xor_sync(0xffffffffu, la, 4);
        la += __shfl_xor_sync(0xffffffffu, la, 8);
        la += __shfl_xor_sync(0xffffffffu, la, 16);
        lb += __shfl_xor_sync(0xffffffffu, lb, 4);
        lb += __shfl_xor_sync(0xffffffffu, lb, 8);
        lb += __shfl_xor_sync(0xffffffffu, lb, 16);
        float *sm, *sl, *so;
        if (rec >= 2) {  // a foreign state of row bh (cross-row stealing)
            const int64_t fs = bh * a.fslots + (rec - 2);
            sm = a.fslot_m + fs * a.group;
            sl = a.fslot_l + fs * a.group;
            so = a.fslot_o + fs * a.group * int64_t(D);
        } else {
            const int seg = static_cast<int>(bh - bh_first);
            const int sub = a.slot_warps == W ? warp : 2 * warp + rec;
            const int64_t slot = (int64_t(c) * a.slot_warps + sub) * a.maxseg + seg;
            sm = a.slot_m + slot * a.group;
            sl = a.slot_l + slot * a.group;
            so = a.slot_o + slot * a.group * int64_t(D);
            flushed |= 1ull << (2 * seg + rec);
        }
        if (lane < 4) {
            if (hA < a.group) { sm[hA] = m0; sl[hA] = la; }
            if (hB < a.group) { sm[hB] = m1; sl[hB] = lb; }
        }
#pragma unroll
        for (int md = 0; md < MD; ++md) {
            const int d0 = md * 16 + eta;
            if (hA < a.group) {
                so[hA * D + d0] = o[md][0];
                so[hA * D + d0 + 8] = o[md][2];
            }
            if (hB < a.group) {
                so[hB * D + d0] = o[md][1];
                so[hB * D + d0 + 8] = o[md][3];
            }
        }
        if (a.sflag && rec >= 2) publish(a.sflag + int64_t(a.ctas) * W + bh * a.fslots + (rec - 2));
    };
    // streamed combine: the warp's static part is done -- its untouched static
    // slots become empty partials and the warp's flag is published; the split K2,
    // resident from here on, folds these states while the chunks still stream
    bool s_pub = a.sflag == nullptr;
    auto publish_static = [&]() {
        for (int seg = 0; seg < a.maxseg; ++seg) {
            if (flushed & (1ull << (2 * seg))) continue;
            const int64_t slot = (int64_t(c) * a.slot_warps + warp) * a.maxseg + seg;
            for (int h = lane; h < a.group; h += 32) {
                a.slot_m[slot * a.group + h] = -CUDART_INF_F;
                a.slot_l[slot * a.group + h] = 0.f;
            }
            flushed |= 1ull << (2 * seg);
        }
        if (!((a.reverse & 4) && c == 0 && warp == 0))  // debug (TD_DEBUG_REVERSE=4): one state never published
            publish(a.sflag + int64_t(c) * W + warp);
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        s_pub = true;
    };

    // the first static tile's q before the rest of the first tiles are requested:
    // its load is then not queued behind this CTA's burst of TMA reads
    if (x1 > x0 + warp) load_q((x0 + warp) / A);
    for (int s = pre; s < S; ++s) refill(s);
    reset();
    for (int64_t kk = 0;; ++kk) {
        const int s = static_cast<int>(kk % S);
        const uint32_t phase = static_cast<uint32_t>((kk / S) & 1);
        const int64_t bh = st_bh[warp][s];
        if (bh < 0) break;  // stream exhausted (tiles are consumed in issue order)
        const int64_t tok0 = st_tb[warp][s] * T;
        const int rec = st_rec[warp][s];
        if (bh != cur_bh || rec != cur_rec) {
            if (!s_pub && rec >= 2) {  // the first chunk: the static states are final
                if (cur_bh >= 0) {
                    flush(cur_bh, cur_rec);
                    reset();
                    cur_bh = -1;
                }
                publish_static();
            }
            if (cur_bh >= 0) {
                flush(cur_bh, cur_rec);
                reset();
            }
            if (bh != q_bh) load_q(bh);
            cur_bh = bh;
            cur_rec = rec;
        }
        const int64_t rem = a.t - tok0;
        const int nvalid = rem < T ? static_cast<int>(rem) : T;

        // fused KV append: this tile holds the row's newest token, which is only in
        // the caller's buffers. Its loads are issued before the wait for the tile so
        // their latency hides behind the TMA; after it the token goes into the staged
        // tile (the SWIZZLE_128B layout: 16-byte chunk c of row r sits at chunk
        // c ^ (r & 7) of its 128-byte box row) and into the cache for later steps.
        constexpr int CH = D / 8;                 // 16-byte chunks per row of K (and of V)
        constexpr int PV = (2 * CH + 31) / 32;    // of K|V per lane
        const bool patched = a.app_k && a.app_pos >= tok0 && a.app_pos < tok0 + T;
        uint4 pv[PV];
        if (patched) {
#pragma unroll
            for (int i = 0; i < PV; ++i) {
                const int cc = lane + 32 * i;
                if (cc < 2 * CH)
                    pv[i] = __ldcg(reinterpret_cast<const uint4*>(cc >= CH ? a.app_v : a.app_k) + bh * CH + cc % CH);
            }
        }
        mbar_wait(&bars[warp][s], phase);
        if (patched) {
            const int r = static_cast<int>(a.app_pos - tok0);
#pragma unroll
            for (int i = 0; i < PV; ++i) {
                const int cc = lane + 32 * i;
                if (cc >= 2 * CH) continue;
                const int which = cc / CH, c = cc % CH;
                const uint4 val = pv[i];
                uint8_t* tile = wsm + size_t(s) * STAGE_BYTES + (which ? TILE_BYTES : 0);
                *reinterpret_cast<uint4*>(tile + (c >> 3) * BOX_BYTES + r * 128 + (((c & 7) ^ (r & 7)) << 4)) = val;
                uint4* cache = reinterpret_cast<uint4*>(const_cast<void*>(which ? a.v : a.k));
                cache[(bh * a.row_stride + a.app_pos) * CH + c] = val;
            }
            // generic-proxy writes to a stage the TMA (async proxy) refills later
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
        }
        const uint32_t kb = smem_u32(wsm + size_t(s) * STAGE_BYTES);
        const uint32_t vb = kb + TILE_BYTES;

        // ---- S^T = K . Q^T ------------------------------------------------
        float sc[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) sc[mt][0] = sc[mt][1] = sc[mt][2] = sc[mt][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int bx = (ks * 16) / 64;
            const int chunk = (((ks * 16) % 64) >> 3) + (i4 >> 1);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const int tok = mt * 16 + r8 + (i4 & 1) * 8;
                const uint32_t addr = kb + bx * BOX_BYTES + tok * 128 + ((chunk ^ r8) << 4);
                uint32_t a0, a1, a2, a3;
                ldsm_x4(addr, a0, a1, a2, a3);
                mma_bf16(sc[mt], a0, a1, a2, a3, qf[ks][0], qf[ks][1]);
            }
        }
        // ---- online softmax (log2 domain) -----------------------------------
        float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int tk = mt * 16 + eta;
            sc[mt][0] = tk < nvalid ? sc[mt][0] * a.scale_log2 : -CUDART_INF_F;
            sc[mt][1] = tk < nvalid ? sc[mt][1] * a.scale_log2 : -CUDART_INF_F;
            sc[mt][2] = tk + 8 < nvalid ? sc[mt][2] * a.scale_log2 : -CUDART_INF_F;
            sc[mt][3] = tk + 8 < nvalid ? sc[mt][3] * a.scale_log2 : -CUDART_INF_F;
            mx0 = fmaxf(mx0, fmaxf(sc[mt][0], sc[mt][2]));
            mx1 = fmaxf(mx1, fmaxf(sc[mt][1], sc[mt][3]));
        }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 4));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 8));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 16));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 4));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 8));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 16));
        const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
        const float c0 = fast_exp2(m0 - n0), c1 = fast_exp2(m1 - n1);
        m0 = n0;
        m1 = n1;
        float ps0 = 0.f, ps1 = 0.f;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            sc[mt][0] = fast_exp2(sc[mt][0] - n0);
            sc[mt][1] = fast_exp2(sc[mt][1] - n1);
            sc[mt][2] = fast_exp2(sc[mt][2] - n0);
            sc[mt][3] = fast_exp2(sc[mt][3] - n1);
            ps0 += sc[mt][0] + sc[mt][2];
            ps1 += sc[mt][1] + sc[mt][3];
        }
        l0 = l0 * c0 + ps0;
        l1 = l1 * c1 + ps1;
#pragma unroll
        for (int md = 0; md < MD; ++md) {
            o[md][0] *= c0;
            o[md][1] *= c1;
            o[md][2] *= c0;
            o[md][3] *= c1;
        }
        // ---- P^T as B fragments: hi + lo bf16, transposed with shuffles ------
        uint32_t bh_[MT][2], bl_[MT][2];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const uint32_t h01 = pack_bf16(sc[mt][0], sc[mt][1]);
            const uint32_t h23 = pack_bf16(sc[mt][2], sc[mt][3]);
            const uint32_t g01 = pack_bf16(sc[mt][0] - bf16_lo(h01), sc[mt][1] - bf16_hi(h01));
            const uint32_t g23 = pack_bf16(sc[mt][2] - bf16_lo(h23), sc[mt][3] - bf16_hi(h23));
            uint32_t xa = __shfl_sync(0xffffffffu, h01, srcA), xb = __shfl_sync(0xffffffffu, h01, srcB);
            bh_[mt][0] = __byte_perm(xa, xb, sel);
            xa = __shfl_sync(0xffffffffu, h23, srcA);
            xb = __shfl_sync(0xffffffffu, h23, srcB);
            bh_[mt][1] = __byte_perm(xa, xb, sel);
            xa = __shfl_sync(0xffffffffu, g01, srcA);
            xb = __shfl_sync(0xffffffffu, g01, srcB);
            bl_[mt][0] = __byte_perm(xa, xb, sel);
            xa = __shfl_sync(0xffffffffu, g23, srcA);
            xb = __shfl_sync(0xffffffffu, g23, srcB);
            bl_[mt][1] = __byte_perm(xa, xb, sel);
        }
        // ---- O^T += V^T . P^T ------------------------------------------------
#pragma unroll
        for (int md = 0; md < MD; ++md) {
            const int bx = (md * 16) / 64;
            const int chunk = (((md * 16) % 64) >> 3) + (i4 & 1);
#pragma unroll
            for (int kt = 0; kt < MT; ++kt) {
                const int tok = kt * 16 + r8 + (i4 >> 1) * 8;
                const uint32_t addr = vb + bx * BOX_BYTES + tok * 128 + ((chunk ^ r8) << 4);
                uint32_t a0, a1, a2, a3;
                ldsm_x4_t(addr, a0, a1, a2, a3);
                mma_bf16(o[md], a0, a1, a2, a3, bh_[kt][0], bh_[kt][1]);
                mma_bf16(o[md], a0, a1, a2, a3, bl_[kt][0], bl_[kt][1]);
            }
        }
        __syncwarp();
        refill(s);
    }
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (cur_bh >= 0) flush(cur_bh, cur_rec);
    if (a.sflag) {  // streamed combine: K2 merges the warp states themselves
        if (!s_pub) publish_static();
        if (a.tl && lane == 0) atomicMax(a.tl + 2, gtimer());
        return;
    }
    // untouched slots are empty partials (m = -inf)
    const int phases = a.slot_warps == W ? 1 : 2;
    for (int seg = 0; seg < a.maxseg; ++seg)
        for (int ph = 0; ph < phases; ++ph) {
            if (flushed & (1ull << (2 * seg + ph))) continue;
            const int sub = phases == 1 ? warp : 2 * warp + ph;
            const int64_t slot = (int64_t(c) * a.slot_warps + sub) * a.maxseg + seg;
            for (int h = lane; h < a.group; h += 32) {
                a.slot_m[slot * a.group + h] = -CUDART_INF_F;
                a.slot_l[slot * a.group + h] = 0.f;
            }
        }
    __syncthreads();
    if (phases == 2) cta_merge_batched<2 * W, D, 8>(a, c, reinterpret_cast<float*>(smem));
    else cta_merge_batched<W, D, 8>(a, c, reinterpret_cast<float*>(smem));
    if (a.tl && threadIdx.x == 0) {
        const unsigned long long t_end = gtimer();
        atomicMax(a.tl + 2, t_end);
        if (a.tl_cta && c < 1024) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            a.tl_cta[2048 + c] = smid;
            a.tl_cta[4096 + 2 * c] = t_go;
            a.tl_cta[4097 + 2 * c] = t_end;
        }
    }
    if (a.dbg && threadIdx.x == 0) {
        const unsigned long long t_end = gtimer();
        atomicMin(a.dbg + 0, t_start);
        atomicMax(a.dbg + 1, t_end);
        if (c < 1024) {  // per-CTA [start, end] at dbg[4096 + 2c], SM id at dbg[2048 + c]
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            a.dbg[4096 + 2 * c] = t_start;
            a.dbg[4096 + 2 * c + 1] = t_end;
            a.dbg[2048 + c] = smid;
        }
    }
}

// =========================================================================
// K1, fp32 (d = 128): lane j owns dims [4j, 4j+4); per-warp bulk-copy ring.
// Scores of the 32 tokens of a tile are formed with a butterfly
// reduce-scatter (31 shuffles for 32 tokens) so lane j ends with token j.
// The ring holds E half-tile entries (a K or a V tile of T tokens, 16 KB),
// each with its own mbarrier: half h of the warp's sequence is tile h / 2's
// K (h even) or V (h odd) and lands in entry h % E. A K entry is refilled as
// soon as the scores are formed, before P.V waits for its V.
// =========================================================================
template <int T, int W, int E, int G>
__global__ void __launch_bounds__(W * 32, 1) k1_f32(const K1Args a) {
    constexpr int D = 128;
    // T = 32: lane j ends the reduce-scatter with token j; T = 16: lanes j and j + 16
    // both hold token j (the half-warp butterfly plus one exchange across halves)
    static_assert(T == 32 || T == 16, "32 or 16 tokens per tile");
    static_assert(E >= 2, "a tile's K and V entries are in flight together");
    constexpr int TILE_BYTES = T * D * 4;
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bars[W][E];
    uint8_t* smem = smem_raw + ((128 - (smem_u32(smem_raw) & 127)) & 127);

    const unsigned long long t_start = (a.dbg || a.tl) ? gtimer() : 0ull;
    // PDL: K2 may be scheduled as soon as CTAs of this grid retire; it waits
    // (griddepcontrol.wait) for this grid's completion before reading.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = (a.reverse & 1) ? a.ctas - 1 - static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x);
    const int64_t x0 = a.x_table ? a.x_table[c] : cta_begin(a.total_tiles, c, a.ctas);
    const int64_t x1 = a.x_table ? a.x_table[c + 1] : cta_begin(a.total_tiles, c + 1, a.ctas);
    const int64_t span = x1 - x0;
    const int64_t nmine = span > warp ? (span - warp + W - 1) / W : 0;
    const int64_t bh_first = x0 / (a.tiles_per_bh > 0 ? a.tiles_per_bh : 1);
    const int64_t rows_total = a.bh_count * a.row_stride;
    uint8_t* wsm = smem + size_t(warp) * E * TILE_BYTES;
    const float* kg = static_cast<const float*>(a.k);
    const float* vg = static_cast<const float*>(a.v);

    if (lane == 0) {
        for (int s = 0; s < E; ++s) mbar_init(&bars[warp][s], 1);
        mbar_fence_init();
    }
    __syncwarp();
    // this grid is itself a programmatic dependent: inputs only after the wait
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.tl && threadIdx.x == 0) {
        atomicMin(a.tl + 0, t_start);
        atomicMin(a.tl + 1, gtimer());
    }
    const uint64_t pol = policy_evict_first();
    const int64_t nhalf = 2 * nmine;
    auto issue = [&](int64_t h) {  // half h into entry h % E
        const int64_t x = x0 + warp + (h >> 1) * W;
        const int64_t bh = x / a.tiles_per_bh;
        const int64_t row = bh * a.row_stride + (x - bh * a.tiles_per_bh) * T;
        const int64_t avail = rows_total - row;
        const uint32_t bytes = static_cast<uint32_t>((avail < T ? avail : T) * D * 4);
        const int e = static_cast<int>(h % E);
        mbar_expect_tx(&bars[warp][e], bytes);
        bulk_load(wsm + size_t(e) * TILE_BYTES, ((h & 1) ? vg : kg) + row * D, bytes, &bars[warp][e], pol);
    };
    auto wait_half = [&](int64_t h) {
        mbar_wait(&bars[warp][static_cast<int>(h % E)], static_cast<uint32_t>((h / E) & 1));
        return reinterpret_cast<const float*>(wsm + size_t(h % E) * TILE_BYTES);
    };
    float qv[G][4], o[G][4], m[G], l[G];
    int64_t cur_bh = -1;
    uint32_t flushed = 0;
    auto load_q = [&](int64_t bh) {
        const int64_t b = bh / a.n_kv, kvh = bh % a.n_kv;
#pragma unroll
        for (int h = 0; h < G; ++h) {
            const float4 qq = __ldcg(reinterpret_cast<const float4*>(
                static_cast<const float*>(a.q) + ((b * a.n_q) + kvh * G + h) * int64_t(D)) + lane);
            // raw q: no arithmetic on the loaded value here, so the warp does not
            // wait for it before issuing its first bulk copies (the scale is applied
            // to the reduced score instead)
            qv[h][0] = qq.x;
            qv[h][1] = qq.y;
            qv[h][2] = qq.z;
            qv[h][3] = qq.w;
        }
    };
    auto reset = [&]() {
#pragma unroll
        for (int h = 0; h < G; ++h) {
            o[h][0] = o[h][1] = o[h][2] = o[h][3] = 0.f;
            m[h] = -CUDART_INF_F;
            l[h] = 0.f;
        }
    };
    auto flush = [&](int seg) {
        const int64_t slot = (int64_t(c) * W + warp) * a.maxseg + seg;
#pragma unroll
        for (int h = 0; h < G; ++h) {
            float lt = l[h];
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) lt += __shfl_xor_sync(0xffffffffu, lt, off);
            if (lane == 0) {
                a.slot_m[slot * G + h] = m[h];
                a.slot_l[slot * G + h] = lt;
            }
            reinterpret_cast<float4*>(a.slot_o + (slot * G + h) * int64_t(D))[lane] =
                make_float4(o[h][0], o[h][1], o[h][2], o[h][3]);
        }
        flushed |= 1u << seg;
    };

    reset();
    // the first tile's q before this warp's bulk copies: its load is then not
    // queued behind the CTA's burst of KV reads (it misses L2 after a flush)
    if (nmine > 0) {
        cur_bh = (x0 + warp) / a.tiles_per_bh;
        load_q(cur_bh);
    }
    if (lane == 0)
        for (int64_t h = 0; h < E && h < nhalf; ++h) issue(h);
    for (int64_t kk = 0; kk < nmine; ++kk) {
        const int64_t x = x0 + warp + kk * W;
        const int64_t bh = x / a.tiles_per_bh;
        const int64_t tok0 = (x - bh * a.tiles_per_bh) * T;
        if (bh != cur_bh) {
            if (cur_bh >= 0) {
                flush(static_cast<int>(cur_bh - bh_first));
                reset();
            }
            cur_bh = bh;
            load_q(bh);
        }
        const int64_t rem = a.t - tok0;
        const int nvalid = rem < T ? static_cast<int>(rem) : T;
        const float* ks_ = wait_half(2 * kk);
        if (a.reverse & 2) {  // debug (TD_DEBUG_REVERSE=2): no math, the stream alone
            wait_half(2 * kk + 1);
            __syncwarp();
            if (lane == 0 && 2 * kk + E < nhalf) issue(2 * kk + E);
            if (lane == 0 && 2 * kk + 1 + E < nhalf) issue(2 * kk + 1 + E);
            continue;
        }

        float sc[G];
#pragma unroll
        for (int h = 0; h < G; ++h) {
            float part[T];
#pragma unroll
            for (int tk = 0; tk < T; ++tk) {
                const float4 kk4 = reinterpret_cast<const float4*>(ks_ + tk * D)[lane];
                part[tk] = qv[h][0] * kk4.x + qv[h][1] * kk4.y + qv[h][2] * kk4.z + qv[h][3] * kk4.w;
            }
            // reduce-scatter: after step k, lane bit k selects the kept half
#pragma unroll
            for (int k = T / 2; k >= 1; k >>= 1) {
                const bool up = (lane & k) != 0;
#pragma unroll
                for (int i = 0; i < k; ++i) {
                    const float send = up ? part[i] : part[i + k];
                    const float keep = up ? part[i + k] : part[i];
                    part[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
                }
            }
            if (T == 16) part[0] += __shfl_xor_sync(0xffffffffu, part[0], 16);  // the other half-warp's dims
            sc[h] = (lane % T) < nvalid ? part[0] * a.scale_log2 : -CUDART_INF_F;
        }
        float p[G];
#pragma unroll
        for (int h = 0; h < G; ++h) {
            float mx = sc[h];
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            const float mn = fmaxf(m[h], mx);
            const float cr = fast_exp2(m[h] - mn);
            m[h] = mn;
            p[h] = fast_exp2(sc[h] - mn);
            l[h] = l[h] * cr + (lane < T ? p[h] : 0.f);  // (T = 16: each token's p sits on two lanes)
            o[h][0] *= cr;
            o[h][1] *= cr;
            o[h][2] *= cr;
            o[h][3] *= cr;
        }
        __syncwarp();  // every lane has read the K entry
        if (lane == 0 && 2 * kk + E < nhalf) issue(2 * kk + E);
        const float* vs_ = wait_half(2 * kk + 1);
#pragma unroll 8
        for (int tk = 0; tk < nvalid; ++tk) {
            const float4 vv = reinterpret_cast<const float4*>(vs_ + tk * D)[lane];
#pragma unroll
            for (int h = 0; h < G; ++h) {
                const float pt = __shfl_sync(0xffffffffu, p[h], tk);
                o[h][0] += pt * vv.x;
                o[h][1] += pt * vv.y;
                o[h][2] += pt * vv.z;
                o[h][3] += pt * vv.w;
            }
        }
        __syncwarp();
        if (lane == 0 && 2 * kk + 1 + E < nhalf) issue(2 * kk + 1 + E);
    }
    if (cur_bh >= 0) flush(static_cast<int>(cur_bh - bh_first));
    for (int seg = 0; seg < a.maxseg; ++seg) {
        if (flushed & (1u << seg)) continue;
        const int64_t slot = (int64_t(c) * W + warp) * a.maxseg + seg;
        if (lane < G) {
            a.slot_m[slot * G + lane] = -CUDART_INF_F;
            a.slot_l[slot * G + lane] = 0.f;
        }
    }
    __syncthreads();
    cta_merge_batched<W, D, 8>(a, c, reinterpret_cast<float*>(smem));
    if (a.tl && threadIdx.x == 0) atomicMax(a.tl + 2, gtimer());
    if (a.dbg && threadIdx.x == 0) {
        const unsigned long long t_end = gtimer();
        atomicMin(a.dbg + 0, t_start);
        atomicMax(a.dbg + 1, t_end);
        if (c < 1024) {  // per-CTA [start, end] at dbg[4096 + 2c], SM id at dbg[2048 + c]
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            a.dbg[4096 + 2 * c] = t_start;
            a.dbg[4096 + 2 * c + 1] = t_end;
            a.dbg[2048 + c] = smid;
        }
    }
}

// =========================================================================
// K1, generic: any d <= 256, bf16 or fp32, any group; one head at a time,
// 32 tokens per tile (lane = token for scores, lane = dim for P.V).
// =========================================================================
template <typename TIn>
__device__ __forceinline__ float to_f(TIn x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename TIn>
__global__ void __launch_bounds__(128) k1_generic(const K1Args a) {
    constexpr int T = 32;
    constexpr int W = 4;
    extern __shared__ float gen_smem[];
    const unsigned long long t_start = a.dbg ? gtimer() : 0ull;
    // PDL: K2 may be scheduled as soon as CTAs of this grid retire; it waits
    // (griddepcontrol.wait) for this grid's completion before reading.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // this grid is itself a programmatic dependent: inputs only after the wait
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = (a.reverse & 1) ? a.ctas - 1 - static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x);
    const int64_t x0 = a.x_table ? a.x_table[c] : cta_begin(a.total_tiles, c, a.ctas);
    const int64_t x1 = a.x_table ? a.x_table[c + 1] : cta_begin(a.total_tiles, c + 1, a.ctas);
    const int64_t span = x1 - x0;
    const int64_t nmine = span > warp ? (span - warp + W - 1) / W : 0;
    const int64_t bh_first = x0 / (a.tiles_per_bh > 0 ? a.tiles_per_bh : 1);
    const TIn* q = static_cast<const TIn*>(a.q);
    const TIn* kg = static_cast<const TIn*>(a.k);
    const TIn* vg = static_cast<const TIn*>(a.v);
    const int D = a.d;
    const int nd = (D + 31) / 32;

    for (int h = 0; h < a.group; ++h) {
        float o[8], m = -CUDART_INF_F, l = 0.f;
        for (int i = 0; i < 8; ++i) o[i] = 0.f;
        int64_t cur_bh = -1;
        uint32_t flushed = 0;
        const TIn* qrow = nullptr;
        const TIn* srow = nullptr;
        auto flush = [&](int seg) {
            float lt = l;
            for (int off = 16; off >= 1; off >>= 1) lt += __shfl_xor_sync(0xffffffffu, lt, off);
            const int64_t slot = (int64_t(c) * W + warp) * a.maxseg + seg;
            if (lane == 0) {
                a.slot_m[slot * a.group + h] = m;
                a.slot_l[slot * a.group + h] = lt;
            }
            for (int i = 0; i < nd; ++i) {
                const int j = lane + 32 * i;
                if (j < D) a.slot_o[(slot * a.group + h) * D + j] = o[i];
            }
            flushed |= 1u << seg;
        };
        for (int64_t kk = 0; kk < nmine; ++kk) {
            const int64_t x = x0 + warp + kk * W;
            const int64_t bh = x / a.tiles_per_bh;
            const int64_t tok0 = (x - bh * a.tiles_per_bh) * T;
            if (bh != cur_bh) {
                if (cur_bh >= 0) {
                    flush(static_cast<int>(cur_bh - bh_first));
                    m = -CUDART_INF_F;
                    l = 0.f;
                    for (int i = 0; i < 8; ++i) o[i] = 0.f;
                }
                cur_bh = bh;
                const int64_t b = bh / a.n_kv, kvh = bh % a.n_kv;
                qrow = q + (b * a.n_q + kvh * a.group + h) * int64_t(D);
                if (a.src) srow = static_cast<const TIn*>(a.src) + (b * a.n_q + kvh * a.group + h) * int64_t(D);
            }
            const int64_t rem = a.t - tok0;
            const int nvalid = rem < T ? static_cast<int>(rem) : T;
            const int64_t row0 = bh * a.row_stride + tok0;
            float s = -CUDART_INF_F;
            if (lane < nvalid) {
                // fp32 inputs: the dot in double, so the score carries only the
                // fp32 rounding of the reference's Float32 mode (energy stats are
                // log-domain values judged to 1e-5 absolute)
                using Acc = typename std::conditional<std::is_same<TIn, float>::value, double, float>::type;
                const TIn* kr = kg + (row0 + lane) * D;
                Acc acc = 0;
                for (int j = 0; j < D; ++j) acc += Acc(to_f(qrow[j])) * Acc(to_f(kr[j]));
                if (srow) {  // energy source (energy.cpp:27-47): + source . v_a
                    const TIn* vr = vg + (row0 + lane) * D;
                    for (int j = 0; j < D; ++j) acc += Acc(to_f(srow[j])) * Acc(to_f(vr[j]));
                }
                s = static_cast<float>(acc) * a.scale_log2;
            }
            float mx = s;
            for (int off = 16; off >= 1; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            const float mn = fmaxf(m, mx);
            const float cr = fast_exp2(m - mn);
            m = mn;
            const float p = fast_exp2(s - mn);
            l = l * cr + p;
            for (int i = 0; i < nd; ++i) o[i] *= cr;
            for (int tk = 0; tk < nvalid; ++tk) {
                const float pt = __shfl_sync(0xffffffffu, p, tk);
                const TIn* vr = vg + (row0 + tk) * D;
                for (int i = 0; i < nd; ++i) {
                    const int j = lane + 32 * i;
                    if (j < D) o[i] += pt * to_f(vr[j]);
                }
            }
        }
        if (cur_bh >= 0) flush(static_cast<int>(cur_bh - bh_first));
        for (int seg = 0; seg < a.maxseg; ++seg) {
            if (flushed & (1u << seg)) continue;
            const int64_t slot = (int64_t(c) * W + warp) * a.maxseg + seg;
            if (lane == 0) {
                a.slot_m[slot * a.group + h] = -CUDART_INF_F;
                a.slot_l[slot * a.group + h] = 0.f;
            }
        }
    }
    __syncthreads();
    cta_merge<W>(a, c, gen_smem);
}

// =========================================================================
// K2: merge the split states of one (b, q-head) row into the shard's
// partial: out = O/L, lse = (M + log2 L) ln 2, row_max = M ln 2. Empty
// rows give the identity (-inf, -inf, 0), like attention_chunk_partial on
// an empty chunk (attention.cpp:56-61). One block of K2_THREADS per row;
// warps stride over the candidate (cta, warp) slots.
// =========================================================================
constexpr int K2_THREADS = 128;  // at most 4 warps (= 4 output rows at a time) per block

// The CTA states covering one bh: CTAs c_lo .. c_lo + S - 1; the first one
// holds bh in its segment seg_lo, the others in segment 0. Reads only
// host-written tables, so K2 computes it before griddepcontrol.wait.
struct Cover {
    int64_t c_lo = 0, seg_lo = 0;
    int S = 0;
    int nf = 0;  // foreign states (cross-row stealing) of the row's bh: set after the wait
};
// The foreign states K1 claimed for bh (read after griddepcontrol.wait).
__device__ __forceinline__ int foreign_of(const K1Args& a, int64_t bh) {
    if (a.dpool) return a.fslots;  // every chunk of the deterministic pool has its state
    if (a.fslots <= 0 || !a.fcnt) return 0;
    const unsigned n = __ldcg(a.fcnt + bh);
    return static_cast<int>(n < unsigned(a.fslots) ? n : unsigned(a.fslots));
}
__device__ __forceinline__ Cover cover_of(const K1Args& a, int64_t bh) {
    Cover cv;
    int64_t c_hi = -1;
    if (a.bh_table) {
        cv.c_lo = __ldg(a.bh_table + 3 * bh);
        c_hi = __ldg(a.bh_table + 3 * bh + 1);
        cv.seg_lo = __ldg(a.bh_table + 3 * bh + 2);
    } else if (a.tiles_per_bh > 0 && a.total_tiles > 0) {
        const int64_t X = bh * a.tiles_per_bh, Xe = X + a.tiles_per_bh - 1;
        cv.c_lo = div_nn((X + 1) * a.ctas + a.total_tiles - 1, a.total_tiles) - 1;
        c_hi = div_nn((Xe + 1) * a.ctas + a.total_tiles - 1, a.total_tiles) - 1;
        cv.seg_lo = bh - div_nn(cta_begin(a.total_tiles, static_cast<int>(cv.c_lo), a.ctas), a.tiles_per_bh);
    }
    cv.S = static_cast<int>(c_hi - cv.c_lo + 1);
    return cv;
}

// Lane columns of a row of D floats: chunk c, element v is column
// (c * 32 + lane) * V + v (V = 4: float4 loads).
template <int V, int NC>
struct LaneRow {
    float v[NC][V];
};

// Merges the CTA states of row r into the lane's columns and returns
// (lse, row_max) in natural log units; one warp per row, no shared memory,
// no barrier. Every lane loads the (m, l, o-columns) of BO candidates at
// once -- m and l are broadcast loads -- so a row with S <= BO candidates
// costs a single L2 round trip; M is the max over the candidates already in
// registers (a lane-parallel pass + shuffles only when S > BO).
template <int V, int NC, int BO>
__device__ __forceinline__ void merge_row_warp(const K1Args& a, int64_t r, const Cover& cv, LaneRow<V, NC>& res,
                                               float& lse_o, float& rmax_o, int colb = 0) {
    using vec = typename std::conditional<V == 4, float4, float>::type;
    static_assert(BO <= 32, "one candidate (m, l) per lane");
    const int lane = threadIdx.x & 31;
    const int h = static_cast<int>(r % a.group);
    const int D = a.d, g = a.group, S = cv.S, T = cv.S + cv.nf;
    auto cs_of = [&](int i) { return (cv.c_lo + i) * a.maxseg + (i == 0 ? cv.seg_lo : 0); };
    // 32-bit float offsets (the state arrays are small): static candidate i >= 1 sits
    // at a fixed stride from candidate 1, candidate 0 has its own segment; candidates
    // i >= S are the row's foreign states (cross-row stealing), stride g
    const int st = a.maxseg * g;
    const int b0 = static_cast<int>(cs_of(0) * g + h), b1 = static_cast<int>(cs_of(1) * g + h);
    const int fb = static_cast<int>((r / g) * a.fslots * g + h);
    const int col0 = colb + lane * V;  // colb: first column of this warp's share of the row
    auto off_of = [&](int i) { return i >= S ? fb + (i - S) * g : (i == 0 ? b0 : b1 + (i - 1) * st); };
    vec ov[BO][NC];
    if (cv.nf == 0 && T >= 2 && T <= BO) {
        // one batch of static candidates (the common case), branch-free: the o
        // load of slot u reads candidate min(u, T - 1) -- slots past T repeat
        // the last candidate with weight 0 -- at a fixed stride from candidate
        // 1, so each load is one independent address op for the single warp
        float ml1 = -CUDART_INF_F, ll1 = 0.f;
        if (lane < T) {
            const int off = lane == 0 ? b0 : b1 + (lane - 1) * st;
            ml1 = __ldcg(a.cslot_m + off);
            ll1 = __ldcg(a.cslot_l + off);
        }
        const float* p0 = a.cslot_o + size_t(b0) * D + col0;
        const float* p1 = a.cslot_o + size_t(b1) * D + col0;
        const int64_t sD = int64_t(st) * D;
        bool colok[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) colok[c] = col0 + c * 32 * V < D;
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (colok[c]) ov[0][c] = __ldcg(reinterpret_cast<const vec*>(p0 + c * 32 * V));
#pragma unroll
        for (int u = 1; u < BO; ++u) {
            const float* src = p1 + int64_t(min(u, T - 1) - 1) * sD;
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if (colok[c]) ov[u][c] = __ldcg(reinterpret_cast<const vec*>(src + c * 32 * V));
        }
        float M = ml1;
#pragma unroll
        for (int o2 = 16; o2 >= 1; o2 >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o2));
        const float e_l = ml1 == -CUDART_INF_F ? 0.f : fast_exp2(ml1 - M);
        float L = e_l * ll1;
#pragma unroll
        for (int o2 = 16; o2 >= 1; o2 >>= 1) L += __shfl_xor_sync(0xffffffffu, L, o2);
        float acc[NC][V];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < V; ++v) acc[c][v] = 0.f;
#pragma unroll
        for (int u = 0; u < BO; ++u) {
            const float e = __shfl_sync(0xffffffffu, e_l, u);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const float* o = reinterpret_cast<const float*>(&ov[u][c]);
#pragma unroll
                for (int v = 0; v < V; ++v) acc[c][v] = fmaf(e, colok[c] ? o[v] : 0.f, acc[c][v]);
            }
        }
        const bool empty = M == -CUDART_INF_F;
        const float inv = empty ? 0.f : 1.f / L;
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < V; ++v) res.v[c][v] = acc[c][v] * inv;
        lse_o = empty ? -CUDART_INF_F : (M + log2f(L)) * kLn2;
        rmax_o = empty ? -CUDART_INF_F : M * kLn2;
        return;
    }
    // General path (foreign states, or more than BO candidates): an online merge over
    // batches of BO candidates -- lane i holds (m, l) of the batch's candidate i, every
    // lane the o columns of all of them. When the registers allow two batches, the next
    // batch's loads are issued before the current one is combined, so T candidates cost
    // about one L2 round trip plus the issue of T / BO batches.
    if (T <= 0) {  // no state covers the row (an empty shard): the identity
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < V; ++v) res.v[c][v] = 0.f;
        lse_o = rmax_o = -CUDART_INF_F;
        return;
    }
    constexpr int NB = (V * NC * BO <= 64) ? 2 : 1;
    vec ob[NB][BO][NC];
    float mlb[NB], llb[NB];
    auto load = [&](int i0, auto bufc) {
        constexpr int b = decltype(bufc)::value;
        {
            const int i = i0 + lane;
            mlb[b] = -CUDART_INF_F;
            llb[b] = 0.f;
            if (lane < BO && i < T) {
                const int off = off_of(i);
                mlb[b] = __ldcg((i >= S ? a.fslot_m : a.cslot_m) + off);
                llb[b] = __ldcg((i >= S ? a.fslot_l : a.cslot_l) + off);
            }
        }
#pragma unroll
        for (int u = 0; u < BO; ++u) {
            const int i = i0 + u;
            const int off = off_of(i < T ? i : T - 1);
            const float* obase = (i < T ? i : T - 1) >= S ? a.fslot_o : a.cslot_o;
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if (col0 + c * 32 * V < D)
                    ob[b][u][c] = __ldcg(reinterpret_cast<const vec*>(obase + off * D + col0 + c * 32 * V));
        }
    };
    float M = -CUDART_INF_F, L = 0.f, acc[NC][V];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[c][v] = 0.f;
    auto combine = [&](int i0, auto bufc) {
        constexpr int b = decltype(bufc)::value;
        const float ml = mlb[b], ll = llb[b];
        float Mb = ml;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) Mb = fmaxf(Mb, __shfl_xor_sync(0xffffffffu, Mb, off));
        const float Mn = fmaxf(M, Mb);
        const float cs = M == -CUDART_INF_F ? 0.f : fast_exp2(M - Mn);  // rescale what is merged so far
        L *= cs;
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < V; ++v) acc[c][v] *= cs;
        const float e_l = ml == -CUDART_INF_F ? 0.f : fast_exp2(ml - Mn);
        float lsum = e_l * ll;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, off);
        L += lsum;
#pragma unroll
        for (int u = 0; u < BO; ++u) {
            const float e = __shfl_sync(0xffffffffu, e_l, u);  // 0 past the last candidate
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const float* o = reinterpret_cast<const float*>(&ob[b][u][c]);
#pragma unroll
                for (int v = 0; v < V; ++v)  // an empty state's o is never read as a value (it may be stale)
                    acc[c][v] = fmaf(e, e != 0.f ? o[v] : 0.f, acc[c][v]);
            }
        }
        M = Mn;
    };
    using B0 = std::integral_constant<int, 0>;
    if constexpr (NB == 2) {
        using B1 = std::integral_constant<int, 1>;
        load(0, B0{});
        for (int i0 = 0; i0 < T; i0 += 2 * BO) {
            if (i0 + BO < T) load(i0 + BO, B1{});
            combine(i0, B0{});
            if (i0 + BO >= T) break;
            if (i0 + 2 * BO < T) load(i0 + 2 * BO, B0{});
            combine(i0 + BO, B1{});
        }
    } else {
        for (int i0 = 0; i0 < T; i0 += BO) {
            load(i0, B0{});
            combine(i0, B0{});
        }
    }
    const bool empty = M == -CUDART_INF_F;
    const float inv = empty ? 0.f : 1.f / L;
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int v = 0; v < V; ++v) res.v[c][v] = acc[c][v] * inv;
    lse_o = empty ? -CUDART_INF_F : (M + log2f(L)) * kLn2;
    rmax_o = empty ? -CUDART_INF_F : M * kLn2;
}

template <int V, int NC>
__device__ __forceinline__ void store_row(float* dst, int D, const LaneRow<V, NC>& res, int colb = 0) {
    using vec = typename std::conditional<V == 4, float4, float>::type;
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int col = colb + (c * 32 + lane) * V;
        if (col < D) *reinterpret_cast<vec*>(dst + col) = *reinterpret_cast<const vec*>(res.v[c]);
    }
}

__device__ __forceinline__ int64_t out_row_of(const K1Args& a, int64_t r) {
    const int64_t bh = r / a.group, h = r % a.group;
    return (bh / a.n_kv) * a.n_q + (bh % a.n_kv) * a.group + h;
}

// =========================================================================
// K2 (launched with programmatic dependent launch: its blocks are scheduled
// as K1's CTAs retire and wait in griddepcontrol.wait, so the kernel
// boundary costs no launch latency). Warp w of the grid merges rows
// r = w, w + warps, ... of the shard (merge_row_warp over the CTA states) and,
// per a.tail.mode:
//   kTailPartial  row_max / lse / out of the shard -- attention_chunk_partial
//                 (attention.cpp:146-168), combine_partials across CTAs
//                 (attention.cpp:207-241)
//   kTailFinal    out only (p = 1: the partial is the decode result)
// =========================================================================
template <int V, int NC, int BO>
__global__ void __launch_bounds__(K2_THREADS) k2_combine(const K1Args a) {
    const unsigned long long t_pre = a.dbg ? gtimer() : 0ull;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next step's K1 may get resident
    const int64_t rows = a.bh_count * a.group;
    const int64_t w0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    // host-written tables only: overlaps K1's tail
    const Cover cv0 = w0 < rows ? cover_of(a, w0 / a.group) : Cover{};
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // the other parity's pool counters are the next launch's: zero them
    if (a.pool_tiles > 0)
        for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.bh_count;
             i += int64_t(gridDim.x) * blockDim.x) {
            a.pool_next[i] = 0u;
            if (a.fcnt_next) a.fcnt_next[i] = 0u;
        }
    unsigned long long* ts = (a.dbg && w0 < 512 && (threadIdx.x & 31) == 0) ? a.dbg + 8 + 8 * w0 : nullptr;
    if (ts) {
        ts[0] = gtimer();
        ts[3] = t_pre;
    }
    const Tail& t = a.tail;
    for (int64_t r = w0; r < rows; r += nw) {
        const int64_t orow = out_row_of(a, r);
        float l, m;
        LaneRow<V, NC> res;
        Cover cv = r == w0 ? cv0 : cover_of(a, r / a.group);
        cv.nf = foreign_of(a, r / a.group);
        if (ts && r == w0) {  // debug: one candidate load's round trip
            const float pv = __ldcg(a.cslot_m + (cv.c_lo * a.maxseg + cv.seg_lo) * a.group);
            if (pv == 1.2345e-30f) ts[5] = 1;
            ts[1] = gtimer();
        }
        merge_row_warp<V, NC, BO>(a, r, cv, res, l, m);
        store_row(t.out + orow * a.d, a.d, res);
        if (ts && r == w0) ts[2] = gtimer();
        if (t.mode == kTailPartial && (threadIdx.x & 31) == 0) {
            t.lse[orow] = l;
            t.row_max[orow] = m;
        }
    }
    if (ts) ts[4] = gtimer();
    if (a.tl && (threadIdx.x & 31) == 0) atomicMax(a.tl + 3, gtimer());
    signal_done(a);
}

// K2 with each row split by columns over Q warps (d = 32 Q, one float per
// lane): a warp loads one 128-byte line per candidate instead of Q, so the
// merge's loads of a row spread over Q SMs. Same results as k2_combine (the
// per-column arithmetic is identical).
template <int Q>
__global__ void __launch_bounds__(K2_THREADS) k2_combine_cols(const K1Args a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next step's K1 may get resident
    const int64_t rows = a.bh_count * a.group, units = rows * Q;
    const int64_t u0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const Cover cv0 = u0 < units ? cover_of(a, (u0 / Q) / a.group) : Cover{};  // host-written tables only
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.pool_tiles > 0)
        for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.bh_count;
             i += int64_t(gridDim.x) * blockDim.x) {
            a.pool_next[i] = 0u;
            if (a.fcnt_next) a.fcnt_next[i] = 0u;
        }
    const Tail& t = a.tail;
    for (int64_t u = u0; u < units; u += nw) {
        const int64_t r = u / Q;
        const int colb = static_cast<int>(u % Q) * 32;
        const int64_t orow = out_row_of(a, r);
        float l, m;
        LaneRow<1, 1> res;
        Cover cv = u == u0 ? cv0 : cover_of(a, r / a.group);
        cv.nf = foreign_of(a, r / a.group);
        merge_row_warp<1, 1, 32>(a, r, cv, res, l, m, colb);
        store_row(t.out + orow * a.d, a.d, res, colb);
        if (t.mode == kTailPartial && colb == 0 && (threadIdx.x & 31) == 0) {
            t.lse[orow] = l;
            t.row_max[orow] = m;
        }
    }
    if (a.tl && (threadIdx.x & 31) == 0) atomicMax(a.tl + 3, gtimer());
    signal_done(a);
}

// K2 for rows with many candidate states (few (b, kv-head) rows over many CTAs,
// e.g. cfg1's single row merges ~148 CTA states): each (row, column quarter)
// gets a block of WS warps that split the candidates -- each warp merges its
// share (at most 32 per L2 round trip) into an unnormalised (M, L, o) -- and warp
// 0 combines the WS partials from shared memory. One warp walking 148
// candidates took ~7 us; this takes about one round trip per warp plus the
// shared-memory combine. Same arithmetic per column as k2_combine_cols.
// ---- streamed combine (K1Args::sflag) --------------------------------------
// Waits until every lane's candidate flag (idx >= 0) carries this launch's
// epoch; bounded (~1 s of clocks, then *err if given) so a missing state cannot
// hang the GPU. Afterwards every lane may read every lane's candidate.
__device__ __forceinline__ void wait_flags(const unsigned* f, int idx, unsigned ep, int spin, int* err) {
    const long long t0 = clock64();
    for (;;) {
        const bool ok = idx < 0 || ld_acquire_gpu(f + idx) == ep;
        if (__all_sync(0xffffffffu, ok)) break;
        if (clock64() - t0 > (1ll << 31)) {
            if (err) *reinterpret_cast<volatile int*>(err) = 1;
            break;
        }
        __nanosleep(spin);
    }
    __syncwarp();
    __threadfence();  // the states behind every lane's flag, for every lane
}

// One online-softmax fold of n <= NB candidate states into the warp's running
// (M, L, acc) of column col: lane i < n holds candidate i's element offset.
// The loads of all n states are issued before any is used (one L2 round trip).
template <int NB>
__device__ __forceinline__ void fold_batch(const float* bm, const float* bl, const float* bo, int off, int n,
                                           int col, int D, float& M, float& L, float& acc) {
    const int lane = threadIdx.x & 31;
    float ml = -CUDART_INF_F, ll = 0.f;
    if (lane < n) {
        ml = __ldcg(bm + off);
        ll = __ldcg(bl + off);
    }
    float ov[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const int ok = __shfl_sync(0xffffffffu, off, k);
        ov[k] = (k < n && col < D) ? __ldcg(bo + int64_t(ok) * D + col) : 0.f;
    }
    float Mb = ml;
#pragma unroll
    for (int o2 = 16; o2 >= 1; o2 >>= 1) Mb = fmaxf(Mb, __shfl_xor_sync(0xffffffffu, Mb, o2));
    const float Mn = fmaxf(M, Mb);
    const float cs = M == -CUDART_INF_F ? 0.f : fast_exp2(M - Mn);
    L *= cs;
    acc *= cs;
    const float e_l = ml == -CUDART_INF_F ? 0.f : fast_exp2(ml - Mn);
    float ls = e_l * ll;
#pragma unroll
    for (int o2 = 16; o2 >= 1; o2 >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o2);
    L += ls;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const float e = __shfl_sync(0xffffffffu, e_l, k);
        acc = fmaf(e, e != 0.f ? ov[k] : 0.f, acc);
    }
    M = Mn;
}

__device__ __forceinline__ void fold_any(const float* bm, const float* bl, const float* bo, int off, int n, int col,
                                         int D, float& M, float& L, float& acc) {
    if (n <= 8) fold_batch<8>(bm, bl, bo, off, n, col, D, M, L, acc);
    else if (n <= 16) fold_batch<16>(bm, bl, bo, off, n, col, D, M, L, acc);
    else fold_batch<32>(bm, bl, bo, off, n, col, D, M, L, acc);
}

// Warp `warp` of a split K2 block folds its share of row r's candidates as K1
// publishes them: the static warp states (CTAs c_lo.. of the cover, every warp;
// segment seg_lo in the first CTA, 0 after) in contiguous shares, then the chunk
// states k = warp, warp + WS, ... (the grid-wide queue completes chunks in about
// k order, so the last ones spread over the warps). The assignment and the order
// are fixed: results stay bitwise reproducible.
template <int WS>
__device__ __forceinline__ void stream_fold(const K1Args& a, int64_t r, const Cover& cv, int col, float& M,
                                            float& L, float& acc, int* err) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = a.group, W = a.slot_warps, D = a.d;
    const int h = static_cast<int>(r % g);
    const int64_t bh = r / g;
    const int ns = cv.S * W;
    const int s_lo = ns * warp / WS, s_hi = ns * (warp + 1) / WS;
    for (int i0 = s_lo; i0 < s_hi; i0 += 32) {
        const int n = min(32, s_hi - i0);
        int off = 0, fi = -1;
        if (lane < n) {
            const int i = i0 + lane, cw = i / W;
            const int64_t cc = cv.c_lo + cw;
            const int64_t slot = (cc * W + (i - cw * W)) * a.maxseg + (cw == 0 ? cv.seg_lo : 0);
            off = static_cast<int>(slot * g + h);
            fi = static_cast<int>(cc * W + (i - cw * W));
        }
        wait_flags(a.sflag, fi, a.sepoch, a.sspin, err);
        fold_any(a.slot_m, a.slot_l, a.slot_o, off, n, col, D, M, L, acc);
    }
    const int nf = cv.nf;
    const int nc = nf > warp ? (nf - warp + WS - 1) / WS : 0;
    for (int j0 = 0; j0 < nc; j0 += 32) {
        const int n = min(32, nc - j0);
        int off = 0, fi = -1;
        if (lane < n) {
            const int64_t fs = bh * a.fslots + warp + int64_t(j0 + lane) * WS;
            off = static_cast<int>(fs * g + h);
            fi = static_cast<int>(int64_t(a.ctas) * W + fs);
        }
        wait_flags(a.sflag, fi, a.sepoch, a.sspin, err);
        fold_any(a.fslot_m, a.fslot_l, a.fslot_o, off, n, col, D, M, L, acc);
    }
}

template <int Q, int WS, bool SF = false>
__global__ void __launch_bounds__(32 * WS) k2_combine_split(const K1Args a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    __shared__ float sm_m[WS], sm_l[WS], sm_o[WS][32];
    const int64_t rows = a.bh_count * a.group, units = rows * Q;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Cover cv0 = blockIdx.x < units ? cover_of(a, (int64_t(blockIdx.x) / Q) / a.group) : Cover{};
    // streamed combine: no grid-completion wait before the merge (the states are
    // awaited one by one); the other parity's counters were last used by the
    // previous K1, which completed before this grid's K1 passed its own wait
    if constexpr (!SF) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.pool_tiles > 0)
        for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.bh_count;
             i += int64_t(gridDim.x) * blockDim.x) {
            a.pool_next[i] = 0u;
            if (a.fcnt_next) a.fcnt_next[i] = 0u;
        }
    const Tail& t = a.tail;
    const int D = a.d, g = a.group, st = a.maxseg * g;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int64_t r = u / Q;
        const int col = static_cast<int>(u % Q) * 32 + lane;
        const int h = static_cast<int>(r % g);
        Cover cv = u == blockIdx.x ? cv0 : cover_of(a, r / g);
        cv.nf = foreign_of(a, r / g);
        const int S = cv.S, T = cv.S + cv.nf;
        const int b0 = static_cast<int>((cv.c_lo * a.maxseg + cv.seg_lo) * g + h);
        const int b1 = static_cast<int>((cv.c_lo + 1) * a.maxseg * g + h);
        const int fb = static_cast<int>((r / g) * a.fslots * g + h);
        auto off_of = [&](int i) { return i >= S ? fb + (i - S) * g : (i == 0 ? b0 : b1 + (i - 1) * st); };
        const int i_lo = static_cast<int>(int64_t(T) * warp / WS), i_hi = static_cast<int>(int64_t(T) * (warp + 1) / WS);
        float M = -CUDART_INF_F, L = 0.f, acc = 0.f;
        if constexpr (SF) stream_fold<WS>(a, r, cv, col, M, L, acc, a.serr);
        for (int i0 = i_lo; !SF && i0 < i_hi; i0 += 32) {
            const int n = min(32, i_hi - i0);
            float ml = -CUDART_INF_F, ll = 0.f;
            if (lane < n) {
                const int i = i0 + lane, off = off_of(i);
                ml = __ldcg((i >= S ? a.fslot_m : a.cslot_m) + off);
                ll = __ldcg((i >= S ? a.fslot_l : a.cslot_l) + off);
            }
            float ov[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int i = i0 + min(k, n - 1);
                ov[k] = __ldcg((i >= S ? a.fslot_o : a.cslot_o) + int64_t(off_of(i)) * D + col);
            }
            float Mb = ml;
#pragma unroll
            for (int o2 = 16; o2 >= 1; o2 >>= 1) Mb = fmaxf(Mb, __shfl_xor_sync(0xffffffffu, Mb, o2));
            const float Mn = fmaxf(M, Mb);
            const float cs = M == -CUDART_INF_F ? 0.f : fast_exp2(M - Mn);
            L *= cs;
            acc *= cs;
            const float e_l = ml == -CUDART_INF_F ? 0.f : fast_exp2(ml - Mn);
            float ls = e_l * ll;
#pragma unroll
            for (int o2 = 16; o2 >= 1; o2 >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o2);
            L += ls;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const float e = __shfl_sync(0xffffffffu, e_l, k);
                acc = fmaf(e, e != 0.f ? ov[k] : 0.f, acc);
            }
            M = Mn;
        }
        if (lane == 0) {
            sm_m[warp] = M;
            sm_l[warp] = L;
        }
        sm_o[warp][lane] = acc;
        __syncthreads();
        if (warp == 0) {
            float Mx = -CUDART_INF_F;
#pragma unroll
            for (int w = 0; w < WS; ++w) Mx = fmaxf(Mx, sm_m[w]);
            float Lt = 0.f, O = 0.f;
#pragma unroll
            for (int w = 0; w < WS; ++w) {
                const float mw = sm_m[w];
                const float e = (mw == -CUDART_INF_F) ? 0.f : fast_exp2(mw - Mx);
                Lt += e * sm_l[w];
                O += e != 0.f ? e * sm_o[w][lane] : 0.f;
            }
            const bool empty = Mx == -CUDART_INF_F;
            const int64_t orow = out_row_of(a, r);
            if (col < D) t.out[orow * D + col] = empty ? 0.f : O / Lt;
            if (t.mode == kTailPartial && col == 0) {
                t.lse[orow] = empty ? -CUDART_INF_F : (Mx + log2f(Lt)) * kLn2;
                t.row_max[orow] = empty ? -CUDART_INF_F : Mx * kLn2;
            }
        }
        __syncthreads();
    }
    if constexpr (SF) asm volatile("griddepcontrol.wait;" ::: "memory");  // complete only after K1
    if (a.tl && lane == 0) atomicMax(a.tl + 3, gtimer());
    signal_done(a);
}

// =========================================================================
// K2x: K2 fused with the one-shot NVLink exchange (kTailExchange), LL
// protocol: every 8-byte word of the exchange buffer is (value, epoch), so a
// word's data and its readiness travel in one single-copy-atomic store over
// NVLink -- no system fence, no separate flag. Each warp merges its rows
// (merge_row_warp) and stores [out | lse] of them into slot `rank` of every
// peer's buffer (CUDA-IPC mapped HBM); then it reads, word by word, the p
// sources of its rows (spinning until a word carries this step's epoch) and
// combines: shift = max lse, w = e^(lse - shift), out = sum w o / sum w -- the
// allreduce(max), partial_to_numerator, allreduce(sum) and n/d of
// decode.cpp:129-173 in one exchange. Slots alternate by epoch parity (a rank
// cannot overwrite a slot a peer still reads: it would first need the peer's
// next-step words). The grid never exceeds the co-resident capacity and every
// warp pushes all its rows before it reads, so the exchange cannot deadlock;
// each spin is bounded (~2 s) and reports through x.error.
// =========================================================================
__device__ __forceinline__ void st_ll(uint2* p, float v, unsigned e) {
    asm volatile("st.volatile.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(__float_as_uint(v)), "r"(e)
                 : "memory");
}
#ifndef TD_XCHG_LD
#define TD_XCHG_LD "ld.volatile.global.v2.u32"
#endif
__device__ __forceinline__ uint2 ld_word(const uint2* p) {  // one poll, no wait
    uint2 w;
    asm volatile(TD_XCHG_LD " {%0, %1}, [%2];" : "=r"(w.x), "=r"(w.y) : "l"(p) : "memory");
    return w;
}
__device__ __forceinline__ float ld_ll(const uint2* p, unsigned e, int* err) {
    unsigned v, f;
    const long long t0 = clock64();
    for (;;) {
        asm volatile("ld.volatile.global.v2.u32 {%0, %1}, [%2];" : "=r"(v), "=r"(f) : "l"(p) : "memory");
        if (f == e) break;
        if (clock64() - t0 > (1ll << 32)) {  // ~2 s: a peer never arrived
            *reinterpret_cast<volatile int*>(err) = 1;  // mapped host memory: a plain store
            break;
        }
    }
    return __uint_as_float(v);
}


template <int V, int NC, int BO, int Q>
__global__ void __launch_bounds__(K2_THREADS) k2_exchange(const K1Args a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next step's K1 may get resident
    const int64_t rows = a.bh_count * a.group, units = rows * Q;  // Q warps per row (column split)
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    const Cover cv0 = w0 < units ? cover_of(a, (w0 / Q) / a.group) : Cover{};
    const Xchg& x = a.tail.x;
    constexpr int PMAX = 8;  // peers held in registers (the exchange spans one NVLink domain)
    uint2* pp[PMAX];         // peer buffers, read before the wait (host-written)
#pragma unroll
    for (int k = 0; k < PMAX; ++k) pp[k] = k < x.p ? reinterpret_cast<uint2* const*>(x.peers)[k] : nullptr;
    const uint2* own = reinterpret_cast<uint2* const*>(x.peers)[x.rank];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // the other parity's pool counters are the next launch's: zero them
    if (a.pool_tiles > 0)
        for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.bh_count;
             i += int64_t(gridDim.x) * blockDim.x) {
            a.pool_next[i] = 0u;
            if (a.fcnt_next) a.fcnt_next[i] = 0u;
        }
    const int D = a.d;
    const unsigned par = x.epoch & 1u;
    const int64_t stride = x.max_rows * int64_t(D + 1);  // words per (parity, source)
    uint2* const* peers = reinterpret_cast<uint2* const*>(x.peers);
    unsigned long long* ts = (a.dbg && w0 < 512 && lane == 0) ? a.dbg + 8 + 8 * w0 : nullptr;
    if (ts) ts[0] = gtimer();
    for (int64_t u = w0; u < units; u += nw) {  // merge + push
        const int64_t r = u / Q;
        const int colb = static_cast<int>(u % Q) * (32 * V * NC);
        const int64_t orow = out_row_of(a, r);
        float l, m;
        LaneRow<V, NC> res;
        Cover cv = u == w0 ? cv0 : cover_of(a, r / a.group);
        cv.nf = foreign_of(a, r / a.group);
        merge_row_warp<V, NC, BO>(a, r, cv, res, l, m, colb);
        if (ts && u == w0) ts[2] = gtimer();
        const int64_t off = (int64_t(par) * x.p + x.rank) * stride + orow * (D + 1);
        auto push = [&](uint2* dst) {  // LL words of this row into slot `rank` of one buffer
#pragma unroll
            for (int c = 0; c < NC; ++c)
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const int col = colb + (c * 32 + lane) * V + v;
                    if (col < D) st_ll(dst + col, res.v[c][v], x.epoch);
                }
            if (lane == 0 && colb == 0) st_ll(dst + D, l, x.epoch);
        };
        if (x.pull) {
            push(peers[x.rank] + off);  // own buffer only: the peers read it over NVLink
        } else {
#pragma unroll
            for (int q = 0; q < PMAX; ++q)
                if (q < x.p) push(pp[q] + off);
            for (int q = PMAX; q < x.p; ++q) push(peers[q] + off);
        }
    }
    if (ts) ts[1] = gtimer();
    for (int64_t u = w0; u < units; u += nw) {  // exact combine of the p partials
        const int64_t r = u / Q;
        const int colb = static_cast<int>(u % Q) * (32 * V * NC);
        const int64_t orow = out_row_of(a, r);
        // source k's words: push -- slot k of the own buffer; pull -- slot k of k's buffer
        const int64_t roff = int64_t(par) * x.p * stride + orow * (D + 1);
        const uint2* base = own + roff;
        // every word of the first PMAX sources (lse + this lane's columns) is polled in
        // one batch, and re-polled -- again as a batch -- until all carry this epoch
        uint2 wl[PMAX], wo[PMAX][NC][V];
        const long long t0 = clock64();
        for (;;) {
            bool all = true;
#pragma unroll
            for (int k = 0; k < PMAX; ++k) {
                if (k >= x.p) continue;
                const uint2* slot = (x.pull ? pp[k] + roff : base) + k * stride;
                wl[k] = ld_word(slot + D);
#pragma unroll
                for (int c = 0; c < NC; ++c)
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        const int col = colb + (c * 32 + lane) * V + v;
                        if (col < D) wo[k][c][v] = ld_word(slot + col);
                    }
            }
#pragma unroll
            for (int k = 0; k < PMAX; ++k) {
                if (k >= x.p) continue;
                all &= wl[k].y == x.epoch;
#pragma unroll
                for (int c = 0; c < NC; ++c)
#pragma unroll
                    for (int v = 0; v < V; ++v)
                        if (colb + (c * 32 + lane) * V + v < D) all &= wo[k][c][v].y == x.epoch;
            }
            if (__all_sync(0xffffffffu, all)) break;
            if (clock64() - t0 > (1ll << 32)) {  // ~2 s: a peer never arrived
                // mapped host memory, a plain store: 1 | first missing source << 8 | rank << 16
                int miss = 255;
#pragma unroll
                for (int k = PMAX - 1; k >= 0; --k)
                    if (k < x.p && wl[k].y != x.epoch) miss = k;
                *reinterpret_cast<volatile int*>(x.error) = 1 | (miss << 8) | (x.rank << 16);
                break;
            }
        }
        if (ts && u == w0) ts[3] = gtimer();
        float shift = -CUDART_INF_F, den = 0.f;
#pragma unroll
        for (int k = 0; k < PMAX; ++k)
            if (k < x.p) shift = fmaxf(shift, __uint_as_float(wl[k].x));
        for (int q = PMAX; q < x.p; ++q)
            shift = fmaxf(shift, ld_ll((x.pull ? peers[q] + roff : base) + q * stride + D, x.epoch, x.error));
        float num[NC][V];
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < V; ++v) num[c][v] = 0.f;
#pragma unroll
        for (int k = 0; k < PMAX; ++k) {
            if (k >= x.p) continue;
            const float l = __uint_as_float(wl[k].x);
            const float wgt = l == -CUDART_INF_F ? 0.f : expf(l - shift);
            den += wgt;
#pragma unroll
            for (int c = 0; c < NC; ++c)
#pragma unroll
                for (int v = 0; v < V; ++v) num[c][v] += wgt * __uint_as_float(wo[k][c][v].x);
        }
        for (int q = PMAX; q < x.p; ++q) {  // beyond one NVLink domain: word by word
            const uint2* slot = (x.pull ? peers[q] + roff : base) + q * stride;
            const float l = ld_ll(slot + D, x.epoch, x.error);
            const float wgt = l == -CUDART_INF_F ? 0.f : expf(l - shift);
            den += wgt;
#pragma unroll
            for (int c = 0; c < NC; ++c)
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const int col = colb + (c * 32 + lane) * V + v;
                    if (col < D) num[c][v] += wgt * ld_ll(slot + col, x.epoch, x.error);
                }
        }
        float* dst = a.tail.out + orow * D;
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int col = colb + (c * 32 + lane) * V + v;
                if (col < D) dst[col] = num[c][v] / den;
            }
    }
    if (ts) ts[4] = gtimer();
    if (a.tl && lane == 0) atomicMax(a.tl + 3, gtimer());
    signal_done(a);
}

// K2x for rows with many candidate states (the deterministic chunk pool, or few
// rows over many CTAs): the split merge of k2_combine_split per (row, column
// quarter) block, then warp 0 pushes the row's LL words into every peer and,
// after all of this block's units are pushed, polls and combines them like
// k2_exchange (one column per lane).
template <int Q, int WS, bool SF = false>
__global__ void __launch_bounds__(32 * WS) k2_exchange_split(const K1Args a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    constexpr int PMAX = 8;
    __shared__ float sm_m[WS], sm_l[WS], sm_o[WS][32];
    const int64_t rows = a.bh_count * a.group, units = rows * Q;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Xchg& x = a.tail.x;
    uint2* pp[PMAX];
#pragma unroll
    for (int k = 0; k < PMAX; ++k) pp[k] = k < x.p ? reinterpret_cast<uint2* const*>(x.peers)[k] : nullptr;
    const uint2* own = reinterpret_cast<uint2* const*>(x.peers)[x.rank];
    uint2* const* peers = reinterpret_cast<uint2* const*>(x.peers);
    const Cover cv0 = blockIdx.x < units ? cover_of(a, (int64_t(blockIdx.x) / Q) / a.group) : Cover{};
    if constexpr (!SF) asm volatile("griddepcontrol.wait;" ::: "memory");  // (streamed: see k2_combine_split)
    if (a.pool_tiles > 0)
        for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.bh_count;
             i += int64_t(gridDim.x) * blockDim.x) {
            a.pool_next[i] = 0u;
            if (a.fcnt_next) a.fcnt_next[i] = 0u;
        }
    const int D = a.d, g = a.group, st = a.maxseg * g;
    const unsigned par = x.epoch & 1u;
    const int64_t stride = x.max_rows * int64_t(D + 1);
    float lit_val = 0.f, lit_lse = -CUDART_INF_F;  // kTailLiteral: this block's unit (warp 0)
    int64_t lit_row = -1;
    int lit_col = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {  // merge + push
        const int64_t r = u / Q;
        const int col = static_cast<int>(u % Q) * 32 + lane;
        const int h = static_cast<int>(r % g);
        Cover cv = u == blockIdx.x ? cv0 : cover_of(a, r / g);
        cv.nf = foreign_of(a, r / g);
        const int S = cv.S, T = cv.S + cv.nf;
        const int b0 = static_cast<int>((cv.c_lo * a.maxseg + cv.seg_lo) * g + h);
        const int b1 = static_cast<int>((cv.c_lo + 1) * a.maxseg * g + h);
        const int fb = static_cast<int>((r / g) * a.fslots * g + h);
        auto off_of = [&](int i) { return i >= S ? fb + (i - S) * g : (i == 0 ? b0 : b1 + (i - 1) * st); };
        const int i_lo = static_cast<int>(int64_t(T) * warp / WS), i_hi = static_cast<int>(int64_t(T) * (warp + 1) / WS);
        float M = -CUDART_INF_F, L = 0.f, acc = 0.f;
        if constexpr (SF) stream_fold<WS>(a, r, cv, col, M, L, acc, a.serr);
        for (int i0 = i_lo; !SF && i0 < i_hi; i0 += 32) {
            const int n = min(32, i_hi - i0);
            float ml = -CUDART_INF_F, ll = 0.f;
            if (lane < n) {
                const int i = i0 + lane, off = off_of(i);
                ml = __ldcg((i >= S ? a.fslot_m : a.cslot_m) + off);
                ll = __ldcg((i >= S ? a.fslot_l : a.cslot_l) + off);
            }
            float ov[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const int i = i0 + min(k, n - 1);
                ov[k] = col < D ? __ldcg((i >= S ? a.fslot_o : a.cslot_o) + int64_t(off_of(i)) * D + col) : 0.f;
            }
            float Mb = ml;
#pragma unroll
            for (int o2 = 16; o2 >= 1; o2 >>= 1) Mb = fmaxf(Mb, __shfl_xor_sync(0xffffffffu, Mb, o2));
            const float Mn = fmaxf(M, Mb);
            const float cs = M == -CUDART_INF_F ? 0.f : fast_exp2(M - Mn);
            L *= cs;
            acc *= cs;
            const float e_l = ml == -CUDART_INF_F ? 0.f : fast_exp2(ml - Mn);
            float ls = e_l * ll;
#pragma unroll
            for (int o2 = 16; o2 >= 1; o2 >>= 1) ls += __shfl_xor_sync(0xffffffffu, ls, o2);
            L += ls;
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                const float e = __shfl_sync(0xffffffffu, e_l, k);
                acc = fmaf(e, e != 0.f ? ov[k] : 0.f, acc);
            }
            M = Mn;
        }
        if (lane == 0) {
            sm_m[warp] = M;
            sm_l[warp] = L;
        }
        sm_o[warp][lane] = acc;
        __syncthreads();
        if (warp == 0) {
            float Mx = -CUDART_INF_F;
#pragma unroll
            for (int w = 0; w < WS; ++w) Mx = fmaxf(Mx, sm_m[w]);
            float Lt = 0.f, O = 0.f;
#pragma unroll
            for (int w = 0; w < WS; ++w) {
                const float mw = sm_m[w];
                const float e = (mw == -CUDART_INF_F) ? 0.f : fast_exp2(mw - Mx);
                Lt += e * sm_l[w];
                O += e != 0.f ? e * sm_o[w][lane] : 0.f;
            }
            const bool empty = Mx == -CUDART_INF_F;
            const float val = empty ? 0.f : O / Lt;
            const float lse = empty ? -CUDART_INF_F : (Mx + log2f(Lt)) * kLn2;
            const int64_t orow = out_row_of(a, r);
            const int64_t off = (int64_t(par) * x.p + x.rank) * stride + orow * (D + 1);
            auto push = [&](uint2* dst) {
                if (col < D) st_ll(dst + col, val, x.epoch);
                if (lane == 0 && col == 0) st_ll(dst + D, lse, x.epoch);
            };
            if (SF && a.tail.mode == kTailLiteral) {
                // round 1 of the literal combine: this rank's lse of the row into slot
                // (parity, rank) of region A of every rank's window (one unit per block)
                lit_val = val;
                lit_lse = lse;
                lit_row = orow;
                lit_col = col;
                if (lane == 0 && col == 0)
                    for (int q = 0; q < x.p; ++q) st_ll(peers[q] + (int64_t(par) * x.p + x.rank) * x.max_rows + orow, lse, x.epoch);
            } else if (x.pull) {
                push(peers[x.rank] + off);
            } else {
#pragma unroll
                for (int q = 0; q < PMAX; ++q)
                    if (q < x.p) push(pp[q] + off);
                for (int q = PMAX; q < x.p; ++q) push(peers[q] + off);
            }
        }
        __syncthreads();
    }
    if (SF && a.tail.mode == kTailLiteral) {
        if (warp == 0 && lit_row >= 0) {
            // round 1 receive: max over the p ranks' lse of the row
            const uint2* ownw = peers[x.rank];
            float m = -CUDART_INF_F;
            for (int k = lane; k < x.p; k += 32)
                m = fmaxf(m, ld_ll(ownw + (int64_t(par) * x.p + k) * x.max_rows + lit_row, x.epoch, x.error));
#pragma unroll
            for (int s2 = 16; s2 >= 1; s2 >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, s2));
            // partial_to_numerator, then round 2: [n | d] into slot (parity, rank) of region B
            const float wgt = lit_lse == -CUDART_INF_F ? 0.f : expf(lit_lse - m);
            const float nv = lit_val * wgt;
            const int64_t b0 = 2 * int64_t(x.p) * x.max_rows;
            const int64_t sstride = x.max_rows * int64_t(D + 1);
            const int64_t boff = b0 + (int64_t(par) * x.p + x.rank) * sstride + lit_row * (D + 1);
            for (int q = 0; q < x.p; ++q) {
                uint2* dst = (q < PMAX ? pp[q] : peers[q]) + boff;
                if (lit_col < D) st_ll(dst + lit_col, nv, x.epoch);
                if (lane == 0 && lit_col == 0) st_ll(dst + D, wgt, x.epoch);
            }
            // round 2 receive: sum the p sources' [n | d] (the first PMAX as one batch), n / d
            const uint2* base = ownw + b0 + int64_t(par) * x.p * sstride + lit_row * (D + 1);
            uint2 wd[PMAX], wn[PMAX];
            const long long t0 = clock64();
            for (;;) {
                bool all = true;
#pragma unroll
                for (int k = 0; k < PMAX; ++k) {
                    if (k >= x.p) continue;
                    wd[k] = ld_word(base + k * sstride + D);
                    if (lit_col < D) wn[k] = ld_word(base + k * sstride + lit_col);
                }
#pragma unroll
                for (int k = 0; k < PMAX; ++k) {
                    if (k >= x.p) continue;
                    all &= wd[k].y == x.epoch;
                    if (lit_col < D) all &= wn[k].y == x.epoch;
                }
                if (__all_sync(0xffffffffu, all)) break;
                if (clock64() - t0 > (1ll << 32)) {  // ~2 s: a rank never arrived
                    *reinterpret_cast<volatile int*>(x.error) = 1 | (255 << 8) | (x.rank << 16);
                    break;
                }
            }
            float den = 0.f, num = 0.f;
#pragma unroll
            for (int k = 0; k < PMAX; ++k) {
                if (k >= x.p) continue;
                den += __uint_as_float(wd[k].x);
                if (lit_col < D) num += __uint_as_float(wn[k].x);
            }
            for (int k = PMAX; k < x.p; ++k) {
                den += ld_ll(base + k * sstride + D, x.epoch, x.error);
                if (lit_col < D) num += ld_ll(base + k * sstride + lit_col, x.epoch, x.error);
            }
            if (lit_col < D) a.tail.out[lit_row * D + lit_col] = num / den;
        }
    } else if (warp == 0) {
        for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {  // exact combine of the p partials
            const int64_t r = u / Q;
            const int col = static_cast<int>(u % Q) * 32 + lane;
            const int64_t orow = out_row_of(a, r);
            const int64_t roff = int64_t(par) * x.p * stride + orow * (D + 1);
            const uint2* base = own + roff;
            uint2 wl[PMAX], wo[PMAX];
            const long long t0 = clock64();
            for (;;) {
                bool all = true;
#pragma unroll
                for (int k = 0; k < PMAX; ++k) {
                    if (k >= x.p) continue;
                    const uint2* slot = (x.pull ? pp[k] + roff : base) + k * stride;
                    wl[k] = ld_word(slot + D);
                    if (col < D) wo[k] = ld_word(slot + col);
                }
#pragma unroll
                for (int k = 0; k < PMAX; ++k) {
                    if (k >= x.p) continue;
                    all &= wl[k].y == x.epoch;
                    if (col < D) all &= wo[k].y == x.epoch;
                }
                if (__all_sync(0xffffffffu, all)) break;
                if (clock64() - t0 > (1ll << 32)) {  // ~2 s: a peer never arrived
                    int miss = 255;
#pragma unroll
                    for (int k = PMAX - 1; k >= 0; --k)
                        if (k < x.p && wl[k].y != x.epoch) miss = k;
                    *reinterpret_cast<volatile int*>(x.error) = 1 | (miss << 8) | (x.rank << 16);
                    break;
                }
            }
            float shift = -CUDART_INF_F, den = 0.f, num = 0.f;
#pragma unroll
            for (int k = 0; k < PMAX; ++k)
                if (k < x.p) shift = fmaxf(shift, __uint_as_float(wl[k].x));
            for (int q = PMAX; q < x.p; ++q)
                shift = fmaxf(shift, ld_ll((x.pull ? peers[q] + roff : base) + q * stride + D, x.epoch, x.error));
#pragma unroll
            for (int k = 0; k < PMAX; ++k) {
                if (k >= x.p) continue;
                const float l = __uint_as_float(wl[k].x);
                const float wgt = l == -CUDART_INF_F ? 0.f : expf(l - shift);
                den += wgt;
                if (col < D) num += wgt * __uint_as_float(wo[k].x);
            }
            for (int q = PMAX; q < x.p; ++q) {
                const uint2* slot = (x.pull ? peers[q] + roff : base) + q * stride;
                const float l = ld_ll(slot + D, x.epoch, x.error);
                const float wgt = l == -CUDART_INF_F ? 0.f : expf(l - shift);
                den += wgt;
                if (col < D) num += wgt * ld_ll(slot + col, x.epoch, x.error);
            }
            if (col < D) a.tail.out[orow * D + col] = num / den;
        }
    }
    if constexpr (SF) asm volatile("griddepcontrol.wait;" ::: "memory");  // complete only after K1
    if (a.tl && lane == 0) atomicMax(a.tl + 3, gtimer());
    signal_done(a);
}

// =========================================================================
// K2n: the paper-literal combine of decode.cpp:129-173 -- allreduce(max) of the
// shard lse, partial_to_numerator, allreduce(sum) of [n|d], n/d -- as one kernel
// over a symmetric NCCL window (NCCL's device API makes every rank's window
// load/store-addressable: ncclGetLsaPointer, td_nccl_dev.cu). Each allreduce is
// one round of LL words (value, epoch): a warp stores its rows' words into slot
// `rank` of every rank's window, then polls the p slots of its own. It runs as a
// programmatic dependent of K2 (kTailPartial: lse and out per output row).
// Window layout, 8-byte words: A [2 parities][p][max_rows] lse, then
// B [2][p][max_rows][d + 1] [n | d]. Parities alternate by epoch, so a slot is
// rewritten only after every rank has read it (as in K2x). One-warp blocks, at
// most the co-resident count, each pushing all its rows before any wait: the
// exchange cannot deadlock; spins are bounded and report through x.error.
// =========================================================================
template <int NC>
__global__ void __launch_bounds__(32) k2n_literal(const float* lse, const float* o, const XchgArgs x, int64_t rows,
                                                  int d, float* out) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the next step's K1 may get resident
    constexpr int PMAX = 8;  // sources polled as one batch
    const int lane = threadIdx.x & 31;
    uint2* const* peers = reinterpret_cast<uint2* const*>(x.peers);
    uint2* pp[PMAX];
#pragma unroll
    for (int k = 0; k < PMAX; ++k) pp[k] = k < x.p ? peers[k] : nullptr;
    const uint2* own = peers[x.rank];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const unsigned par = x.epoch & 1u;
    const int64_t a_src = x.max_rows;  // region A words per (parity, source)
    const int64_t b0 = 2 * int64_t(x.p) * a_src;                             // region B
    // allreduce(max), send: this rank's lse of each of its rows to every rank
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const float l = __ldcg(lse + r);
        const int64_t off = (int64_t(par) * x.p + x.rank) * a_src + r;
        for (int q = lane; q < x.p; q += 32) st_ll(peers[q] + off, l, x.epoch);
    }
    // receive -> shift; n = o e^(l - shift), d = e^(l - shift); allreduce(sum), send
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        float m = -CUDART_INF_F;
        for (int k = lane; k < x.p; k += 32)
            m = fmaxf(m, ld_ll(own + (int64_t(par) * x.p + k) * a_src + r, x.epoch, x.error));
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, s));
        const float l = __ldcg(lse + r);
        const float wgt = l == -CUDART_INF_F ? 0.f : expf(l - m);
        float nv[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const int col = c * 32 + lane;
            nv[c] = col < d ? __ldcg(o + r * d + col) * wgt : 0.f;
        }
        const int64_t off = b0 + ((int64_t(par) * x.p + x.rank) * x.max_rows + r) * (d + 1);
        for (int q = 0; q < x.p; ++q) {
            uint2* dst = (q < PMAX ? pp[q] : peers[q]) + off;
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if (c * 32 + lane < d) st_ll(dst + c * 32 + lane, nv[c], x.epoch);
            if (lane == 0) st_ll(dst + d, wgt, x.epoch);
        }
    }
    // receive: sum the p sources' [n | d] (first PMAX polled as one batch), n / d
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const uint2* base = own + b0 + (int64_t(par) * x.p * x.max_rows + r) * (d + 1);
        const int64_t sstride = x.max_rows * int64_t(d + 1);
        uint2 wd[PMAX], wn[PMAX][NC];
        const long long t0 = clock64();
        for (;;) {
            bool all = true;
#pragma unroll
            for (int k = 0; k < PMAX; ++k) {
                if (k >= x.p) continue;
                const uint2* slot = base + k * sstride;
                wd[k] = ld_word(slot + d);
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    if (c * 32 + lane < d) wn[k][c] = ld_word(slot + c * 32 + lane);
            }
#pragma unroll
            for (int k = 0; k < PMAX; ++k) {
                if (k >= x.p) continue;
                all &= wd[k].y == x.epoch;
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    if (c * 32 + lane < d) all &= wn[k][c].y == x.epoch;
            }
            if (__all_sync(0xffffffffu, all)) break;
            if (clock64() - t0 > (1ll << 32)) {  // ~2 s: a rank never arrived
                int miss = 255;
#pragma unroll
                for (int k = PMAX - 1; k >= 0; --k)
                    if (k < x.p && wd[k].y != x.epoch) miss = k;
                *reinterpret_cast<volatile int*>(x.error) = 1 | (miss << 8) | (x.rank << 16);
                break;
            }
        }
        float den = 0.f, num[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) num[c] = 0.f;
#pragma unroll
        for (int k = 0; k < PMAX; ++k) {
            if (k >= x.p) continue;
            den += __uint_as_float(wd[k].x);
#pragma unroll
            for (int c = 0; c < NC; ++c) num[c] += __uint_as_float(wn[k][c].x);
        }
        for (int k = PMAX; k < x.p; ++k) {  // past one batch: word by word
            const uint2* slot = base + k * sstride;
            den += ld_ll(slot + d, x.epoch, x.error);
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if (c * 32 + lane < d) num[c] += ld_ll(slot + c * 32 + lane, x.epoch, x.error);
        }
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (c * 32 + lane < d) out[r * d + c * 32 + lane] = num[c] / den;
    }
}

// =========================================================================
// K3 / K4 / K5 / combine_partials / K6
// =========================================================================
__global__ void k3_to_numerator(const float* lse, const float* out, const float* shift,
                                int64_t rows, int d, float* nd) {
    const int64_t n = rows * d;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n + rows;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i < n ? i / d : i - n;
        const float l = lse[r];
        const float w = l == -CUDART_INF_F ? 0.f : expf(l - shift[r]);
        nd[i] = i < n ? out[i] * w : w;
    }
}

__global__ void k4_finalize(const float* nd, int64_t rows, int d, float* out,
                            __nv_bfloat16* out_bf16) {
    const int64_t n = rows * d;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const float y = nd[i] / nd[n + i / d];
        out[i] = y;
        if (out_bf16) out_bf16[i] = __float2bfloat16_rn(y);
    }
}

__global__ void k5_combine_pair(float* lmax, float* llse, float* lout, const float* rmax,
                                const float* rlse, const float* rout, int64_t rows, int d) {
    const int64_t r = blockIdx.x;
    if (r >= rows) return;
    const float la = llse[r], lb = rlse[r];
    float l;
    if (la == -CUDART_INF_F) l = lb;
    else if (lb == -CUDART_INF_F) l = la;
    else {
        const float mm = fmaxf(la, lb);
        l = mm + logf(expf(la - mm) + expf(lb - mm));
    }
    const float wa = la == -CUDART_INF_F ? 0.f : expf(la - l);
    const float wb = lb == -CUDART_INF_F ? 0.f : expf(lb - l);
    for (int j = threadIdx.x; j < d; j += blockDim.x)
        lout[r * d + j] = lout[r * d + j] * wa + rout[r * d + j] * wb;
    __syncthreads();
    if (threadIdx.x == 0) {
        llse[r] = l;
        lmax[r] = fmaxf(lmax[r], rmax[r]);
    }
}

__global__ void k_combine_partials(int P, const float* lse, const float* out, int64_t rows, int d,
                                   float* result, int* bad_row) {
    const int64_t r = blockIdx.x;
    if (r >= rows) return;
    float shift = -CUDART_INF_F;
    for (int p = 0; p < P; ++p) shift = fmaxf(shift, lse[p * rows + r]);
    if (shift == -CUDART_INF_F) {
        if (threadIdx.x == 0) *reinterpret_cast<volatile int*>(bad_row) = 1;  // mapped host flag
        for (int j = threadIdx.x; j < d; j += blockDim.x) result[r * d + j] = 0.f;
        return;
    }
    for (int j = threadIdx.x; j < d; j += blockDim.x) {
        float num = 0.f, den = 0.f;
        for (int p = 0; p < P; ++p) {
            const float l = lse[p * rows + r];
            if (l == -CUDART_INF_F) continue;
            const float w = expf(l - shift);
            den += w;
            num += out[(p * rows + r) * d + j] * w;
        }
        result[r * d + j] = num / den;
    }
}

__global__ void k6_seeded_fill(int dtype, void* dst, uint64_t seed, double half_width,
                               int64_t bh_count, int64_t seq, int64_t start, int64_t len,
                               int64_t d) {
    const int64_t n = bh_count * len * d;
    const int64_t per_bh = len * d;
    for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int64_t bh = e / per_bh;
        const int64_t rem = e - bh * per_bh;
        const int64_t i = rem / d, j = rem - i * d;
        const uint64_t gi = static_cast<uint64_t>((bh * seq + start + i) * d + j);
        const double x = seeded_value(seed, gi, half_width);
        if (dtype == kBF16) static_cast<uint16_t*>(dst)[e] = double_to_bf16_bits(x);
        else if (dtype == kF32) static_cast<float*>(dst)[e] = __double2float_rn(x);
        else static_cast<double*>(dst)[e] = x;
    }
}

// =========================================================================
// host side: planning and launchers
// =========================================================================
namespace {

constexpr int kBf16Tile = 32;
// k1_f32 geometry: tokens per tile x warps x ring entries (a K or a V tile each).
// TD_F32_CFG = 0 (32 x 4 x 2, default), 1 (32 x 2 x 6), 2 (32 x 6 x 2), 3 (16 x 4 x 4),
// 4 (32 x 4 x 3), 5 (32 x 3 x 4: round 1's 3 warps x 2 K+V stages), 6 (16 x 6 x 4),
// 7 (16 x 8 x 2). cfg1 (profiles/r2_cfg1/geometry/): 32 x 4 x 2 streams 64K fp32
// tokens in 17.4 us (ncu, clean L2) against 18.8 for 32 x 3 x 4.
constexpr int kF32Tiles[8] = {32, 32, 32, 16, 32, 32, 16, 16};
constexpr int kF32Warps[8] = {4, 2, 6, 4, 4, 3, 6, 8};
constexpr int kF32Entries[8] = {2, 6, 2, 4, 3, 4, 4, 2};
int f32_cfg() {
    static const int c = [] { const char* e = std::getenv("TD_F32_CFG"); return e ? std::atoi(e) & 7 : 0; }();
    return c;
}
int f32_warps() { return kF32Warps[f32_cfg()]; }
constexpr int kGenTile = 32, kGenWarps = 4;
constexpr int kSmemBudget = 192 * 1024;  // per CTA, one CTA per SM

// bf16: W warps x S stages x (K + V tile of kBf16Tile tokens x D)
constexpr int bf16_warps(int D) { return D >= 256 ? 2 : 4; }
constexpr int bf16_stage_bytes(int D) { return 2 * (D / 64) * kBf16Tile * 128; }
constexpr int bf16_stages(int D) { return kSmemBudget / (bf16_warps(D) * bf16_stage_bytes(D)); }
template <int D>
size_t bf16_smem() {
    return size_t(bf16_warps(D)) * bf16_stages(D) * bf16_stage_bytes(D) + 1024;
}
size_t f32_smem() {
    return size_t(kF32Warps[f32_cfg()]) * kF32Entries[f32_cfg()] * kF32Tiles[f32_cfg()] * 128 * 4 + 128;
}

}  // namespace

// The streamed combine applies to the bf16 kernel with the deterministic chunk pool
// (per-warp static states, one state per chunk) and d = 128 (the split K2).
bool stream_plan(const SplitPlan& p) {
    return p.sflag && p.kernel == 1 && p.dpool && p.fslots > 0 && p.d == 128 && !p.dbg && p.slot_warps == p.warps;
}

namespace {

K1Args make_args(const SplitPlan& p, const void* q, const void* k, const void* v, float scale,
                 void* ws) {
    K1Args a{};
    a.dbg = p.dbg;
    a.tl = p.tl;
    a.tl_cta = p.tl_cta;
    static const int early = [] { const char* e = std::getenv("TD_K1_EARLY_TRIGGER"); return e ? std::atoi(e) : 0; }();
    a.early_trigger = early;
    static const int rev = [] { const char* e = std::getenv("TD_DEBUG_REVERSE"); return e ? std::atoi(e) : 0; }();
    a.reverse = rev;
    a.q = q;
    a.k = k;
    a.v = v;
    a.bh_count = p.bh_count;
    a.t = p.t;
    a.row_stride = p.row_stride > 0 ? p.row_stride : p.t;
    static const int prefetch = [] { const char* e = std::getenv("TD_K1_PREFETCH"); return e ? std::atoi(e) : 1; }();
    a.t_safe = prefetch ? (p.t_safe < p.t ? p.t_safe : p.t) : 0;
    a.tiles_per_bh = p.tiles_per_bh;
    a.total_tiles = p.total_tiles;
    a.d = p.d;
    a.n_q = p.n_q;
    a.n_kv = p.n_kv;
    a.group = p.group;
    a.ctas = p.ctas;
    a.maxseg = p.maxseg;
    a.scale_log2 = scale * kLog2e;
    float* f = static_cast<float*>(ws);
    const int64_t ns = p.slots() * p.group;
    a.slot_m = f;
    a.slot_l = f + ns;
    a.slot_o = f + 2 * ns;
    float* cf = f + ns * (2 + int64_t(p.d));
    const int64_t nc = int64_t(p.ctas) * p.maxseg * p.group;
    a.cslot_m = cf;
    a.cslot_l = cf + nc;
    a.cslot_o = cf + 2 * nc;
    a.pool_first = p.pool_first;
    a.pool_tiles = p.pool_tiles;
    a.pool_chunk = p.pool_chunk;
    a.slot_warps = p.slot_warps;
    a.x_table = p.x_table;
    a.sm_to_cta = p.sm_to_cta;
    a.claims = p.claims;
    a.epoch = p.epoch;
    a.bh_table = p.bh_table;
    a.done_ctr = p.done_ctr;
    a.app_k = p.app_k;
    a.app_v = p.app_v;
    a.app_pos = p.app_pos;
    a.done_flag = p.done_flag;
    a.done_epoch = p.done_epoch;
    a.sflag = stream_plan(p) ? p.sflag : nullptr;
    a.serr = p.serr;
    a.solo = p.pdl ? 1 : 0;
    a.sepoch = p.sepoch;
    static const int sspin = [] { const char* e = std::getenv("TD_K2_STREAM_SLEEP"); return e ? std::atoi(e) : 64; }();
    a.sspin = sspin;
    if (p.pool_tiles > 0) {
        unsigned* cnt = p.counters;  // [2 parities][bh_count] pool, then [2][bh_count] foreign
        a.pool_ctr = cnt + p.parity * p.bh_count;
        a.pool_next = cnt + (1 - p.parity) * p.bh_count;
        a.fcnt = cnt + (2 + p.parity) * p.bh_count;
        a.fcnt_next = cnt + (3 - p.parity) * p.bh_count;
        a.fslots = p.fslots;
        a.dpool = p.dpool ? 1 : 0;
        static const int scans = [] { const char* e = std::getenv("TD_STEAL_SCANS"); return e ? std::atoi(e) : 2; }();
        static const int smin = [] { const char* e = std::getenv("TD_STEAL_MIN"); return e ? std::atoi(e) : 4; }();
        a.steal_scans = scans;
        a.steal_min = smin;
        float* ff = cf + nc * (2 + int64_t(p.d));
        const int64_t nf = p.bh_count * int64_t(p.fslots) * p.group;
        a.fslot_m = ff;
        a.fslot_l = ff + nf;
        a.fslot_o = ff + 2 * nf;
    }
    return a;
}

template <typename K>
cudaError_t set_smem(K kernel, size_t bytes) {
    // the attribute is per kernel and per device; set it once (a driver call per
    // launch would sit on the host side of every decode step)
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = done[{reinterpret_cast<const void*>(kernel), dev}];
    if (cur >= bytes) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(bytes));
    if (e == cudaSuccess) cur = bytes;
    return e;
}

// Kernels sharing the stream with K1 ask for K1's shared-memory carveout, so an
// SM never has to be reconfigured (drained) between K1 and its neighbours.
template <typename K>
cudaError_t prefer_max_smem(K kernel) {
    static const bool on = [] { const char* e = std::getenv("TD_CARVEOUT"); return !e || std::atoi(e) != 0; }();
    if (!on) return cudaSuccess;
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, bool> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    bool& d = done[{reinterpret_cast<const void*>(kernel), dev}];
    if (d) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                               cudaSharedmemCarveoutMaxShared);
    if (e == cudaSuccess) d = true;
    return e;
}

}  // namespace

__global__ void k_stamp(unsigned long long* p) { *p = gtimer(); }
cudaError_t launch_stamp(unsigned long long* p, cudaStream_t st) {
    prefer_max_smem(k_stamp);
    k_stamp<<<1, 1, 0, st>>>(p);
    return cudaGetLastError();
}

bool plan_split(int dtype, int64_t b, int n_q, int n_kv, int64_t t, int d, int sm_count,
                SplitPlan& p, std::string& msg, int pool_mode, bool generic_only) {
    if (b < 1 || n_q < 1 || n_kv < 1 || d < 1 || t < 0) {
        msg = "decode: dimensions must be positive";
        return false;
    }
    if (n_q % n_kv != 0) {
        msg = "decode: q heads must be a multiple of kv heads (GQA group)";
        return false;
    }
    if (dtype != kBF16 && dtype != kF32) {
        msg = "decode: the GPU path computes on bf16 or f32 inputs (f64 unsupported)";
        return false;
    }
    if (d > 256) {
        msg = "decode: head_dim must be <= 256";
        return false;
    }
    p = SplitPlan{};
    p.dtype = dtype;
    p.bh_count = b * n_kv;
    p.t = t;
    p.d = d;
    p.n_q = n_q;
    p.n_kv = n_kv;
    p.group = n_q / n_kv;
    const bool mma_ok = !generic_only && dtype == kBF16 && (d == 64 || d == 128 || d == 256) && p.group <= 8 &&
                        p.bh_count * t < (int64_t(1) << 31);
    const bool f32_ok = !generic_only && dtype == kF32 && d == 128 && (p.group == 1 || p.group == 2);
    if (mma_ok) {
        p.kernel = 1;
        p.tile = kBf16Tile;
        p.warps = bf16_warps(d);
    } else if (f32_ok) {
        p.kernel = 2;
        p.tile = kF32Tiles[f32_cfg()];
        p.warps = f32_warps();
    } else {
        p.kernel = 0;
        p.tile = kGenTile;
        p.warps = kGenWarps;
    }
    p.full_tiles_per_bh = (t + p.tile - 1) / p.tile;
    // Dynamic pool (bf16 kernel): the last pool_frac of every bh's tiles are
    // handed out at run time, so SMs that stream slower (their share of HBM
    // bandwidth differs by up to ~20%) do less of them.
    static const double pool_frac = [] {
        const char* e = std::getenv("TD_POOL_FRAC");
        return e ? std::atof(e) : 0.15;
    }();
    static const int pool_chunk = [] {
        const char* e = std::getenv("TD_POOL_CHUNK");
        return e ? std::max(1, std::atoi(e)) : 2;
    }();
    // Deterministic chunk pool: the last dpool_frac of every row (at most
    // dpool_maxch chunks of dpool_chunk tiles), each chunk its own merge candidate.
    // 64 x 5 tiles measured best at 131K among 32x6..192x2 (profiles/r2_balance_131k/)
    static const double dpool_frac = [] {
        const char* e = std::getenv("TD_DPOOL_FRAC");
        return e ? std::atof(e) : 0.08;
    }();
    static const int dpool_chunk = [] {
        const char* e = std::getenv("TD_DPOOL_CHUNK");
        return e ? std::max(1, std::atoi(e)) : 5;
    }();
    static const int dpool_maxch = [] {
        const char* e = std::getenv("TD_DPOOL_MAXCH");
        return e ? std::max(1, std::atoi(e)) : 64;
    }();
    int64_t pool = 0;
    // only where the merge stays one K2 block per (row, column quarter): the chunk
    // states multiply every row's merge candidates
    const bool dpool = pool_mode == 2 && p.kernel == 1 && p.full_tiles_per_bh >= 32 && dpool_frac > 0.0 &&
                       b * int64_t(n_q) * 4 <= sm_count;
    if (pool_mode == 1 && p.kernel == 1 && p.full_tiles_per_bh >= 16 && pool_frac > 0.0)
        pool = std::min<int64_t>(p.full_tiles_per_bh / 2, static_cast<int64_t>(p.full_tiles_per_bh * pool_frac));
    int chunk = pool_chunk;
    if (dpool) {  // at most dpool_maxch chunk states per row (one round trip of the split K2)
        pool = std::min<int64_t>(p.full_tiles_per_bh / 2, static_cast<int64_t>(p.full_tiles_per_bh * dpool_frac));
        chunk = dpool_chunk;
        pool = std::min<int64_t>(pool, int64_t(dpool_maxch) * chunk);
    }
    p.dpool = dpool && pool > 0;
    p.pool_tiles = pool;
    p.pool_first = p.full_tiles_per_bh - pool;
    p.pool_chunk = chunk;
    // cross-row stealing pays on long shards (measured: -2 % at 1M tokens and on
    // cfg4's 8.6 GB, +1-2 % at 131K, where the scans and the extra merge
    // candidates cost more than the imbalance they remove): on when a CTA
    // streams >= 1024 tiles; TD_STEAL_SLOTS forces the slot count (0 = off)
    static const int fslots_env = [] {
        const char* e = std::getenv("TD_STEAL_SLOTS");
        return e ? std::max(0, std::atoi(e)) : -1;
    }();
    const int64_t tiles_per_cta = sm_count > 0 ? p.bh_count * p.full_tiles_per_bh / sm_count : 0;
    const int fslots = fslots_env >= 0 ? fslots_env : (tiles_per_cta >= 1024 ? 16 : 0);
    p.fslots = pool > 0 ? fslots : 0;
    if (p.dpool) p.fslots = static_cast<int>((pool + chunk - 1) / chunk);  // one state per chunk
    p.tiles_per_bh = p.full_tiles_per_bh - pool;
    p.total_tiles = p.bh_count * p.tiles_per_bh;
    // one CTA per SM (the per-warp pipelines fill shared memory); without a
    // pool never more CTAs than tiles.
    int64_t ctas = sm_count;
    if (pool == 0 && p.total_tiles < ctas) ctas = p.total_tiles > 0 ? p.total_tiles : 1;
    p.ctas = static_cast<int>(ctas);
    p.slot_warps = p.warps * (pool > 0 && !p.dpool ? 2 : 1);  // chunk states live in fslot
    const int64_t per_cta = (p.total_tiles + p.ctas - 1) / p.ctas;
    const int64_t tpb = p.tiles_per_bh > 0 ? p.tiles_per_bh : 1;
    p.maxseg = static_cast<int>((per_cta + tpb - 1) / tpb + 1);
    if (p.maxseg > kMaxSegments) {
        msg = "decode: too many (batch, head) rows per CTA for a split plan";
        return false;
    }
    return true;
}

void build_partition(SplitPlan& p, const float* w, int64_t* x, int* bh) {
    const int G = p.ctas;
    const int64_t T = p.total_tiles, A = p.tiles_per_bh > 0 ? p.tiles_per_bh : 1;
    double tot = 0.0;
    for (int c = 0; c < G; ++c) tot += w[c] > 0.f ? w[c] : 0.f;
    double acc = 0.0;
    x[0] = 0;
    for (int c = 0; c < G; ++c) {
        acc += w[c] > 0.f ? w[c] : 0.f;
        int64_t e = c + 1 == G ? T : static_cast<int64_t>(std::llround(double(T) * acc / (tot > 0 ? tot : 1.0)));
        x[c + 1] = std::min(T, std::max(x[c], e));
    }
    int maxseg = 1;
    for (int c = 0; c < G; ++c)
        if (x[c + 1] > x[c]) maxseg = std::max<int>(maxseg, static_cast<int>((x[c + 1] - 1) / A - x[c] / A + 1));
    for (int64_t b = 0; b < p.bh_count; ++b) {
        const int64_t X = b * A, Xe = X + A - 1;
        // the CTA c with x[c] <= X < x[c + 1] (never an empty range)
        const int lo = static_cast<int>(std::upper_bound(x, x + G + 1, X) - x) - 1;
        const int hi = static_cast<int>(std::upper_bound(x, x + G + 1, Xe) - x) - 1;
        bh[3 * b] = lo;
        bh[3 * b + 1] = hi;
        bh[3 * b + 2] = static_cast<int>(b - x[lo] / A);
    }
    p.maxseg = std::max(p.maxseg, maxseg);
}

bool make_tensor_map(CUtensorMap* map, const void* base, int64_t rows, int d, int tile_rows,
                     std::string& msg) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static EncodeFn encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess ||
            !fn) {
            msg = "cuTensorMapEncodeTiled unavailable";
            return false;
        }
        encode = reinterpret_cast<EncodeFn>(fn);
    }
    const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows > 0 ? rows : 1)};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(d) * 2};
    const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(tile_rows)};
    const cuuint32_t estride[2] = {1, 1};
    const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim,
                              gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        msg = "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")";
        return false;
    }
    return true;
}

namespace {

// K1 is launched as a programmatic dependent of whatever kernel precedes it on
// the stream (typically the previous step's K2): its CTAs get resident while
// that kernel drains and wait in griddepcontrol.wait before touching any input,
// so the ~3-5 us kernel-to-kernel launch gap leaves the critical path.
template <typename Kern, typename... Args>
cudaError_t launch_pdl(Kern kernel, int grid, int block, size_t smem, cudaStream_t st, bool allow, Args... args) {
    static const bool env_on = [] { const char* e = std::getenv("TD_K1_PDL"); return !e || std::atoi(e) != 0; }();
    const bool on = env_on && allow;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(block));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = on ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// One K1 launch (any variant) with the tail configured in a.
cudaError_t launch_k1(const SplitPlan& p, const K1Args& a, const CUtensorMap* tmk,
                      const CUtensorMap* tmv, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1) {
    cudaError_t e = cudaSuccess;
    if (ev0 && (e = cudaEventRecord(ev0, st)) != cudaSuccess) return e;
    if (p.kernel == 1) {
        if (!tmk || !tmv) return cudaErrorInvalidValue;
        switch (p.d) {
#define TD_LAUNCH_BF16(DD)                                                                  \
    case DD: {                                                                              \
        auto kern = k1_bf16<DD, kBf16Tile, bf16_warps(DD), bf16_stages(DD)>;                \
        const size_t sm = bf16_smem<DD>();                                                  \
        if ((e = set_smem(kern, sm)) != cudaSuccess) return e;                              \
        if ((e = launch_pdl(kern, p.ctas, bf16_warps(DD) * 32, sm, st, p.pdl, a, *tmk, *tmv)) != cudaSuccess) return e; \
        break;                                                                              \
    }
            TD_LAUNCH_BF16(64)
            TD_LAUNCH_BF16(128)
            TD_LAUNCH_BF16(256)
#undef TD_LAUNCH_BF16
        default: return cudaErrorInvalidValue;
        }
    } else if (p.kernel == 2) {
        const size_t sm = f32_smem();
        switch (p.group) {
#define TD_LAUNCH_F32_WS(GG, TT, WW, SS)                                        \
    {                                                                       \
        auto kern = k1_f32<TT, WW, SS, GG>;                                 \
        if ((e = set_smem(kern, sm)) != cudaSuccess) return e;              \
        if ((e = launch_pdl(kern, p.ctas, WW * 32, sm, st, p.pdl, a)) != cudaSuccess) return e; \
    }
#define TD_LAUNCH_F32(GG)                                                   \
    case GG:                                                                \
        switch (f32_cfg()) {                                                \
        case 1: TD_LAUNCH_F32_WS(GG, 32, 2, 6) break;                       \
        case 2: TD_LAUNCH_F32_WS(GG, 32, 6, 2) break;                       \
        case 3: TD_LAUNCH_F32_WS(GG, 16, 4, 4) break;                       \
        case 4: TD_LAUNCH_F32_WS(GG, 32, 4, 3) break;                       \
        case 5: TD_LAUNCH_F32_WS(GG, 32, 3, 4) break;                       \
        case 6: TD_LAUNCH_F32_WS(GG, 16, 6, 4) break;                       \
        case 7: TD_LAUNCH_F32_WS(GG, 16, 8, 2) break;                       \
        default: TD_LAUNCH_F32_WS(GG, 32, 4, 2) break;                      \
        }                                                                   \
        break;
            TD_LAUNCH_F32(1)
            TD_LAUNCH_F32(2)
#undef TD_LAUNCH_F32
#undef TD_LAUNCH_F32_WS
        default: return cudaErrorInvalidValue;
        }
    } else {
        size_t sm = sizeof(float) * 3 * kGenWarps * p.maxseg * p.group;
        if (p.dtype == kBF16) {
            if ((e = set_smem(k1_generic<__nv_bfloat16>, sm)) != cudaSuccess) return e;
            if ((e = launch_pdl(k1_generic<__nv_bfloat16>, p.ctas, kGenWarps * 32, sm, st, p.pdl, a)) != cudaSuccess) return e;
        } else {
            if ((e = set_smem(k1_generic<float>, sm)) != cudaSuccess) return e;
            if ((e = launch_pdl(k1_generic<float>, p.ctas, kGenWarps * 32, sm, st, p.pdl, a)) != cudaSuccess) return e;
        }
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (ev1 && (e = cudaEventRecord(ev1, st)) != cudaSuccess) return e;
    return cudaSuccess;
}

}  // namespace

namespace {

// K2 right behind K1 with programmatic stream serialization (PDL); one warp
// per row, the lane-column layout chosen by d.
template <int V, int NC, int BO>
cudaError_t launch_k2_t(const K1Args& a, int64_t blocks, int warps, bool exchange, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(blocks < 1 ? 1 : blocks));
    cfg.blockDim = dim3(32 * warps);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = exchange ? prefer_max_smem(k2_exchange<V, NC, BO, 1>) : prefer_max_smem(k2_combine<V, NC, BO>);
    if (e != cudaSuccess) return e;
    return exchange ? cudaLaunchKernelEx(&cfg, k2_exchange<V, NC, BO, 1>, a)
                    : cudaLaunchKernelEx(&cfg, k2_combine<V, NC, BO>, a);
}

// One warp per output row, one warp per block, at most one block per SM (ctas
// blocks): large row counts (batch x heads) loop over the warps. Every extra
// resident K2 warp measurably slows the neighbouring K1 under PDL: with 1024
// rows (cfg4), one warp per row made the step 7 % slower, and 4-warp blocks
// (592 warps) were as slow; 148 single warps match the serial launch. The
// longer K2 tail (~13 us at 1024 rows) is the cheaper side of that trade.
cudaError_t launch_k2(const K1Args& a, int64_t max_blocks, bool exchange, cudaStream_t st) {
    const int64_t rows = a.bh_count * a.group;
    static const int cap = [] { const char* e = std::getenv("TD_K2_MAX_BLOCKS"); return e ? std::atoi(e) : 0; }();
    int64_t limit = cap > 0 ? cap : (a.ctas > 0 ? a.ctas : 1);
    if (limit > max_blocks) limit = max_blocks;
    static const int force_w = [] { const char* e = std::getenv("TD_K2_WARPS"); return e ? std::atoi(e) : 0; }();
    int warps = force_w > 0 ? force_w : 1;
    warps = warps < 1 ? 1 : (warps > K2_THREADS / 32 ? K2_THREADS / 32 : warps);
    int64_t blocks = (rows + warps - 1) / warps;
    if (blocks > limit) blocks = limit;
#define TD_K2(VV, NN, BB) launch_k2_t<VV, NN, BB>(a, blocks, warps, exchange, st)
    static const int cols = [] { const char* e = std::getenv("TD_K2_COLS"); return e ? std::atoi(e) : 4; }();
    // few rows with many candidate states each (e.g. one row over every CTA): split
    // each (row, quarter)'s candidates over the warps of a block
    // CTAs covering a row, plus the chunk states of the deterministic pool
    // (streamed combine: K2 merges every warp's state, and only the split kernels can)
    const bool stream = a.sflag != nullptr;
    const int64_t cands = (a.bh_count > 0 ? int64_t(a.ctas) / a.bh_count + 2 : 0) * (stream ? a.slot_warps : 1) +
                          (a.dpool ? a.fslots : 0);
    static const int split_env = [] { const char* e = std::getenv("TD_K2_SPLIT"); return e ? std::atoi(e) : 1; }();
    const bool split = stream || (split_env && force_w == 0 && cands > 32 && !a.dbg);
    if (stream && a.d != 128) return cudaErrorInvalidValue;
    if (split && exchange && a.d == 128) {
        const int64_t units = rows * 4;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(units < limit ? units : limit));
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (stream) {
            cfg.blockDim = dim3(32 * 8);
            if (cudaError_t e = prefer_max_smem(k2_exchange_split<4, 8, true>)) return e;
            return cudaLaunchKernelEx(&cfg, k2_exchange_split<4, 8, true>, a);
        }
        if (cands > 128) {
            cfg.blockDim = dim3(32 * 8);
            if (cudaError_t e = prefer_max_smem(k2_exchange_split<4, 8>)) return e;
            return cudaLaunchKernelEx(&cfg, k2_exchange_split<4, 8>, a);
        }
        cfg.blockDim = dim3(32 * 4);
        if (cudaError_t e = prefer_max_smem(k2_exchange_split<4, 4>)) return e;
        return cudaLaunchKernelEx(&cfg, k2_exchange_split<4, 4>, a);
    }
    if (split && !exchange && a.d == 128) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(rows * 4 < limit ? rows * 4 : limit));
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (stream) {
            cfg.blockDim = dim3(32 * 8);
            if (cudaError_t e = prefer_max_smem(k2_combine_split<4, 8, true>)) return e;
            return cudaLaunchKernelEx(&cfg, k2_combine_split<4, 8, true>, a);
        }
        if (cands > 128) {
            cfg.blockDim = dim3(32 * 8);
            if (cudaError_t e = prefer_max_smem(k2_combine_split<4, 8>)) return e;
            return cudaLaunchKernelEx(&cfg, k2_combine_split<4, 8>, a);
        }
        cfg.blockDim = dim3(32 * 4);
        if (cudaError_t e = prefer_max_smem(k2_combine_split<4, 4>)) return e;
        return cudaLaunchKernelEx(&cfg, k2_combine_split<4, 4>, a);
    }
    // many rows (rows x 4 > the block cap, e.g. cfg4's 1024): (row, quarter) warp units
    // over 4-warp blocks, TD_K2_WIDE (4) blocks per SM (the exchange: at most its
    // co-resident warp budget), launched after K1 completes -- no programmatic
    // overlap, so no parked K2 warps next to K1, and 4-16 times the warps of the
    // single-warp PDL launch below. cfg4 at N=1: 1201.9-1203.7 (4 per SM) / 1207.2-1210.3
    // (2) / 1214.5-1221.1 (1) / 1225.1-1226.1 us (PDL); N=4: 340.4-343.2 vs 362.9-364.3
    // (profiles/r2_k2_wide/); TD_K2_WIDE=0 restores the PDL launch
    static const int wide = [] { const char* e = std::getenv("TD_K2_WIDE"); return e ? std::atoi(e) : 4; }();
    // (an exchange among workers sharing a GPU keeps the old launch: their grids must
    // all be co-resident, and four times the warps per worker might not be)
    if (wide && a.d == 128 && force_w == 0 && rows * 4 > limit && !a.dbg && !stream && (a.solo || !exchange)) {
        const int64_t units = rows * 4;
        int64_t blk = (units + 3) / 4;
        const int64_t bcap = std::min<int64_t>(int64_t(wide) * (a.ctas > 0 ? a.ctas : 1),  // wide blocks per SM
                                               std::max<int64_t>(1, max_blocks / 4));
        if (blk > bcap) blk = bcap;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(blk));
        cfg.blockDim = dim3(128);
        cfg.stream = st;
        cfg.numAttrs = 0;
        cudaError_t e = exchange ? prefer_max_smem(k2_exchange<1, 1, 32, 4>) : prefer_max_smem(k2_combine_cols<4>);
        if (e != cudaSuccess) return e;
        return exchange ? cudaLaunchKernelEx(&cfg, k2_exchange<1, 1, 32, 4>, a)
                        : cudaLaunchKernelEx(&cfg, k2_combine_cols<4>, a);
    }
    if (cols == 4 && a.d == 128 && force_w == 0 && rows * 4 <= limit && !a.dbg) {
        const int64_t b4 = rows * 4;  // one (row, column quarter) per single-warp block
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(b4 < 1 ? 1 : b4));
        cfg.blockDim = dim3(32);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t e = exchange ? prefer_max_smem(k2_exchange<1, 1, 32, 4>) : prefer_max_smem(k2_combine_cols<4>);
        if (e != cudaSuccess) return e;
        return exchange ? cudaLaunchKernelEx(&cfg, k2_exchange<1, 1, 32, 4>, a)
                        : cudaLaunchKernelEx(&cfg, k2_combine_cols<4>, a);
    }
    if (a.d % 4 == 0 && a.d <= 128) return TD_K2(4, 1, 32);
    if (a.d % 4 == 0) return TD_K2(4, 2, 16);
    return TD_K2(1, 8, 8);
#undef TD_K2
}

}  // namespace

const void* k1_function(const SplitPlan& p) {
    if (p.kernel == 1) {
        switch (p.d) {
        case 64: return reinterpret_cast<const void*>(k1_bf16<64, kBf16Tile, bf16_warps(64), bf16_stages(64)>);
        case 128: return reinterpret_cast<const void*>(k1_bf16<128, kBf16Tile, bf16_warps(128), bf16_stages(128)>);
        case 256: return reinterpret_cast<const void*>(k1_bf16<256, kBf16Tile, bf16_warps(256), bf16_stages(256)>);
        default: return nullptr;
        }
    }
    if (p.kernel == 2) {
#define TD_F32_FN(TT, WW, EE) \
    (p.group == 1 ? reinterpret_cast<const void*>(k1_f32<TT, WW, EE, 1>) \
                  : reinterpret_cast<const void*>(k1_f32<TT, WW, EE, 2>))
        switch (f32_cfg()) {
        case 1: return TD_F32_FN(32, 2, 6);
        case 2: return TD_F32_FN(32, 6, 2);
        case 3: return TD_F32_FN(16, 4, 4);
        case 4: return TD_F32_FN(32, 4, 3);
        case 5: return TD_F32_FN(32, 3, 4);
        case 6: return TD_F32_FN(16, 6, 4);
        case 7: return TD_F32_FN(16, 8, 2);
        default: return TD_F32_FN(32, 4, 2);
        }
#undef TD_F32_FN
    }
    return p.dtype == kBF16 ? reinterpret_cast<const void*>(k1_generic<__nv_bfloat16>)
                            : reinterpret_cast<const void*>(k1_generic<float>);
}

cudaError_t graph_set_k1_epoch(cudaGraphExec_t exec, cudaGraphNode_t node, const SplitPlan& p) {
    cudaKernelNodeParams kp{};
    cudaError_t e = cudaGraphKernelNodeGetParams(node, &kp);
    if (e != cudaSuccess) return e;
    K1Args a = *static_cast<const K1Args*>(kp.kernelParams[0]);
    a.epoch = p.epoch;
    a.sepoch = p.sepoch;
    void* args[3] = {&a, nullptr, nullptr};
    if (p.kernel == 1) {  // k1_bf16(K1Args, CUtensorMap, CUtensorMap)
        args[1] = kp.kernelParams[1];
        args[2] = kp.kernelParams[2];
    }
    kp.kernelParams = args;
    return cudaGraphExecKernelNodeSetParams(exec, node, &kp);
}

const void* k2_stream_function() { return reinterpret_cast<const void*>(k2_combine_split<4, 8, true>); }

cudaError_t graph_set_k2_epoch(cudaGraphExec_t exec, cudaGraphNode_t node, const SplitPlan& p) {
    cudaKernelNodeParams kp{};
    cudaError_t e = cudaGraphKernelNodeGetParams(node, &kp);
    if (e != cudaSuccess) return e;
    K1Args a = *static_cast<const K1Args*>(kp.kernelParams[0]);
    a.sepoch = p.sepoch;
    void* args[1] = {&a};
    kp.kernelParams = args;
    return cudaGraphExecKernelNodeSetParams(exec, node, &kp);
}

cudaError_t launch_decode_partial(const SplitPlan& p, const void* q, const void* k,
                                  const void* v, float scale, const CUtensorMap* tmk,
                                  const CUtensorMap* tmv, void* ws, float* row_max, float* lse,
                                  float* out, cudaStream_t st, cudaEvent_t ev0,
                                  cudaEvent_t ev1, const void* src) {
    if (src && p.kernel != 0) return cudaErrorInvalidValue;  // the source term lives in k1_generic
    K1Args a = make_args(p, q, k, v, scale, ws);
    a.src = src;
    a.tail.mode = kTailPartial;
    a.tail.row_max = row_max;
    a.tail.lse = lse;
    a.tail.out = out;
    cudaError_t e = launch_k1(p, a, tmk, tmv, st, ev0, ev1);
    if (e != cudaSuccess) return e;
    return launch_k2(a, 4096, false, st);
}

cudaError_t launch_decode_final(const SplitPlan& p, const void* q, const void* k, const void* v,
                                float scale, const CUtensorMap* tmk, const CUtensorMap* tmv,
                                void* ws, float* out, cudaStream_t st, cudaEvent_t ev0,
                                cudaEvent_t ev1) {
    K1Args a = make_args(p, q, k, v, scale, ws);
    a.tail.mode = kTailFinal;
    a.tail.out = out;
    cudaError_t e = launch_k1(p, a, tmk, tmv, st, ev0, ev1);
    if (e != cudaSuccess) return e;
    return launch_k2(a, 4096, false, st);
}

cudaError_t launch_decode_exchange(const SplitPlan& p, const void* q, const void* k, const void* v,
                                   float scale, const CUtensorMap* tmk, const CUtensorMap* tmv,
                                   void* ws, const XchgArgs& xa, float* out, cudaStream_t st,
                                   cudaEvent_t ev0, cudaEvent_t ev1, int parts) {
    K1Args a = make_args(p, q, k, v, scale, ws);
    a.tail.mode = kTailExchange;
    a.tail.out = out;
    a.tail.x.peers = xa.peers;
    a.tail.x.p = xa.p;
    a.tail.x.rank = xa.rank;
    a.tail.x.epoch = xa.epoch;
    a.tail.x.max_rows = xa.max_rows;
    a.tail.x.error = xa.error;
    a.tail.x.pull = xa.pull;
    if (parts & 1) {
        cudaError_t e = launch_k1(p, a, tmk, tmv, st, ev0, ev1);
        if (e != cudaSuccess) return e;
    }
    return (parts & 2) ? launch_k2(a, xa.max_blocks, true, st) : cudaSuccess;
}

namespace {
unsigned grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > 148 * 16) g = 148 * 16;
    return static_cast<unsigned>(g);
}
}  // namespace

cudaError_t launch_decode_literal(const SplitPlan& p, const void* q, const void* k, const void* v, float scale,
                                  const CUtensorMap* tmk, const CUtensorMap* tmv, void* ws, const XchgArgs& xa,
                                  float* out, cudaStream_t st, cudaEvent_t ev0, cudaEvent_t ev1) {
    K1Args a = make_args(p, q, k, v, scale, ws);
    if (!a.sflag || a.bh_count * a.group * 4 > xa.max_blocks || a.bh_count * a.group * 4 > a.ctas)
        return cudaErrorInvalidValue;  // the fused literal combine needs the streamed split K2x, one unit per block
    a.tail.mode = kTailLiteral;
    a.tail.out = out;
    a.tail.x.peers = xa.peers;
    a.tail.x.p = xa.p;
    a.tail.x.rank = xa.rank;
    a.tail.x.epoch = xa.epoch;
    a.tail.x.max_rows = xa.max_rows;
    a.tail.x.error = xa.error;
    a.tail.x.pull = 0;
    cudaError_t e = launch_k1(p, a, tmk, tmv, st, ev0, ev1);
    if (e != cudaSuccess) return e;
    return launch_k2(a, xa.max_blocks, true, st);
}

cudaError_t launch_literal_combine(const float* lse, const float* o, const XchgArgs& xa, int64_t rows, int d,
                                   float* out, cudaStream_t st) {
    const int grid = static_cast<int>(std::min<int64_t>(rows, xa.max_blocks));
    if (grid < 1) return cudaSuccess;
    switch ((d + 31) / 32) {
        case 1: return launch_pdl(k2n_literal<1>, grid, 32, 0, st, true, lse, o, xa, rows, d, out);
        case 2: return launch_pdl(k2n_literal<2>, grid, 32, 0, st, true, lse, o, xa, rows, d, out);
        case 3:
        case 4: return launch_pdl(k2n_literal<4>, grid, 32, 0, st, true, lse, o, xa, rows, d, out);
        default: return launch_pdl(k2n_literal<8>, grid, 32, 0, st, true, lse, o, xa, rows, d, out);
    }
}

cudaError_t launch_to_numerator(const float* lse, const float* out, const float* shift,
                                int64_t rows, int d, float* nd, cudaStream_t st) {
    k3_to_numerator<<<grid_for(rows * d + rows, 256), 256, 0, st>>>(lse, out, shift, rows, d, nd);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const float* nd, int64_t rows, int d, float* out, void* out_bf16,
                            cudaStream_t st) {
    k4_finalize<<<grid_for(rows * d, 256), 256, 0, st>>>(nd, rows, d, out,
                                                          static_cast<__nv_bfloat16*>(out_bf16));
    return cudaGetLastError();
}

__global__ void k_to_bf16(const float* src, int64_t n, __nv_bfloat16* dst) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = __float2bfloat16_rn(src[i]);
}

cudaError_t launch_to_bf16(const float* src, int64_t n, void* dst, cudaStream_t st) {
    if (n < 1) return cudaSuccess;
    k_to_bf16<<<grid_for(n, 256), 256, 0, st>>>(src, n, static_cast<__nv_bfloat16*>(dst));
    return cudaGetLastError();
}

cudaError_t launch_combine_pair(float* l_max, float* l_lse, float* l_out, const float* r_max,
                                const float* r_lse, const float* r_out, int64_t rows, int d,
                                cudaStream_t st) {
    if (rows < 1) return cudaSuccess;
    k5_combine_pair<<<static_cast<unsigned>(rows), 128, 0, st>>>(l_max, l_lse, l_out, r_max, r_lse,
                                                                  r_out, rows, d);
    return cudaGetLastError();
}

cudaError_t launch_combine_partials(int P, const float* lse, const float* out, int64_t rows,
                                    int d, float* result, int* bad_row, cudaStream_t st) {
    if (rows < 1) return cudaSuccess;
    k_combine_partials<<<static_cast<unsigned>(rows), 128, 0, st>>>(P, lse, out, rows, d, result,
                                                                     bad_row);
    return cudaGetLastError();
}

// ---- energy formulation (energy.cpp:152-259) -------------
// Per row, from P partials (row_max, lse natural log) of disjoint key chunks:
// row_max = max_c row_max_c, shifted = log sum_c e^(lse_c - row_max), value =
// row_max + shifted -- the tree max and lse reductions of
// energy_forward_parallel. Empty rows give (-inf, -inf, -inf).
__global__ void k_energy_combine(int P, const float* rmax, const float* lse, int64_t rows, float* value,
                                 float* rmax_out, float* shifted) {
    const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (r >= rows) return;
    float m = -CUDART_INF_F;
    for (int c = 0; c < P; ++c) m = fmaxf(m, rmax[c * rows + r]);
    float s = 0.f;
    if (m != -CUDART_INF_F)
        for (int c = 0; c < P; ++c) {
            const float l = lse[c * rows + r];
            if (l != -CUDART_INF_F) s += expf(l - m);
        }
    const float sh = m == -CUDART_INF_F ? -CUDART_INF_F : logf(s);
    rmax_out[r] = m;
    shifted[r] = sh;
    value[r] = m == -CUDART_INF_F ? -CUDART_INF_F : m + sh;
}

// grad = sum_c e^(lse_c - F) out_c with F = row_max + shifted (the saved
// forward): energy_grad_parallel's per-chunk sums sum_a e^(s_a - F) v_a, since a
// chunk partial holds out_c = sum_a e^(s_a - lse_c) v_a.
__global__ void k_energy_grad_combine(int P, const float* lse, const float* out, const float* rmax,
                                      const float* shifted, int64_t rows, int d, float* grad) {
    const int64_t n = rows * d;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / d;
        const float f = rmax[r] + shifted[r];
        float g = 0.f;
        for (int c = 0; c < P; ++c) {
            const float l = lse[c * rows + r];
            if (l != -CUDART_INF_F) g += expf(l - f) * out[c * n + i];
        }
        grad[i] = g;
    }
}

// Distributed forward, step 2 (after allreduce(max) of row_max into m):
// x = e^(lse - m); step 3 (after allreduce(sum) of x into s): the outputs.
__global__ void k_energy_shift(const float* lse, const float* m, int64_t rows, float* x) {
    const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (r < rows) x[r] = (lse[r] == -CUDART_INF_F || m[r] == -CUDART_INF_F) ? 0.f : expf(lse[r] - m[r]);
}
__global__ void k_energy_finish(const float* m, const float* s, int64_t rows, float* value, float* rmax_out,
                                float* shifted) {
    const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (r >= rows) return;
    const float mm = m[r];
    const float sh = mm == -CUDART_INF_F ? -CUDART_INF_F : logf(s[r]);
    rmax_out[r] = mm;
    shifted[r] = sh;
    value[r] = mm == -CUDART_INF_F ? -CUDART_INF_F : mm + sh;
}
// F = row_max + shifted (the log partition function of the saved forward)
__global__ void k_energy_logz(const float* rmax, const float* shifted, int64_t rows, float* f) {
    const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (r < rows) f[r] = rmax[r] + shifted[r];
}

cudaError_t launch_energy_combine(int P, const float* rmax, const float* lse, int64_t rows, float* value,
                                  float* rmax_out, float* shifted, cudaStream_t st) {
    k_energy_combine<<<grid_for(rows, 256), 256, 0, st>>>(P, rmax, lse, rows, value, rmax_out, shifted);
    return cudaGetLastError();
}
cudaError_t launch_energy_grad_combine(int P, const float* lse, const float* out, const float* rmax,
                                       const float* shifted, int64_t rows, int d, float* grad, cudaStream_t st) {
    k_energy_grad_combine<<<grid_for(rows * d, 256), 256, 0, st>>>(P, lse, out, rmax, shifted, rows, d, grad);
    return cudaGetLastError();
}
cudaError_t launch_energy_shift(const float* lse, const float* m, int64_t rows, float* x, cudaStream_t st) {
    k_energy_shift<<<grid_for(rows, 256), 256, 0, st>>>(lse, m, rows, x);
    return cudaGetLastError();
}
cudaError_t launch_energy_finish(const float* m, const float* s, int64_t rows, float* value, float* rmax_out,
                                 float* shifted, cudaStream_t st) {
    k_energy_finish<<<grid_for(rows, 256), 256, 0, st>>>(m, s, rows, value, rmax_out, shifted);
    return cudaGetLastError();
}
cudaError_t launch_energy_logz(const float* rmax, const float* shifted, int64_t rows, float* f, cudaStream_t st) {
    k_energy_logz<<<grid_for(rows, 256), 256, 0, st>>>(rmax, shifted, rows, f);
    return cudaGetLastError();
}

// ---- KV append: one new token per (b, kv-head) row ---------
// A kernel rather than two strided copies so that it keeps the stream's
// programmatic-launch chain: it starts under the previous step's K2 and the
// next K1 starts under it. Row r of the shard receives the token at position
// pos (rows are cap tokens apart).
__global__ void k_kv_append(uint16_t* kc, uint16_t* vc, const uint16_t* kt, const uint16_t* vt, int64_t rows,
                            int64_t pitch, int64_t pos, int words) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t n = rows * words;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / words, j = i - r * words;
        const int64_t dst = r * pitch + pos * words + j;
        kc[dst] = kt[i];
        vc[dst] = vt[i];
    }
}

cudaError_t launch_kv_append(int dtype, void* k, void* v, const void* kt, const void* vt, int64_t rows,
                             int64_t cap, int64_t pos, int d, cudaStream_t st) {
    const int words = d * dtype_bytes(dtype) / 2;  // 16-bit words per token row
    const int64_t n = rows * words;
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, 1024));
    return launch_pdl(k_kv_append, grid < 1 ? 1 : grid, 256, 0, st, true, static_cast<uint16_t*>(k),
                      static_cast<uint16_t*>(v), static_cast<const uint16_t*>(kt), static_cast<const uint16_t*>(vt),
                      rows, cap * words, pos, words);
}

cudaError_t launch_seeded_fill(int dtype, void* dst, uint64_t seed, double scale,
                               int64_t bh_count, int64_t seq, int64_t start, int64_t len,
                               int64_t d, cudaStream_t st) {
    const int64_t n = bh_count * len * d;
    if (n == 0) return cudaSuccess;
    const double half_width = __builtin_sqrt(3.0) * scale;
    k6_seeded_fill<<<grid_for(n, 256), 256, 0, st>>>(dtype, dst, seed, half_width, bh_count, seq,
                                                       start, len, d);
    return cudaGetLastError();
}

}  // namespace td
