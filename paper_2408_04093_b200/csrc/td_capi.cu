// td_capi.cu -- C-ABI of the B200 tree-decode library (include/treedec_b200.h).
//
// One td_context per GPU / rank. The tree path is the paper's Algorithm 3
// as the reference implements it in tree_decode
// (decode.cpp:100-184): local partial (K1+K2) -> nccl().AllReduce(max) of lse
// -> K3 rescale -> one fused nccl().AllReduce(sum) of [n|d] -> K4 n/d. The ring
// path is ring_decode (decode.cpp:186-251) with the KV shards really moving
// (ncclSend/ncclRecv), overlapped with the partial of the chunk in hand.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/treedec_b200.h"
#include "td_internal.h"

using td::SplitPlan;

namespace {

thread_local std::string g_err;
int g_deterministic = 1;  // td_set_deterministic: static split by default (bitwise reproducible)

// Static split (bitwise reproducible) unless the call or the process asks for the
// dynamic pool: TD_DETERMINISTIC forces it on, TD_DYNAMIC off, else the
// process setting (td_set_deterministic, on by default).
bool call_deterministic(int flags) {
    if (flags & TD_DETERMINISTIC) return true;
    if (flags & TD_DYNAMIC) return false;
    return g_deterministic != 0;
}

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define TD_CUDA(call)                                                                  \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess)                                                         \
            return set_err(TD_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define TD_NCCL(call)                                                                    \
    do {                                                                                 \
        if (!nccl().ok) return set_err(TD_ENCCL, nccl().err);                            \
        ncclResult_t r_ = (call);                                                        \
        if (r_ != ncclSuccess)                                                           \
            return set_err(TD_ENCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
    } while (0)

// NCCL is resolved at run time: if the process already holds a libnccl.so.2
// (torch loads its own), that copy is used, so the library never forces a
// second, older NCCL into a torch process.
struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    // symmetric memory (NCCL >= 2.27, optional): registered windows let NCCL run its
    // low-latency symmetric kernels for the two small allreduces
    ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
    ncclResult_t (*MemFree)(void*) = nullptr;
    ncclResult_t (*WindowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
    ncclResult_t (*WindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
    bool symmetric() const { return MemAlloc && MemFree && WindowRegister && WindowDeregister; }
    // device API (NCCL >= 2.28): the load/store-accessible team of this rank
    struct Team {
        int nRanks, rank, stride;
    };
    Team (*TeamLsa)(ncclComm_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.err = std::string("libnccl.so.2 not loadable: ") + dlerror();
            return a;
        }
        bool all = true;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            all = all && fn != nullptr;
        };
        sym(a.GetUniqueId, "ncclGetUniqueId");
        sym(a.CommInitRank, "ncclCommInitRank");
        sym(a.CommDestroy, "ncclCommDestroy");
        sym(a.AllReduce, "ncclAllReduce");
        sym(a.Send, "ncclSend");
        sym(a.Recv, "ncclRecv");
        sym(a.GroupStart, "ncclGroupStart");
        sym(a.GroupEnd, "ncclGroupEnd");
        sym(a.GetErrorString, "ncclGetErrorString");
        sym(a.GetVersion, "ncclGetVersion");
        a.ok = all;
        auto opt = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
        };
        opt(a.MemAlloc, "ncclMemAlloc");
        opt(a.MemFree, "ncclMemFree");
        opt(a.WindowRegister, "ncclCommWindowRegister");
        opt(a.WindowDeregister, "ncclCommWindowDeregister");
        opt(a.TeamLsa, "ncclTeamLsa");
        if (!all) a.err = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    return api;
}

int sm_count_of(int device) {
    int n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n;
}

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaSuccess) cap = bytes;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <typename T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

std::vector<int64_t> chunk_extents(int64_t n, int p) {  // attention.cpp:268-275
    std::vector<int64_t> ext(static_cast<size_t>(p), n / p);
    for (int64_t i = 0; i < n % p; ++i) ext[static_cast<size_t>(i)] += 1;
    return ext;
}

}  // namespace

struct td_context {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;  // compute
    cudaStream_t xfer = nullptr;    // ring send/recv
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;

    // placed KV shard ([b][n_kv][len][d])
    bool kv_ok = false;
    int dtype = td::kBF16;
    int64_t b = 0, n_kv = 0, seq_len = 0, d = 0, start = 0, len = 0;
    int64_t cap = 0;  // tokens per bh row allocated (>= len: room for td_kv_append)
    // tokens of every row that no kernel still in flight may be writing: the whole
    // cache after a synchronising placement, else the length the last decode's K1
    // saw (appends write past it); SplitPlan::t_safe
    int64_t kv_safe = 0;
    // fused KV append: a device-source token appended since the last decode that the
    // next bf16 split kernel writes into the cache itself (SplitPlan::app_*); any other
    // reader of the cache flushes it first with the append kernel (flush_append)
    const void* pend_k = nullptr;
    const void* pend_v = nullptr;
    int64_t pend_pos = -1;
    std::vector<int64_t> lens;  // every rank's shard length (chunk_extents, then appends on rank p-1)
    DevBuf k, v;
    CUtensorMap tmk{}, tmv{};
    bool tm_ok = false;

    DevBuf ws;                                   // split slots
    DevBuf rows;                                 // per-row fp32 buffers
    float *row_max = nullptr, *lse = nullptr, *out_local = nullptr, *shift = nullptr,
          *nd = nullptr, *out = nullptr, *r_max = nullptr, *r_lse = nullptr, *r_out = nullptr;
    DevBuf q_dev, out_bf16;
    DevBuf ring[2][2];                           // [buffer][k|v]
    DevBuf ring_own[2];                          // own shard packed contiguously (cap > len)
    std::vector<cudaEvent_t> ring_ev;            // compute-done / recv-done

    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timers;
    size_t timers_used = 0;
    // TD_TIME_PHASES: per call, up to 8 marks
    std::vector<std::vector<cudaEvent_t>> phase_sets;
    size_t phase_used = 0;
    std::vector<cudaEvent_t>* cur_phase = nullptr;
    size_t cur_mark = 0;

    int last_kernels = 0;
    double last_kv_bytes = 0.0;
    int last_split_kernel = -1;

    // one-shot NVLink exchange (td_p2p_*)
    DevBuf xbuf;                      // [2][p][max_rows][d + 1] LL words (value, epoch)
    int64_t x_max_rows = 0, x_d = 0;
    std::vector<void*> x_opened;      // IPC mappings to close
    DevBuf x_ptrs;                    // device array: peers[p]
    int* x_err = nullptr;             // exchange timeout flag, mapped pinned host memory (K2x stores 1)
    unsigned x_epoch = 0;
    bool x_ready = false;

    // debug instrumentation of the current call (debug_begin), copied into every plan
    unsigned long long* cur_dbg = nullptr;
    unsigned long long* cur_tl = nullptr;
    unsigned long long* cur_tl_cta = nullptr;
    bool shared_device = false;       // another context of this process runs on the same GPU (td_group)

    // TD_PINNED_IO fast path: the K2 warp counter (device) and the completion
    // word (mapped pinned host memory)
    DevBuf sig;
    unsigned* done_host = nullptr;
    unsigned done_epoch = 0;
    int host_ptr_ok = -1;             // pinned host pointers usable by kernels as is (UVA), probed once

    // streamed combine (SplitPlan::sflag): flag words, the last launch's epoch and the
    // timeout word (mapped pinned host memory)
    DevBuf sflags;
    unsigned s_epoch = 0;
    int* s_err = nullptr;

    DevBuf dbg;  // TD_DEBUG_TS stamps
    int64_t tl_count = -1;  // TD_DEBUG_TIMELINE: calls stamped so far (-1: not initialised)
    float* mapped_for = nullptr;   // this call's host output buffer and its device alias (or null)
    float* mapped_dev = nullptr;
    DevBuf tlbuf;           // TD_DEBUG_TIMELINE stamps (read back as dbg[5000..6144))

    // calibrated static partition: per-CTA streaming speed of this GPU's SMs
    // (blocks land on the same SMs launch after launch), measured once
    std::vector<float> cal_w;
    bool cal_failed = false;
    int64_t cal_bytes = 0;      // KV bytes of the shard the weights were measured on
    double cal_gain = 0.0;      // measured K1 gain of the weights over the equal split
    DevBuf sm_map, claims;      // SM affinity of the calibrated CTA indices
    bool sm_map_ok = false;
    unsigned claim_epoch = 0;
    DevBuf cal_q;
    struct PartTab {
        int64_t total = -1, per_bh = 0, bh = 0;
        int ctas = 0, maxseg = 0;
        DevBuf buf;                   // int64 x[ctas + 1] then int bh[3 * bh_count]
        void* host = nullptr;         // pinned staging of the tables (async upload)
        size_t host_cap = 0;
        cudaEvent_t used = nullptr;   // after the last launch that read buf
    };
    PartTab tabs[4];
    int tab_next = 0;
    unsigned tabs_touched = 0;        // entries selected since the last note_table_use

    bool det = false;  // this call: static split only (TD_DETERMINISTIC)
    // paper-literal NCCL combine: [lse | shift | n, d] of the step in one
    // ncclMemAlloc block registered as a symmetric window (collective, once per size)
    void* win_buf = nullptr;
    size_t win_bytes = 0;
    ncclWindow_t win = nullptr;
    int win_state = 0;  // 0 untried, 1 registered, -1 unavailable (plain buffers)
    // TD_NCCL_DEVICE: K2n's LL words in a second symmetric window; nx_ptrs holds
    // every rank's copy's address (ncclGetLsaPointer)
    void* nx_buf = nullptr;
    ncclWindow_t nx_win = nullptr;
    int64_t nx_rows = 0, nx_d = 0;
    DevBuf nx_ptrs;
    unsigned nx_epoch = 0;
    bool nx_ready = false;

    // TD_GRAPH: the paper-literal NCCL step (K1, K2, allreduce(max), K3,
    // allreduce(sum), K4) captured once per shape and replayed; only the split
    // kernel's SM-affinity claim epoch changes between replays
    struct Graph {
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaGraphNode_t k1 = nullptr;
        cudaGraphNode_t k2s = nullptr;  // the streamed split K2 (null without the streamed combine)
        const unsigned* sflag = nullptr;
        const void* q = nullptr;
        float* out = nullptr;
        double scale = 0.0;
        int64_t rows = 0, total = -1, per_bh = 0, len = 0, cap = 0, t_safe = -1;
        int ctas = 0, maxseg = 0, kernel = -1;
        const void* x_table = nullptr;
        const void* k = nullptr;
        float* lse = nullptr;
    } graph[2];  // one per pool-counter parity (launches alternate them)

    DevBuf ctr;        // K1 dynamic-pool counters (SplitPlan::counters)
    int64_t ctr_bh = -1;
    int kpar = 0;      // parity of the next launch
};

namespace {

int require_ctx(td_context* ctx) {
    if (!ctx) return set_err(TD_EINVAL, "null td_context");
    cudaSetDevice(ctx->device);
    return TD_OK;
}

// per-row buffers for rows = b * n_q (max) and d
int ensure_rows(td_context* ctx, int64_t rows, int64_t d) {
    const size_t rd = size_t(rows) * size_t(d), r = size_t(rows);
    auto pad = [](size_t n) { return (n + 15) / 16 * 16; };
    // row_max, lse, shift, r_max, r_lse: r each; out_local, out, r_out: rd; nd: rd + r
    const size_t floats = 5 * pad(r) + 3 * pad(rd) + pad(rd + r);
    TD_CUDA(ctx->rows.ensure(floats * sizeof(float)));
    float* f = ctx->rows.as<float>();
    auto take = [&](size_t n) {
        float* p = f;
        f += (n + 15) / 16 * 16;
        return p;
    };
    ctx->row_max = take(r);
    ctx->lse = take(r);
    ctx->shift = take(r);
    ctx->r_max = take(r);
    ctx->r_lse = take(r);
    ctx->out_local = take(rd);
    ctx->out = take(rd);
    ctx->r_out = take(rd);
    ctx->nd = take(rd + r);
    return TD_OK;
}

// The pending fused append as an append kernel, for every reader of the cache
// other than the bf16 split kernel (and before the cache is reallocated).
int flush_append(td_context* ctx) {
    if (!ctx->pend_k) return TD_OK;
    const void* k = ctx->pend_k;
    const void* v = ctx->pend_v;
    ctx->pend_k = ctx->pend_v = nullptr;
    TD_CUDA(td::launch_kv_append(ctx->dtype, ctx->k.p, ctx->v.p, k, v, ctx->b * ctx->n_kv, ctx->cap, ctx->pend_pos,
                                 static_cast<int>(ctx->d), ctx->stream));
    ctx->pend_pos = -1;
    return TD_OK;
}

bool calibration_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TD_CALIBRATE");
        return !e || std::atoi(e) != 0;
    }();
    return on;
}

bool sm_affinity_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TD_SM_AFFINITY");
        return !e || std::atoi(e) != 0;
    }();
    return on;
}

// Device tables of the speed-weighted static partition of `plan` (cached).
// After the launches of a call: the selected partition tables are in use up to here.
int note_table_use(td_context* ctx) {
    for (int i = 0; i < 4; ++i) {
        if (!(ctx->tabs_touched & (1u << i))) continue;
        auto& tb = ctx->tabs[i];
        if (!tb.used) TD_CUDA(cudaEventCreateWithFlags(&tb.used, cudaEventDisableTiming));
        TD_CUDA(cudaEventRecord(tb.used, ctx->stream));
    }
    ctx->tabs_touched = 0;
    return TD_OK;
}

int apply_partition(td_context* ctx, SplitPlan& plan) {
    for (int i = 0; i < 4; ++i) {
        auto& tb = ctx->tabs[i];
        if (tb.total == plan.total_tiles && tb.per_bh == plan.tiles_per_bh && tb.bh == plan.bh_count &&
            tb.ctas == plan.ctas) {
            plan.maxseg = std::max(plan.maxseg, tb.maxseg);
            plan.x_table = static_cast<const int64_t*>(tb.buf.p);
            plan.bh_table = reinterpret_cast<const int*>(static_cast<const int64_t*>(tb.buf.p) + plan.ctas + 1);
            ctx->tabs_touched |= 1u << i;
            return TD_OK;
        }
    }
    std::vector<int64_t> x(size_t(plan.ctas) + 1);
    std::vector<int> bh(3 * size_t(plan.bh_count));
    SplitPlan weighted = plan;
    td::build_partition(weighted, ctx->cal_w.data(), x.data(), bh.data());
    // the weighted ranges may cover more (batch, head) rows per CTA than the
    // kernels' per-warp segment masks hold: keep the equal split then
    if (weighted.maxseg > td::kMaxSegments) return TD_OK;
    plan.maxseg = weighted.maxseg;
    const int idx = ctx->tab_next;
    auto& tb = ctx->tabs[idx];
    ctx->tab_next = (ctx->tab_next + 1) % 4;
    const size_t xb = x.size() * sizeof(int64_t), bb = bh.size() * sizeof(int);
    // no stream drain when the sequence grows (a new shape every 32 appended tokens):
    // wait only for the last launch that read this entry, then upload from pinned
    // staging on the stream, ahead of the launch that will read it
    if (tb.used) TD_CUDA(cudaEventSynchronize(tb.used));
    if (tb.host_cap < xb + bb) {  // pinned allocations can stall the device: size generously, once
        if (tb.host) cudaFreeHost(tb.host);
        tb.host = nullptr;
        tb.host_cap = 0;
        const size_t want = std::max<size_t>(xb + bb, 64 * 1024);
        TD_CUDA(cudaMallocHost(&tb.host, want));
        tb.host_cap = want;
    }
    if (tb.buf.cap < xb + bb) TD_CUDA(tb.buf.ensure(std::max<size_t>(xb + bb, 64 * 1024)));
    std::memcpy(tb.host, x.data(), xb);
    std::memcpy(static_cast<char*>(tb.host) + xb, bh.data(), bb);
    TD_CUDA(tb.buf.ensure(xb + bb));
    TD_CUDA(cudaMemcpyAsync(tb.buf.p, tb.host, xb + bb, cudaMemcpyHostToDevice, ctx->stream));
    ctx->tabs_touched |= 1u << idx;
    tb.total = plan.total_tiles;
    tb.per_bh = plan.tiles_per_bh;
    tb.bh = plan.bh_count;
    tb.ctas = plan.ctas;
    tb.maxseg = plan.maxseg;
    plan.x_table = static_cast<const int64_t*>(tb.buf.p);
    plan.bh_table = reinterpret_cast<const int*>(static_cast<const int64_t*>(tb.buf.p) + plan.ctas + 1);
    return TD_OK;
}

int ensure_rows(td_context* ctx, int64_t rows, int64_t d);

// Measures how fast each CTA of the split kernel streams on this GPU (per-CTA
// globaltimer stamps, static split, two rounds: equal ranges, then ranges
// weighted by the first round's speeds) and keeps speed weights per CTA index
// together with the SM each index ran on (sm_map): later launches give index c
// to the CTA that lands on that SM, so the weights hold whatever order the CTAs
// launch in (e.g. early, under PDL). They only move work, never change what is
// computed.
int calibrate(td_context* ctx, int64_t n_q) {
    if (int rc = flush_append(ctx)) return rc;  // the calibration launches read the whole cache
    SplitPlan p;
    std::string msg;
    if (!td::plan_split(ctx->dtype, ctx->b, static_cast<int>(n_q), static_cast<int>(ctx->n_kv), ctx->len,
                        static_cast<int>(ctx->d), ctx->sm_count, p, msg, false) ||
        p.kernel != 1 || !ctx->tm_ok)
        return set_err(TD_EINVAL, "calibration not applicable");
    p.row_stride = ctx->cap;
    const int G = p.ctas;
    if (G > 1024) return set_err(TD_EINVAL, "calibration: too many CTAs");
    const int64_t rows = ctx->b * n_q;
    if (int rc = ensure_rows(ctx, rows, ctx->d)) return rc;
    TD_CUDA(ctx->cal_q.ensure(size_t(rows) * size_t(ctx->d) * 2));
    TD_CUDA(cudaMemsetAsync(ctx->cal_q.p, 0, size_t(rows) * size_t(ctx->d) * 2, ctx->stream));
    TD_CUDA(ctx->dbg.ensure(6144 * sizeof(unsigned long long)));
    std::vector<unsigned long long> st(6144);
    DevBuf tab;
    // one static-split launch under weights w (per CTA index); stamps into st;
    // returns the span first CTA start -> last CTA end (ns)
    auto run = [&](const std::vector<float>& w, const int* sm_to_cta, unsigned epoch, std::vector<int64_t>& x,
                   double& span) -> int {
        SplitPlan pr = p;
        x.assign(size_t(G) + 1, 0);
        std::vector<int> bh(3 * size_t(pr.bh_count));
        td::build_partition(pr, w.data(), x.data(), bh.data());
        if (pr.maxseg > td::kMaxSegments) return set_err(TD_EINVAL, "calibration: weighted ranges span too many rows");
        const size_t xb = x.size() * sizeof(int64_t), bb = bh.size() * sizeof(int);
        TD_CUDA(tab.ensure(xb + bb));
        TD_CUDA(cudaMemcpy(tab.p, x.data(), xb, cudaMemcpyHostToDevice));
        TD_CUDA(cudaMemcpy(static_cast<char*>(tab.p) + xb, bh.data(), bb, cudaMemcpyHostToDevice));
        pr.x_table = static_cast<const int64_t*>(tab.p);
        pr.bh_table = reinterpret_cast<const int*>(static_cast<const int64_t*>(tab.p) + G + 1);
        pr.sm_to_cta = sm_to_cta;
        pr.claims = static_cast<unsigned*>(ctx->claims.p);
        pr.epoch = epoch;
        TD_CUDA(ctx->ws.ensure(pr.workspace_bytes()));
        TD_CUDA(cudaMemsetAsync(ctx->dbg.p, 0, 6144 * sizeof(unsigned long long), ctx->stream));
        TD_CUDA(cudaMemsetAsync(ctx->dbg.p, 0xff, sizeof(unsigned long long), ctx->stream));
        pr.dbg = static_cast<unsigned long long*>(ctx->dbg.p);
        pr.tl = pr.tl_cta = nullptr;
        TD_CUDA(td::launch_decode_partial(pr, ctx->cal_q.p, ctx->k.p, ctx->v.p, 1.0f, &ctx->tmk, &ctx->tmv,
                                          ctx->ws.p, ctx->r_max, ctx->r_lse, ctx->r_out, ctx->stream));
        TD_CUDA(cudaMemcpyAsync(st.data(), ctx->dbg.p, st.size() * sizeof(unsigned long long),
                                cudaMemcpyDeviceToHost, ctx->stream));
        TD_CUDA(cudaStreamSynchronize(ctx->stream));
        span = st[1] > st[0] ? double(st[1] - st[0]) : 0.0;
        return TD_OK;
    };
    TD_CUDA(ctx->claims.ensure(size_t(G) * sizeof(unsigned)));
    TD_CUDA(cudaMemset(ctx->claims.p, 0, size_t(G) * sizeof(unsigned)));
    // 1. per-SM streaming speed: tiles / (end - start) of each CTA, indexed by the
    // SM it ran on (the SM, not the block index, is what is fast or slow), over
    // 3 rounds x 3 measured launches; each round re-weights the ranges
    std::vector<double> sp_sum(1024, 0.0);
    std::vector<int> sp_n(1024, 0);
    std::vector<float> w(size_t(G), 1.f);
    std::vector<int64_t> x;
    std::vector<int> smid_of(size_t(G), -1);
    double span = 0.0;
    for (int round = 0; round < 3; ++round) {
        for (int rep = 0; rep < 4; ++rep) {
            if (int rc = run(w, nullptr, 0, x, span)) return rc;
            if (rep == 0) continue;  // the first launch of a layout pays cold-start effects
            for (int c = 0; c < G; ++c) {
                const unsigned long long t0 = st[4096 + 2 * size_t(c)], t1 = st[4097 + 2 * size_t(c)];
                const unsigned long long sm = st[2048 + size_t(c)];
                const int64_t tiles = x[size_t(c) + 1] - x[size_t(c)];
                if (t1 > t0 && tiles > 0 && sm < 1024) {
                    sp_sum[size_t(sm)] += double(tiles) / double(t1 - t0);
                    ++sp_n[size_t(sm)];
                }
                smid_of[size_t(c)] = sm < 1024 ? static_cast<int>(sm) : -1;
            }
        }
        double mean = 0.0;
        int n = 0;
        for (int c = 0; c < G; ++c) {
            const int sm = smid_of[size_t(c)];
            if (sm >= 0 && sp_n[size_t(sm)] > 0) {
                mean += sp_sum[size_t(sm)] / sp_n[size_t(sm)];
                ++n;
            }
        }
        if (n == 0) return set_err(TD_ECUDA, "calibration: no stamps");
        mean /= n;
        for (int c = 0; c < G; ++c) {
            const int sm = smid_of[size_t(c)];
            if (sm >= 0 && sp_n[size_t(sm)] > 0)
                w[size_t(c)] = static_cast<float>(std::min(1.5, std::max(0.5, sp_sum[size_t(sm)] / sp_n[size_t(sm)] / mean)));
        }
    }
    // 2. SM affinity: index c belongs to the SM it ran on in the last launch
    std::vector<int> m(1024, -1);
    bool ok = true;
    for (int c = 0; c < G && ok; ++c) {
        const int sm = smid_of[size_t(c)];
        if (sm < 0 || m[size_t(sm)] != -1) ok = false;
        else m[size_t(sm)] = c;
    }
    ctx->sm_map_ok = false;
    if (!ok) return set_err(TD_ECUDA, "calibration: CTAs did not land one per SM");
    TD_CUDA(ctx->sm_map.ensure(m.size() * sizeof(int)));
    TD_CUDA(cudaMemcpy(ctx->sm_map.p, m.data(), m.size() * sizeof(int), cudaMemcpyHostToDevice));
    // 3. keep the weights only if they beat the equal split (median of 5 launches
    // each, with the SM affinity the real launches use): a noisy calibration must
    // never cost time
    const int* smap = static_cast<const int*>(ctx->sm_map.p);
    const std::vector<float> ones(size_t(G), 1.f);
    std::vector<double> t_eq, t_cal;
    unsigned epoch = 1;
    for (int rep = 0; rep < 6; ++rep) {
        if (int rc = run(ones, smap, epoch++, x, span)) return rc;
        if (rep) t_eq.push_back(span);
        if (int rc = run(w, smap, epoch++, x, span)) return rc;
        if (rep) t_cal.push_back(span);
    }
    std::sort(t_eq.begin(), t_eq.end());
    std::sort(t_cal.begin(), t_cal.end());
    TD_CUDA(cudaMemset(ctx->claims.p, 0, size_t(G) * sizeof(unsigned)));
    tab.release();
    ctx->cal_gain = t_eq.empty() ? 0.0 : (t_eq[t_eq.size() / 2] - t_cal[t_cal.size() / 2]) / t_eq[t_eq.size() / 2];
    ctx->cal_w = ctx->cal_gain > 0.005 ? w : ones;  // equal weights: the affinity alone stays harmless
    ctx->cal_bytes = 2 * ctx->b * ctx->n_kv * ctx->len * ctx->d * td::dtype_bytes(ctx->dtype);
    ctx->sm_map_ok = true;
    return TD_OK;
}

// stride: tokens per bh row in memory (the placed shard's capacity; 0 for a
// contiguous [bh][t][d] buffer such as a ring chunk)
int plan_for(td_context* ctx, int64_t n_q, int64_t t, SplitPlan& plan, int64_t stride,
             bool generic_only = false, bool take_append = false) {
    std::string msg;
    if (n_q < 1 || n_q > (1 << 20)) return set_err(TD_EINVAL, "decode: bad query head count");
    // deterministic calls: the static split plus, unless TD_DPOOL=0, the deterministic
    // chunk pool; TD_DYNAMIC calls: the run-time home pool
    static const bool dpool = [] { const char* e = std::getenv("TD_DPOOL"); return !e || std::atoi(e) != 0; }();
    const int mode = ctx->det ? (dpool ? 2 : 0) : 1;
    if (!td::plan_split(ctx->dtype, ctx->b, static_cast<int>(n_q), static_cast<int>(ctx->n_kv), t,
                        static_cast<int>(ctx->d), ctx->sm_count, plan, msg, mode, generic_only))
        return set_err(TD_EINVAL, msg);
    plan.row_stride = stride;
    plan.t_safe = stride > 0 ? std::min(ctx->kv_safe, t) : 0;  // the context's own cache only
    plan.dbg = ctx->cur_dbg;
    plan.tl = ctx->cur_tl;
    plan.tl_cta = ctx->cur_tl_cta;
    plan.pdl = !ctx->shared_device;
    if (plan.kernel == 1 && calibration_enabled() && plan.total_tiles >= 8 * int64_t(plan.ctas)) {
        // a shard more than 4x larger or smaller than the one the weights were measured
        // on streams differently (ramp, L2): measure again (results change with the
        // partition, which changed shape anyway)
        const int64_t bytes = 2 * ctx->b * ctx->n_kv * t * ctx->d * td::dtype_bytes(ctx->dtype);
        if (!ctx->cal_w.empty() && ctx->cal_bytes > 0 && (bytes > 4 * ctx->cal_bytes || 4 * bytes < ctx->cal_bytes)) {
            ctx->cal_w.clear();
            ctx->cal_failed = false;
            ctx->sm_map_ok = false;
            for (auto& tb : ctx->tabs) tb.total = -1;
        }
        if (ctx->cal_w.size() != size_t(plan.ctas) && !ctx->cal_failed && ctx->kv_ok && !ctx->shared_device) {
            if (calibrate(ctx, n_q) != TD_OK) {
                ctx->cal_failed = true;  // keep the equal split
            } else {
                // staging and device space for the partition tables now, not when a
                // growing sequence changes the shape mid-loop (pinned allocation stalls)
                const size_t need = std::max<size_t>(64 * 1024, (size_t(plan.ctas) + 1) * 8 + 12 * size_t(plan.bh_count));
                for (auto& tb : ctx->tabs) {
                    if (tb.host_cap < need) {
                        if (tb.host) cudaFreeHost(tb.host);
                        tb.host = nullptr;
                        tb.host_cap = 0;
                        TD_CUDA(cudaMallocHost(&tb.host, need));
                        tb.host_cap = need;
                    }
                    TD_CUDA(tb.buf.ensure(need));
                }
            }
        }
        if (ctx->cal_w.size() == size_t(plan.ctas)) {
            if (int rc = apply_partition(ctx, plan)) return rc;
            if (ctx->sm_map_ok && sm_affinity_enabled()) {
                plan.sm_to_cta = static_cast<const int*>(ctx->sm_map.p);
                plan.claims = static_cast<unsigned*>(ctx->claims.p);
                if (++ctx->claim_epoch == 0) ++ctx->claim_epoch;  // 0 marks "never claimed"
                plan.epoch = ctx->claim_epoch;
            }
        }
    }
    if (ctx->pend_k) {  // the fused append rides on a bf16 split kernel over the own cache
        if (take_append && plan.kernel == 1 && stride > 0 && ctx->tm_ok) {
            plan.app_k = ctx->pend_k;
            plan.app_v = ctx->pend_v;
            plan.app_pos = ctx->pend_pos;
        } else if (int rc = flush_append(ctx)) {
            return rc;
        }
    }
    TD_CUDA(ctx->ws.ensure(plan.workspace_bytes()));
    if (plan.pool_tiles > 0) {
        // pool counters: zero at rest except the last launch's parity; a new
        // layout (bh_count) starts from a zeroed buffer
        const size_t cap = ctx->ctr.cap;
        TD_CUDA(ctx->ctr.ensure(plan.counters_bytes()));
        if (ctx->ctr.cap != cap || ctx->ctr_bh != plan.bh_count) {
            TD_CUDA(cudaMemsetAsync(ctx->ctr.p, 0, ctx->ctr.cap, ctx->stream));
            ctx->ctr_bh = plan.bh_count;
            ctx->kpar = 0;
        }
        plan.counters = static_cast<unsigned*>(ctx->ctr.p);
        plan.parity = ctx->kpar;  // advanced by launched() once the launch is in
    }
    return TD_OK;
}

// After a K1 launch of `plan` on the context's own counters: the next launch uses
// the other parity (the one this launch's K2 zeroes). A call that fails before
// launching leaves the parity alone, so the counters at rest stay zero.
void launched(td_context* ctx, const SplitPlan& plan) {
    if (plan.pool_tiles > 0 && plan.counters == ctx->ctr.p) ctx->kpar = plan.parity ^ 1;
    if (plan.sflag && plan.sflag == ctx->sflags.p) ctx->s_epoch = plan.sepoch;
    if (plan.app_k && plan.app_k == ctx->pend_k) {
        // the token is in the cache once this split kernel has run; the next K1 must not
        // load its tile before its own wait (the write is not visible to it earlier)
        ctx->pend_k = ctx->pend_v = nullptr;
        ctx->pend_pos = -1;
    }
}

// Streamed combine for the context's own shard (TD_K2_STREAM, default on): the
// plan's K1 publishes its states with flags and the split K2 folds them as they
// arrive (td_kernels.cu stream_fold). Every launch gets a new epoch (committed by
// launched(); graph replays patch it). Not for worker groups sharing a GPU: their
// K2 warps would spin next to a peer's K1.
int stream_setup(td_context* ctx, SplitPlan& plan) {
    static const bool on = [] { const char* e = std::getenv("TD_K2_STREAM"); return !e || std::atoi(e) != 0; }();
    plan.sflag = nullptr;
    if (!on || ctx->shared_device) return TD_OK;
    SplitPlan probe = plan;
    probe.sflag = reinterpret_cast<unsigned*>(&probe);  // any non-null pointer: the shape test
    if (!td::stream_plan(probe)) return TD_OK;
    const size_t cap = ctx->sflags.cap;
    TD_CUDA(ctx->sflags.ensure(plan.sflag_words() * sizeof(unsigned)));
    unsigned ep = ctx->s_epoch + 1;
    if (ctx->sflags.cap != cap || ep == 0) {  // fresh words (or an epoch wrap): zero, epochs from 1
        TD_CUDA(cudaMemsetAsync(ctx->sflags.p, 0, ctx->sflags.cap, ctx->stream));
        ctx->s_epoch = 0;
        ep = 1;
    }
    if (!ctx->s_err) {
        TD_CUDA(cudaHostAlloc(&ctx->s_err, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
        *reinterpret_cast<volatile int*>(ctx->s_err) = 0;
    }
    plan.sflag = static_cast<unsigned*>(ctx->sflags.p);
    plan.sepoch = ep;
    plan.serr = ctx->s_err;
    return TD_OK;
}

// A streamed combine that waited ~1 s for a split-kernel state which never came
// (the split kernel failed): the step's output is invalid. Reported by the next
// call, or by this call when it synchronised (host buffers).
int stream_failed(td_context* ctx) {
    if (!ctx->s_err || !*reinterpret_cast<volatile int*>(ctx->s_err)) return TD_OK;
    *reinterpret_cast<volatile int*>(ctx->s_err) = 0;
    return set_err(TD_ECUDA, "tree_decode: the combine kernel timed out waiting for the split kernel's states");
}

void phase_begin(td_context* ctx, int flags) {
    ctx->cur_phase = nullptr;
    if (!(flags & TD_TIME_PHASES)) return;
    if (ctx->phase_used == ctx->phase_sets.size()) {
        std::vector<cudaEvent_t> evs(8);
        for (auto& e : evs) cudaEventCreate(&e);
        ctx->phase_sets.push_back(evs);
    }
    ctx->cur_phase = &ctx->phase_sets[ctx->phase_used++];
    ctx->cur_mark = 0;
}

void phase_mark(td_context* ctx) {
    if (!ctx->cur_phase || ctx->cur_mark >= ctx->cur_phase->size()) return;
    cudaEventRecord((*ctx->cur_phase)[ctx->cur_mark++], ctx->stream);
}

cudaEvent_t* next_timer(td_context* ctx) {
    if (ctx->timers_used == ctx->timers.size()) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        ctx->timers.emplace_back(a, b);
    }
    return &ctx->timers[ctx->timers_used++].first;
}

// K1 + K2 over a [b][n_kv][t][d] buffer.
int run_partial(td_context* ctx, const SplitPlan& plan, const void* q, const void* kb,
                const void* vb, int64_t t, double scale, bool own_maps, float* rmax, float* lse,
                float* out, bool timed, td_context* phases = nullptr) {
    CUtensorMap mk, mv;
    const CUtensorMap *pk = nullptr, *pv = nullptr;
    if (plan.kernel == 1) {
        if (own_maps) {
            pk = &ctx->tmk;
            pv = &ctx->tmv;
        } else {
            std::string msg;
            const int64_t rows = ctx->b * ctx->n_kv * t;
            if (!td::make_tensor_map(&mk, kb, rows, static_cast<int>(ctx->d), plan.tile, msg) ||
                !td::make_tensor_map(&mv, vb, rows, static_cast<int>(ctx->d), plan.tile, msg))
                return set_err(TD_ECUDA, msg);
            pk = &mk;
            pv = &mv;
        }
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (timed) {
        cudaEvent_t* pr = next_timer(ctx);
        e0 = pr[0];
        e1 = pr[1];
    } else if (phases && phases->cur_phase && phases->cur_mark < phases->cur_phase->size()) {
        e1 = (*phases->cur_phase)[phases->cur_mark++];  // mark between K1 and K2
    }
    TD_CUDA(td::launch_decode_partial(plan, q, kb, vb, static_cast<float>(scale), pk, pv,
                                      ctx->ws.p, rmax, lse, out, ctx->stream, e0, e1));
    launched(ctx, plan);
    if (kb == ctx->k.p && plan.row_stride > 0)  // later K1s run after this one's wait
        ctx->kv_safe = plan.app_k ? std::min(t, plan.app_pos) : t;  // (a fused token: not before their own)
    ctx->last_kernels += 2;  // K1 + K2
    ctx->last_kv_bytes += 2.0 * double(ctx->b) * double(ctx->n_kv) * double(t) * double(ctx->d) *
                          td::dtype_bytes(ctx->dtype);
    ctx->last_split_kernel = plan.kernel;
    return TD_OK;
}

const void* stage_q(td_context* ctx, const void* q, int64_t n_q, int flags, int* rc) {
    *rc = TD_OK;
    if (!(flags & TD_HOST_IO)) return q;
    const size_t bytes = size_t(ctx->b) * size_t(n_q) * size_t(ctx->d) * td::dtype_bytes(ctx->dtype);
    cudaError_t e = ctx->q_dev.ensure(bytes);
    if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->q_dev.p, q, bytes, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) {
        *rc = set_err(TD_ECUDA, std::string("q upload: ") + cudaGetErrorString(e));
        return nullptr;
    }
    return ctx->q_dev.p;
}

// The device alias of a pinned (cudaHostAlloc / registered) host buffer, or
// nullptr for pageable memory. With UVA pinned memory is mapped, so the final
// kernel can store the result straight into it (no D2H copy on the step).
float* mapped_host(td_context* ctx, float* host) {
    cudaPointerAttributes at{};  // queried on every call: the buffer may have been freed and reused
    float* dev = nullptr;
    if (cudaPointerGetAttributes(&at, host) == cudaSuccess && at.type == cudaMemoryTypeHost && at.devicePointer)
        dev = static_cast<float*>(at.devicePointer);
    cudaGetLastError();
    ctx->mapped_for = host;
    ctx->mapped_dev = dev;
    return dev;
}

// Whether the exchange kernel (K2x) should store a host-buffer call's output
// straight into pinned host memory. Small outputs gain ~2 us that way; large ones
// lose: K2x's warps stall on their PCIe stores between the exchange polls (cfg4 at
// N = 2, 1024 rows x 512 B: e2e 830 us in place vs 704 us with a device buffer and
// one copy). The single-GPU combine K2 has no polls and keeps writing in place.
bool xchg_in_place(int64_t rows, int64_t d) {
    static const int64_t cap = [] { const char* e = std::getenv("TD_XCHG_HOST_MAX"); return e ? std::atoll(e) : 65536; }();
    return rows * d * int64_t(sizeof(float)) <= cap;
}

// A K2x spin that timed out (a peer never delivered this step's words) stores
// 1 into the mapped flag; the step's output is then garbage. Reported as an
// error, after which the exchange must be re-opened on every rank
// (td_p2p_handle / td_p2p_open) so that the epochs agree again.
int exchange_failed(td_context* ctx) {
    if (!ctx->x_err) return TD_OK;
    const int v = *reinterpret_cast<volatile int*>(ctx->x_err);
    if (!v) return TD_OK;
    *reinterpret_cast<volatile int*>(ctx->x_err) = 0;
    ctx->x_ready = false;
    ctx->nx_ready = false;
    const int miss = (v >> 8) & 255;
    return set_err(TD_ECUDA, "tree_decode: NVLink exchange timed out on rank " + std::to_string(ctx->rank) +
                                 " (epoch " + std::to_string(ctx->x_epoch) + ", first missing source " +
                                 (miss == 255 ? std::string("beyond the batched peers") : std::to_string(miss)) +
                                 "); re-open the exchange with td_p2p_handle / td_p2p_open (TD_NCCL_DEVICE: "
                                 "the next call re-registers its window on every rank)");
}

void nccl_dev_close(td_context* ctx) {
    if (ctx->nx_win) nccl().WindowDeregister(ctx->comm, ctx->nx_win);
    if (ctx->nx_buf) nccl().MemFree(ctx->nx_buf);
    ctx->nx_win = nullptr;
    ctx->nx_buf = nullptr;
    ctx->nx_rows = ctx->nx_d = 0;
    ctx->nx_ready = false;
}

// TD_NCCL_DEVICE: K2n's window for rows x d, zeroed (epoch 0 matches no step)
// before the collective registration, so no rank can store into a copy that is
// still being cleared; then every rank's copy's address from the device API.
int nccl_dev_open(td_context* ctx, int64_t rows, int64_t d) {
    if (ctx->nx_ready && rows <= ctx->nx_rows && d == ctx->nx_d) return TD_OK;
    if (!ctx->comm) return set_err(TD_ESTATE, "tree_decode: TD_NCCL_DEVICE needs td_comm_init");
    if (!nccl().symmetric() || !nccl().TeamLsa)
        return set_err(TD_EINVAL, "tree_decode: TD_NCCL_DEVICE needs NCCL >= 2.28 (symmetric windows, device API)");
    const auto team = nccl().TeamLsa(ctx->comm);
    if (team.nRanks != ctx->nranks || team.rank != ctx->rank)
        return set_err(TD_EINVAL, "tree_decode: TD_NCCL_DEVICE needs every rank in one NVLink domain");
    nccl_dev_close(ctx);
    const size_t bytes = td::literal_window_bytes(ctx->nranks, rows, d);
    if (nccl().MemAlloc(&ctx->nx_buf, bytes) != ncclSuccess) {
        ctx->nx_buf = nullptr;
        return set_err(TD_ENCCL, "tree_decode: ncclMemAlloc of the combine window failed");
    }
    TD_CUDA(cudaMemsetAsync(ctx->nx_buf, 0, bytes, ctx->stream));
    TD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (nccl().WindowRegister(ctx->comm, ctx->nx_buf, bytes, &ctx->nx_win, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess) {
        ctx->nx_win = nullptr;
        nccl_dev_close(ctx);
        return set_err(TD_ENCCL, "tree_decode: ncclCommWindowRegister of the combine window failed");
    }
    TD_CUDA(ctx->nx_ptrs.ensure(size_t(ctx->nranks) * sizeof(void*) + 64));
    int* ok = reinterpret_cast<int*>(static_cast<char*>(ctx->nx_ptrs.p) + size_t(ctx->nranks) * sizeof(void*));
    const cudaError_t e = td::launch_lsa_peers(ctx->nx_win, ctx->nranks, static_cast<void**>(ctx->nx_ptrs.p), ok,
                                               ctx->stream);
    if (e == cudaErrorNotSupported) {
        nccl_dev_close(ctx);
        return set_err(TD_EINVAL, "tree_decode: TD_NCCL_DEVICE: library built without NCCL's device headers");
    }
    TD_CUDA(e);
    int ok_h = 0;
    TD_CUDA(cudaMemcpyAsync(&ok_h, ok, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    TD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (!ok_h) {
        nccl_dev_close(ctx);
        return set_err(TD_EINVAL, "tree_decode: TD_NCCL_DEVICE: NVLink-domain rank differs from the world rank");
    }
    if (!ctx->x_err) TD_CUDA(cudaHostAlloc(&ctx->x_err, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
    ctx->nx_rows = rows;
    ctx->nx_d = d;
    ctx->nx_epoch = 0;
    ctx->nx_ready = true;
    return TD_OK;
}

// The NCCL combine's buffers [lse rows | shift rows | n rows*d, d rows] inside a
// symmetric window (every rank reaches this with the same shape: the decode is
// collective). Returns null when symmetric memory is unavailable or switched off
// (TD_NCCL_SYMMETRIC=0): the plain per-row buffers are used then.
float* nccl_window(td_context* ctx, int64_t rows, int64_t d) {
    static const bool on = [] { const char* e = std::getenv("TD_NCCL_SYMMETRIC"); return !e || std::atoi(e) != 0; }();
    if (!on || !ctx->comm || !nccl().symmetric() || ctx->win_state < 0) return nullptr;
    auto pad = [](size_t n) { return (n + 63) / 64 * 64; };
    const size_t need = (2 * pad(size_t(rows)) + pad(size_t(rows) * size_t(d + 1))) * sizeof(float);
    if (ctx->win_state == 1 && need <= ctx->win_bytes) return static_cast<float*>(ctx->win_buf);
    if (ctx->win) nccl().WindowDeregister(ctx->comm, ctx->win);
    if (ctx->win_buf) nccl().MemFree(ctx->win_buf);
    ctx->win = nullptr;
    ctx->win_buf = nullptr;
    ctx->win_bytes = 0;
    const size_t bytes = (need + 4095) / 4096 * 4096;
    if (nccl().MemAlloc(&ctx->win_buf, bytes) != ncclSuccess ||
        nccl().WindowRegister(ctx->comm, ctx->win_buf, bytes, &ctx->win, NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess) {
        if (ctx->win_buf) nccl().MemFree(ctx->win_buf);
        ctx->win_buf = nullptr;
        ctx->win = nullptr;
        ctx->win_state = -1;
        cudaGetLastError();
        return nullptr;
    }
    ctx->win_bytes = bytes;
    ctx->win_state = 1;
    return static_cast<float*>(ctx->win_buf);
}

int deliver_out(td_context* ctx, const float* src, int64_t rows, float* out, int flags) {
    if (int rc = note_table_use(ctx)) return rc;
    const size_t bytes = size_t(rows) * size_t(ctx->d) * sizeof(float);
    if (flags & TD_BF16_OUT) {
        TD_CUDA(ctx->out_bf16.ensure(size_t(rows) * size_t(ctx->d) * 2));
        TD_CUDA(td::launch_to_bf16(src, rows * ctx->d, ctx->out_bf16.p, ctx->stream));
        ctx->last_kernels += 1;
    }
    if (flags & TD_HOST_IO) {
        if (src != ctx->mapped_dev || ctx->mapped_for != out)  // else the kernel stored into `out` already
            TD_CUDA(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
        TD_CUDA(cudaStreamSynchronize(ctx->stream));
    } else if (out != src) {
        TD_CUDA(cudaMemcpyAsync(out, src, bytes, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    return TD_OK;
}

}  // namespace

extern "C" {

int td_version(void) { return 1; }
const char* td_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------- stateless
int td_seeded_fill(int dtype, void* dst, uint64_t seed, double scale, int64_t bh_count,
                   int64_t seq, int64_t start, int64_t len, int64_t d, void* stream) {
    if (!(scale > 0.0)) return set_err(TD_EINVAL, "seeded_random_tensor: scale must be positive");
    if (dtype < 0 || dtype > 2 || bh_count < 0 || d < 0 || len < 0 || start < 0 ||
        start + len > seq)
        return set_err(TD_EINVAL, "td_seeded_fill: bad arguments");
    TD_CUDA(td::launch_seeded_fill(dtype, dst, seed, scale, bh_count, seq, start, len, d,
                                   static_cast<cudaStream_t>(stream)));
    return TD_OK;
}

int td_decode_workspace_bytes(int dtype, int64_t b, int64_t n_q, int64_t n_kv, int64_t t,
                              int64_t d, size_t* bytes) {
    SplitPlan plan;
    std::string msg;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!td::plan_split(dtype, b, static_cast<int>(n_q), static_cast<int>(n_kv), t,
                        static_cast<int>(d), sm_count_of(dev), plan, msg, g_deterministic == 0 ? 1 : 0))
        return set_err(TD_EINVAL, msg);
    // + the pool counters, carved from the end of the caller's workspace
    *bytes = (plan.workspace_bytes() + 255) / 256 * 256 + plan.counters_bytes();
    return TD_OK;
}

int td_set_deterministic(int on) {
    g_deterministic = on != 0;
    return TD_OK;
}

int td_decode_partial(int dtype, const void* q, const void* k, const void* v, int64_t b,
                      int64_t n_q, int64_t n_kv, int64_t t, int64_t d, double scale,
                      float* row_max, float* lse, float* out, void* workspace,
                      size_t workspace_bytes, void* stream) {
    SplitPlan plan;
    std::string msg;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!td::plan_split(dtype, b, static_cast<int>(n_q), static_cast<int>(n_kv), t,
                        static_cast<int>(d), sm_count_of(dev), plan, msg, g_deterministic == 0 ? 1 : 0))
        return set_err(TD_EINVAL, msg);
    const size_t ctr_off = (plan.workspace_bytes() + 255) / 256 * 256;
    if (workspace_bytes < ctr_off + plan.counters_bytes())
        return set_err(TD_EINVAL, "td_decode_partial: workspace too small");
    CUtensorMap mk, mv;
    if (plan.kernel == 1) {
        const int64_t rows = b * n_kv * t;
        if (!td::make_tensor_map(&mk, k, rows, static_cast<int>(d), plan.tile, msg) ||
            !td::make_tensor_map(&mv, v, rows, static_cast<int>(d), plan.tile, msg))
            return set_err(TD_ECUDA, msg);
    }
    if (plan.pool_tiles > 0) {  // stateless: counters zeroed on every call
        plan.counters = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + ctr_off);
        plan.parity = 0;
        TD_CUDA(cudaMemsetAsync(plan.counters, 0, plan.counters_bytes(), static_cast<cudaStream_t>(stream)));
    }
    TD_CUDA(td::launch_decode_partial(plan, q, k, v, static_cast<float>(scale), &mk, &mv, workspace,
                                      row_max, lse, out, static_cast<cudaStream_t>(stream)));
    return TD_OK;
}

// ---- energy formulation ----------------------------------
int td_energy_workspace_bytes(int dtype, int64_t b, int64_t h, int64_t nq, int64_t t, int64_t d,
                              size_t* bytes) {
    SplitPlan plan;
    std::string msg;
    int dev = 0;
    cudaGetDevice(&dev);
    if (nq < 1 || h < 1) return set_err(TD_EINVAL, "energy: need h >= 1 and nq >= 1");
    if (!td::plan_split(dtype, b, static_cast<int>(h * nq), static_cast<int>(h), t, static_cast<int>(d),
                        sm_count_of(dev), plan, msg, false, true))
        return set_err(TD_EINVAL, msg);
    *bytes = plan.workspace_bytes();
    return TD_OK;
}

int td_energy_partial(int dtype, const void* q, const void* src, const void* k, const void* v, int64_t b,
                      int64_t h, int64_t nq, int64_t t, int64_t d, float* row_max, float* lse, float* out,
                      void* workspace, size_t workspace_bytes, void* stream) {
    SplitPlan plan;
    std::string msg;
    int dev = 0;
    cudaGetDevice(&dev);
    if (nq < 1 || h < 1) return set_err(TD_EINVAL, "energy: need h >= 1 and nq >= 1");
    // the nq query rows of head h are a GQA group of size nq over kv head h
    if (!td::plan_split(dtype, b, static_cast<int>(h * nq), static_cast<int>(h), t, static_cast<int>(d),
                        sm_count_of(dev), plan, msg, false, true))
        return set_err(TD_EINVAL, msg);
    if (workspace_bytes < plan.workspace_bytes()) return set_err(TD_EINVAL, "td_energy_partial: workspace too small");
    TD_CUDA(td::launch_decode_partial(plan, q, k, v, 1.0f, nullptr, nullptr, workspace, row_max, lse, out,
                                      static_cast<cudaStream_t>(stream), nullptr, nullptr, src));
    return TD_OK;
}

int td_energy_combine(int P, const float* row_max, const float* lse, int64_t rows, float* value,
                      float* row_max_out, float* shifted, void* stream) {
    if (P < 1 || rows < 0) return set_err(TD_EINVAL, "energy_combine: no parts");
    TD_CUDA(td::launch_energy_combine(P, row_max, lse, rows, value, row_max_out, shifted,
                                      static_cast<cudaStream_t>(stream)));
    return TD_OK;
}

int td_energy_grad_combine(int P, const float* lse, const float* out, const float* row_max,
                           const float* shifted, int64_t rows, int64_t d, float* grad, void* stream) {
    if (P < 1 || rows < 0 || d < 1) return set_err(TD_EINVAL, "energy_grad_combine: bad arguments");
    TD_CUDA(td::launch_energy_grad_combine(P, lse, out, row_max, shifted, rows, static_cast<int>(d), grad,
                                           static_cast<cudaStream_t>(stream)));
    return TD_OK;
}

int td_combine_partials(int P, const float* lse, const float* out, int64_t rows, int64_t d,
                        float* result, void* stream) {
    if (P < 1) return set_err(TD_EINVAL, "combine_partials: no parts");
    // the empty-row verdict: one mapped pinned flag per host thread (portable across
    // devices), allocated once; the call synchronises to raise like the reference
    thread_local int* bad = nullptr;
    if (!bad) TD_CUDA(cudaHostAlloc(&bad, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
    volatile int* flag = bad;
    *flag = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TD_CUDA(td::launch_combine_partials(P, lse, out, rows, static_cast<int>(d), result, bad, st));
    TD_CUDA(cudaStreamSynchronize(st));
    if (*flag) return set_err(TD_EINVAL, "combine_partials: no keys attended");
    return TD_OK;
}

int td_partial_to_numerator(const float* lse, const float* out, const float* shift,
                            int64_t rows, int64_t d, float* nd, void* stream) {
    TD_CUDA(td::launch_to_numerator(lse, out, shift, rows, static_cast<int>(d), nd,
                                    static_cast<cudaStream_t>(stream)));
    return TD_OK;
}

int td_combine_pair(float* l_max, float* l_lse, float* l_out, const float* r_max,
                    const float* r_lse, const float* r_out, int64_t rows, int64_t d,
                    void* stream) {
    TD_CUDA(td::launch_combine_pair(l_max, l_lse, l_out, r_max, r_lse, r_out, rows,
                                    static_cast<int>(d), static_cast<cudaStream_t>(stream)));
    return TD_OK;
}

int td_finalize(const float* nd, int64_t rows, int64_t d, float* out, void* out_bf16,
                void* stream) {
    TD_CUDA(td::launch_finalize(nd, rows, static_cast<int>(d), out, out_bf16,
                                static_cast<cudaStream_t>(stream)));
    return TD_OK;
}

// ---------------------------------------------------------------- context
int td_create(int device, td_context** out) {
    if (!out) return set_err(TD_EINVAL, "td_create: null output");
    int n = 0;
    TD_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) return set_err(TD_EINVAL, "td_create: no such device");
    TD_CUDA(cudaSetDevice(device));
    auto* ctx = new td_context;
    ctx->device = device;
    ctx->sm_count = sm_count_of(device);
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->xfer, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete ctx;
        return set_err(TD_ECUDA, std::string("td_create: ") + cudaGetErrorString(e));
    }
    *out = ctx;
    return TD_OK;
}

int td_destroy(td_context* ctx) {
    if (!ctx) return TD_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->xfer);
    for (auto& g : ctx->graph) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
    }
    if (ctx->win) nccl().WindowDeregister(ctx->comm, ctx->win);
    if (ctx->win_buf) nccl().MemFree(ctx->win_buf);
    nccl_dev_close(ctx);
    ctx->nx_ptrs.release();
    if (ctx->comm) nccl().CommDestroy(ctx->comm);
    ctx->k.release();
    ctx->v.release();
    ctx->ws.release();
    ctx->rows.release();
    ctx->q_dev.release();
    ctx->out_bf16.release();
    for (auto& rb : ctx->ring)
        for (auto& x : rb) x.release();
    for (auto& x : ctx->ring_own) x.release();
    for (auto& ev : ctx->ring_ev) cudaEventDestroy(ev);
    for (auto& pr : ctx->timers) {
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
    }
    for (void* ptr : ctx->x_opened) cudaIpcCloseMemHandle(ptr);
    ctx->xbuf.release();
    ctx->x_ptrs.release();
    if (ctx->x_err) cudaFreeHost(ctx->x_err);
    if (ctx->s_err) cudaFreeHost(ctx->s_err);
    if (ctx->done_host) cudaFreeHost(ctx->done_host);
    ctx->sig.release();
    ctx->sflags.release();
    ctx->ctr.release();
    ctx->dbg.release();
    ctx->tlbuf.release();
    ctx->sm_map.release();
    ctx->claims.release();
    ctx->cal_q.release();
    for (auto& tb : ctx->tabs) {
        tb.buf.release();
        if (tb.host) cudaFreeHost(tb.host);
        if (tb.used) cudaEventDestroy(tb.used);
    }
    cudaStreamDestroy(ctx->stream);
    cudaStreamDestroy(ctx->xfer);
    delete ctx;
    return TD_OK;
}

int td_stream(td_context* ctx, void** stream) {
    if (int rc = require_ctx(ctx)) return rc;
    *stream = ctx->stream;
    return TD_OK;
}

int td_comm_unique_id(unsigned char id[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId uid;
    TD_NCCL(nccl().GetUniqueId(&uid));
    std::memcpy(id, &uid, 128);
    return TD_OK;
}

int td_comm_init(td_context* ctx, int nranks, int rank, const unsigned char id[128]) {
    if (int rc = require_ctx(ctx)) return rc;
    if (nranks < 1 || rank < 0 || rank >= nranks) return set_err(TD_EINVAL, "td_comm_init: bad rank");
    if (ctx->comm) {
        if (ctx->win) nccl().WindowDeregister(ctx->comm, ctx->win);
        if (ctx->win_buf) nccl().MemFree(ctx->win_buf);
        ctx->win = nullptr;
        ctx->win_buf = nullptr;
        ctx->win_bytes = 0;
        ctx->win_state = 0;
        nccl_dev_close(ctx);
        nccl().CommDestroy(ctx->comm);
        ctx->comm = nullptr;
    }
    if (nranks > 1) {
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        TD_NCCL(nccl().CommInitRank(&ctx->comm, nranks, uid, rank));
    }
    ctx->nranks = nranks;
    ctx->rank = rank;
    if (ctx->kv_ok) ctx->lens = chunk_extents(ctx->seq_len, nranks);
    return TD_OK;
}

int td_comm_info(td_context* ctx, int* nranks, int* rank) {
    if (int rc = require_ctx(ctx)) return rc;
    *nranks = ctx->nranks;
    *rank = ctx->rank;
    return TD_OK;
}

}  // extern "C"

// The exchange buffer of one rank, zeroed (epoch 0 matches no step), and its
// timeout flag; the peers' pointers are set by td_p2p_open / td_group_p2p_open.
static int xbuf_alloc(td_context* ctx, int64_t max_rows, int64_t d) {
    if (max_rows < 1 || d < 1 || d > 256) return set_err(TD_EINVAL, "p2p: bad max_rows / head_dim");
    for (void* ptr : ctx->x_opened) cudaIpcCloseMemHandle(ptr);
    ctx->x_opened.clear();
    ctx->x_ready = false;
    // LL words (value, epoch): [2 parities][p sources][max_rows][d + 1] x 8 bytes
    const size_t data = 2 * size_t(ctx->nranks) * size_t(max_rows) * size_t(d + 1) * 2 * sizeof(float);
    ctx->xbuf.release();
    TD_CUDA(ctx->xbuf.ensure(data));
    TD_CUDA(cudaMemset(ctx->xbuf.p, 0, data));
    if (!ctx->x_err) TD_CUDA(cudaHostAlloc(&ctx->x_err, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable));
    *reinterpret_cast<volatile int*>(ctx->x_err) = 0;
    ctx->x_max_rows = max_rows;
    ctx->x_d = d;
    ctx->x_epoch = 0;
    return TD_OK;
}

extern "C" {

int td_p2p_handle(td_context* ctx, int64_t max_rows, int64_t d, unsigned char handle[64]) {
    if (int rc = require_ctx(ctx)) return rc;
    if (int rc = xbuf_alloc(ctx, max_rows, d)) return rc;
    cudaIpcMemHandle_t h;
    TD_CUDA(cudaIpcGetMemHandle(&h, ctx->xbuf.p));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
    std::memcpy(handle, &h, 64);
    return TD_OK;
}

int td_p2p_open(td_context* ctx, const unsigned char* handles) {
    if (int rc = require_ctx(ctx)) return rc;
    if (!ctx->xbuf.p) return set_err(TD_ESTATE, "p2p: call td_p2p_handle first");
    const int p = ctx->nranks;
    std::vector<void*> base(size_t(p), nullptr);
    for (int q = 0; q < p; ++q) {
        if (q == ctx->rank) {
            base[size_t(q)] = ctx->xbuf.p;
            continue;
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handles + 64 * q, 64);
        void* ptr = nullptr;
        TD_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        ctx->x_opened.push_back(ptr);
        base[size_t(q)] = ptr;
    }
    const std::vector<void*>& arr = base;
    TD_CUDA(ctx->x_ptrs.ensure(arr.size() * sizeof(void*)));
    TD_CUDA(cudaMemcpy(ctx->x_ptrs.p, arr.data(), arr.size() * sizeof(void*), cudaMemcpyHostToDevice));
    ctx->x_ready = true;
    return TD_OK;
}

int td_p2p_status(td_context* ctx, int* error) {
    if (int rc = require_ctx(ctx)) return rc;
    *error = 0;
    if (!ctx->x_err) return TD_OK;
    TD_CUDA(cudaStreamSynchronize(ctx->stream));
    volatile int* f = ctx->x_err;
    *error = *f;
    if (*error) {  // the ranks' epochs can no longer be trusted to agree: re-open to resume
        *f = 0;
        ctx->x_ready = false;
    }
    return TD_OK;
}

static int kv_alloc(td_context* ctx, int dtype, int64_t b, int64_t n_kv, int64_t seq_len,
                    int64_t d, int64_t start, int64_t len) {
    if (dtype != TD_F32 && dtype != TD_BF16)
        return set_err(TD_EINVAL, "kv: the GPU path stores f32 or bf16 caches");
    if (b < 1 || n_kv < 1 || d < 1 || d > 256 || seq_len < 1)
        return set_err(TD_EINVAL, "kv: dimensions must be positive (head_dim <= 256)");
    if (start < 0 || len < 0 || start + len > seq_len)
        return set_err(TD_EINVAL, "kv: shard range out of bounds");
    const size_t bytes = size_t(b) * size_t(n_kv) * size_t(len) * size_t(d) * td::dtype_bytes(dtype);
    TD_CUDA(ctx->k.ensure(bytes > 0 ? bytes : 16));
    TD_CUDA(ctx->v.ensure(bytes > 0 ? bytes : 16));
    ctx->dtype = dtype;
    ctx->b = b;
    ctx->n_kv = n_kv;
    ctx->seq_len = seq_len;
    ctx->d = d;
    ctx->start = start;
    ctx->len = len;
    ctx->cap = len;
    ctx->lens = chunk_extents(seq_len, ctx->nranks);
    ctx->kv_ok = false;
    ctx->tm_ok = false;
    ctx->kv_safe = 0;
    ctx->pend_k = ctx->pend_v = nullptr;  // a new cache: a token appended to the old one is gone
    ctx->pend_pos = -1;
    return TD_OK;
}

static int kv_finish(td_context* ctx) {
    ctx->tm_ok = false;
    if (ctx->dtype == TD_BF16 && (ctx->d == 64 || ctx->d == 128 || ctx->d == 256) && ctx->len > 0) {
        std::string msg;
        const int64_t rows = ctx->b * ctx->n_kv * ctx->cap;  // rows of the allocation (stride cap)
        if (rows >= (int64_t(1) << 31)) return set_err(TD_EINVAL, "kv: shard too large for 32-bit TMA rows");
        SplitPlan plan;
        if (!td::plan_split(ctx->dtype, ctx->b, static_cast<int>(ctx->n_kv), static_cast<int>(ctx->n_kv),
                            ctx->len, static_cast<int>(ctx->d), ctx->sm_count, plan, msg))
            return set_err(TD_EINVAL, msg);
        if (!td::make_tensor_map(&ctx->tmk, ctx->k.p, rows, static_cast<int>(ctx->d), plan.tile, msg) ||
            !td::make_tensor_map(&ctx->tmv, ctx->v.p, rows, static_cast<int>(ctx->d), plan.tile, msg))
            return set_err(TD_ECUDA, msg);
        ctx->tm_ok = true;
    }
    TD_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->kv_ok = true;
    ctx->kv_safe = ctx->len;
    return TD_OK;
}

int td_kv_place(td_context* ctx, int dtype, int64_t b, int64_t n_kv, int64_t seq_len, int64_t d,
                int64_t start, int64_t len, const void* k, const void* v, int from_host) {
    if (int rc = require_ctx(ctx)) return rc;
    if (int rc = kv_alloc(ctx, dtype, b, n_kv, seq_len, d, start, len)) return rc;
    const size_t bytes = size_t(b) * size_t(n_kv) * size_t(len) * size_t(d) * td::dtype_bytes(dtype);
    const cudaMemcpyKind kind = from_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    if (bytes) {
        TD_CUDA(cudaMemcpyAsync(ctx->k.p, k, bytes, kind, ctx->stream));
        TD_CUDA(cudaMemcpyAsync(ctx->v.p, v, bytes, kind, ctx->stream));
    }
    return kv_finish(ctx);
}

int td_kv_generate(td_context* ctx, int dtype, int64_t b, int64_t n_kv, int64_t seq_len,
                   int64_t d, uint64_t seed_k, uint64_t seed_v, double scale) {
    if (int rc = require_ctx(ctx)) return rc;
    if (ctx->nranks > seq_len) return set_err(TD_EINVAL, "shard_kv: more workers than keys");
    const std::vector<int64_t> ext = chunk_extents(seq_len, ctx->nranks);
    int64_t start = 0;
    for (int w = 0; w < ctx->rank; ++w) start += ext[static_cast<size_t>(w)];
    const int64_t len = ext[static_cast<size_t>(ctx->rank)];
    if (int rc = kv_alloc(ctx, dtype, b, n_kv, seq_len, d, start, len)) return rc;
    if (int rc = td_seeded_fill(dtype, ctx->k.p, seed_k, scale, b * n_kv, seq_len, start, len, d,
                                ctx->stream))
        return rc;
    if (int rc = td_seeded_fill(dtype, ctx->v.p, seed_v, scale, b * n_kv, seq_len, start, len, d,
                                ctx->stream))
        return rc;
    return kv_finish(ctx);
}

// Grows the placed shard's per-row capacity to `cap` tokens (rows are
// re-strided, the data kept).
static int kv_grow(td_context* ctx, int64_t cap) {
    const size_t esz = td::dtype_bytes(ctx->dtype);
    const size_t row_old = size_t(ctx->cap) * size_t(ctx->d) * esz, row_new = size_t(cap) * size_t(ctx->d) * esz;
    const size_t rows = size_t(ctx->b) * size_t(ctx->n_kv);
    if (int64_t(rows) * cap >= (int64_t(1) << 31)) return set_err(TD_EINVAL, "kv_append: shard too large for 32-bit TMA rows");
    if (int rc = flush_append(ctx)) return rc;
    TD_CUDA(cudaStreamSynchronize(ctx->stream));
    // both new buffers first, so a failed allocation leaves the shard untouched
    void* fresh[2] = {nullptr, nullptr};
    cudaError_t e = cudaMalloc(&fresh[0], rows * row_new);
    if (e == cudaSuccess) e = cudaMalloc(&fresh[1], rows * row_new);
    DevBuf* bufs[2] = {&ctx->k, &ctx->v};
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        // the unused tail of every row is read by partial tiles (masked out of the
        // softmax, but 0 * NaN would poison P.V): keep it zero
        e = cudaMemsetAsync(fresh[i], 0, rows * row_new, ctx->stream);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(fresh[i], row_new, bufs[i]->p, row_old, size_t(ctx->len) * size_t(ctx->d) * esz,
                                  rows, cudaMemcpyDeviceToDevice, ctx->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
        cudaFree(fresh[0]);
        cudaFree(fresh[1]);
        TD_CUDA(e);
    }
    for (int i = 0; i < 2; ++i) {
        bufs[i]->release();
        bufs[i]->p = fresh[i];
        bufs[i]->cap = rows * row_new;
    }
    ctx->cap = cap;
    for (auto& tb : ctx->tabs) tb.total = -1;  // partition tables follow the new shape
    return kv_finish(ctx);
}

int td_kv_append(td_context* ctx, const void* k, const void* v, int from_host) {
    if (int rc = require_ctx(ctx)) return rc;
    if (!ctx->kv_ok) return set_err(TD_ESTATE, "kv_append: no KV shard placed");
    if (ctx->rank != ctx->nranks - 1) {  // every rank: the cache is one token longer, on rank p-1
        ctx->seq_len += 1;
        ctx->lens.back() += 1;
        return TD_OK;
    }
    if (!k || !v) return set_err(TD_EINVAL, "kv_append: the last rank needs the token's k and v");
    if (ctx->len == ctx->cap)  // grows before any state changes: a failure leaves the cache as it was
        if (int rc = kv_grow(ctx, ctx->cap + std::max<int64_t>(1024, ctx->cap / 8))) return rc;
    if (int rc = flush_append(ctx)) return rc;  // one pending token at a time
    static const bool fuse = [] { const char* e = std::getenv("TD_FUSED_APPEND"); return !e || std::atoi(e) != 0; }();
    if (!from_host && fuse && ctx->tm_ok) {
        // device source, bf16 TMA cache: the next decode's split kernel writes it
        ctx->pend_k = k;
        ctx->pend_v = v;
        ctx->pend_pos = ctx->len;
        ctx->len += 1;
        ctx->seq_len += 1;
        ctx->lens.back() += 1;
        return TD_OK;
    }
    const size_t esz = td::dtype_bytes(ctx->dtype);
    const size_t tok = size_t(ctx->d) * esz, pitch = size_t(ctx->cap) * tok;
    const size_t rows = size_t(ctx->b) * size_t(ctx->n_kv);
    if (from_host) {
        TD_CUDA(cudaMemcpy2DAsync(static_cast<char*>(ctx->k.p) + size_t(ctx->len) * tok, pitch, k, tok, tok, rows,
                                  cudaMemcpyHostToDevice, ctx->stream));
        TD_CUDA(cudaMemcpy2DAsync(static_cast<char*>(ctx->v.p) + size_t(ctx->len) * tok, pitch, v, tok, tok, rows,
                                  cudaMemcpyHostToDevice, ctx->stream));
    } else {  // a kernel: keeps the programmatic-launch chain of a decode loop
        TD_CUDA(td::launch_kv_append(ctx->dtype, ctx->k.p, ctx->v.p, k, v, int64_t(rows), ctx->cap, ctx->len,
                                     static_cast<int>(ctx->d), ctx->stream));
    }
    ctx->len += 1;
    ctx->seq_len += 1;
    ctx->lens.back() += 1;
    if (from_host) TD_CUDA(cudaStreamSynchronize(ctx->stream));  // the caller may reuse its buffer
    return TD_OK;
}

int td_kv_reserve(td_context* ctx, int64_t tokens) {
    if (int rc = require_ctx(ctx)) return rc;
    if (!ctx->kv_ok) return set_err(TD_ESTATE, "kv_reserve: no KV shard placed");
    if (tokens < 0) return set_err(TD_EINVAL, "kv_reserve: negative count");
    if (ctx->rank != ctx->nranks - 1 || ctx->len + tokens <= ctx->cap) return TD_OK;
    return kv_grow(ctx, ctx->len + tokens);
}

int td_kv_info(td_context* ctx, int64_t* start, int64_t* len, size_t* bytes) {
    if (int rc = require_ctx(ctx)) return rc;
    if (!ctx->kv_ok) return set_err(TD_ESTATE, "no KV shard placed");
    *start = ctx->start;
    *len = ctx->len;
    *bytes = 2 * size_t(ctx->b) * size_t(ctx->n_kv) * size_t(ctx->len) * size_t(ctx->d) *
             td::dtype_bytes(ctx->dtype);
    return TD_OK;
}

int td_kv_pointers(td_context* ctx, void** k, void** v) {
    if (int rc = require_ctx(ctx)) return rc;
    if (!ctx->kv_ok) return set_err(TD_ESTATE, "no KV shard placed");
    if (int rc = flush_append(ctx)) return rc;  // the caller reads the cache
    *k = ctx->k.p;
    *v = ctx->v.p;
    return TD_OK;
}

// TD_DEBUG_TIMELINE=1: every decode call stamps [K1 first start, first CTA past
// the PDL wait, K1 last end, K2 last done] into dbg[5000 + 4 * (call % 286)],
// without any extra operation on the stream (see scripts/timeline_probe.py).
static int timeline_step(td_context* ctx) {
    static const bool on = [] { const char* e = std::getenv("TD_DEBUG_TIMELINE"); return e && std::atoi(e) != 0; }();
    ctx->cur_tl = ctx->cur_tl_cta = nullptr;
    if (!on) return TD_OK;
    if (ctx->tl_count < 0) {
        std::vector<unsigned long long> init(6144 - 5000);
        for (size_t i = 0; i < init.size(); ++i) init[i] = (i % 4) < 2 ? ~0ull : 0ull;
        TD_CUDA(ctx->tlbuf.ensure(init.size() * sizeof(unsigned long long)));
        TD_CUDA(cudaMemcpy(ctx->tlbuf.p, init.data(), init.size() * sizeof(unsigned long long),
                           cudaMemcpyHostToDevice));
        ctx->tl_count = 0;
    }
    TD_CUDA(ctx->dbg.ensure(6144 * sizeof(unsigned long long)));
    ctx->cur_tl = static_cast<unsigned long long*>(ctx->tlbuf.p) + 4 * (ctx->tl_count % 286);
    ctx->cur_tl_cta = static_cast<unsigned long long*>(ctx->dbg.p);
    ++ctx->tl_count;
    return TD_OK;
}

static int debug_begin(td_context* ctx, int flags) {
    ctx->cur_dbg = nullptr;
    if (int rc = timeline_step(ctx)) return rc;
    if (!(flags & TD_DEBUG_TS)) return TD_OK;
    TD_CUDA(ctx->dbg.ensure(6144 * sizeof(unsigned long long)));
    TD_CUDA(cudaMemsetAsync(ctx->dbg.p, 0, 6144 * sizeof(unsigned long long), ctx->stream));
    TD_CUDA(cudaMemsetAsync(ctx->dbg.p, 0xff, sizeof(unsigned long long), ctx->stream));
    ctx->cur_dbg = static_cast<unsigned long long*>(ctx->dbg.p);
    return TD_OK;
}

int td_debug_stamps(td_context* ctx, unsigned long long* out, int n) {
    if (int rc = require_ctx(ctx)) return rc;
    if (!ctx->dbg.p && !ctx->tlbuf.p) return set_err(TD_ESTATE, "no TD_DEBUG_TS call made");
    TD_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->dbg.p)
        TD_CUDA(cudaMemcpy(out, ctx->dbg.p, sizeof(unsigned long long) * size_t(std::min(n, 6144)),
                           cudaMemcpyDeviceToHost));
    if (ctx->tlbuf.p && n > 5000)
        TD_CUDA(cudaMemcpy(out + 5000, ctx->tlbuf.p, sizeof(unsigned long long) * size_t(std::min(n, 6144) - 5000),
                           cudaMemcpyDeviceToHost));
    return TD_OK;
}

}  // extern "C"

namespace {

// The part of tree_decode before any launch: validation, per-row buffers, the
// split plan (calibrating the partition on a context's first long decode) and
// the query on the device. `q_on_device` overrides the staging of q (td_group
// stages it itself).
struct TreeCall {
    SplitPlan plan;
    const void* qd = nullptr;
    int64_t rows = 0;
    bool fast = false;  // TD_PINNED_IO fast path taken (tree_begin)
};

// TD_PINNED_IO with TD_HOST_IO: out is a pinned host buffer the combine kernel
// writes in place (with UVA a pinned buffer's device address is its host
// address) and then signals through pinned host memory. Taken when the last
// kernel of the step is a signalling K2 / K2x (not the NCCL path's K4) and the
// output needs no bf16 copy.
bool pinned_fast_path(td_context* ctx, int flags, const SplitPlan& plan) {
    static const bool on = [] { const char* e = std::getenv("TD_PINNED_FAST"); return !e || std::atoi(e) != 0; }();
    if (!on || (flags & (TD_HOST_IO | TD_PINNED_IO)) != (TD_HOST_IO | TD_PINNED_IO) ||
        (flags & (TD_BF16_OUT | TD_DEBUG_TS)))
        return false;
    if (flags & TD_TIME_PHASES) return false;
    if (ctx->nranks > 1 && !(flags & TD_P2P)) return false;  // the NCCL path ends in K4, not in a signalling K2
    if (ctx->nranks > 1 && !xchg_in_place(plan.bh_count * plan.group, ctx->d)) return false;
    if (ctx->host_ptr_ok < 0) {
        int uva = 0, reg = 0;
        cudaDeviceGetAttribute(&uva, cudaDevAttrUnifiedAddressing, ctx->device);
        cudaDeviceGetAttribute(&reg, cudaDevAttrCanUseHostPointerForRegisteredMem, ctx->device);
        ctx->host_ptr_ok = uva && reg;
    }
    return ctx->host_ptr_ok == 1;
}

int ensure_signals(td_context* ctx) {
    if (!ctx->sig.p) {
        TD_CUDA(ctx->sig.ensure(sizeof(unsigned)));
        TD_CUDA(cudaMemset(ctx->sig.p, 0, sizeof(unsigned)));
    }
    if (!ctx->done_host) {
        void* h = nullptr;
        TD_CUDA(cudaHostAlloc(&h, 64, cudaHostAllocMapped | cudaHostAllocPortable));
        std::memset(h, 0, 64);
        ctx->done_host = static_cast<unsigned*>(h);
    }
    return TD_OK;
}

// Waits for the combine kernel's completion word (a spin on pinned host memory
// the GPU writes over PCIe: no stream synchronisation on the step). The stream
// is queried now and then so a failed launch surfaces as an error.
int wait_done(td_context* ctx, unsigned epoch) {
    static const bool spin = [] { const char* e = std::getenv("TD_PINNED_SPIN"); return !e || std::atoi(e) != 0; }();
    if (!spin) TD_CUDA(cudaStreamSynchronize(ctx->stream));  // A/B switch: the runtime's wait instead
    volatile unsigned* f = ctx->done_host;
    for (unsigned spins = 1; *f != epoch; ++spins) {
        if ((spins & 1023u) == 0) {
            const cudaError_t e = cudaStreamQuery(ctx->stream);
            if (e == cudaSuccess && *f != epoch)
                return set_err(TD_ECUDA, "tree_decode: the combine kernel finished without its completion word");
            if (e != cudaSuccess && e != cudaErrorNotReady)
                return set_err(TD_ECUDA, std::string("tree_decode: ") + cudaGetErrorString(e));
        }
    }
    return TD_OK;
}

int tree_begin(td_context* ctx, const void* q, int64_t n_q, int strategy, int flags, TreeCall& tc,
               const void* q_on_device = nullptr) {
    if (int rc = require_ctx(ctx)) return rc;
    ctx->det = call_deterministic(flags);
    if (int rc = debug_begin(ctx, flags)) return rc;
    if (!ctx->kv_ok) return set_err(TD_ESTATE, "tree_decode: no KV shard placed");
    if (strategy < 0 || strategy > 2) return set_err(TD_EINVAL, "tree_decode: unknown strategy");
    if (ctx->nranks > ctx->seq_len) return set_err(TD_EINVAL, "tree_decode: more workers than keys");
    if (n_q % ctx->n_kv != 0) return set_err(TD_EINVAL, "tree_decode: q/kv head mismatch");
    ctx->last_kernels = 0;
    ctx->last_kv_bytes = 0.0;
    tc.rows = ctx->b * n_q;
    if (int rc = ensure_rows(ctx, tc.rows, ctx->d)) return rc;
    if (int rc = stream_failed(ctx)) return rc;  // an earlier asynchronous step
    if (int rc = plan_for(ctx, n_q, ctx->len, tc.plan, ctx->cap, false, true)) return rc;
    if (int rc = stream_setup(ctx, tc.plan)) return rc;
    int rc = TD_OK;
    if (!q_on_device && pinned_fast_path(ctx, flags, tc.plan)) {
        // the output goes straight into the caller's pinned buffer and the combine
        // kernel signals completion through pinned host memory (no stream sync)
        SplitPlan& pl = tc.plan;
        if (int rc2 = ensure_signals(ctx)) return rc2;
        pl.done_ctr = static_cast<unsigned*>(ctx->sig.p);
        pl.done_flag = ctx->done_host;
        pl.done_epoch = ++ctx->done_epoch == 0 ? ++ctx->done_epoch : ctx->done_epoch;
        tc.fast = true;
    }
    tc.qd = q_on_device ? q_on_device : stage_q(ctx, q, n_q, flags, &rc);
    if (rc) return rc;
    phase_begin(ctx, flags);
    phase_mark(ctx);
    return TD_OK;
}

// K1 + K2x: split-KV partial, then one exchange + exact combine into xdst
// (device memory or a mapped host buffer); no synchronisation. parts = 1 launches
// K1 only, 2 the exchange kernel only (with the same arguments), 3 both.
int launch_tree_p2p(td_context* ctx, const TreeCall& tc, double scale, float* xdst, int flags, int parts = 3) {
    const SplitPlan& plan = tc.plan;
    const int64_t d = ctx->d;
    if (!ctx->x_ready) return set_err(TD_ESTATE, "tree_decode: TD_P2P without td_p2p_open");
    if (tc.rows > ctx->x_max_rows || d != ctx->x_d)
        return set_err(TD_EINVAL, "tree_decode: exchange buffer too small for b * n_q rows");
    if (parts & 1)
        if (int rc = exchange_failed(ctx)) return rc;  // an earlier asynchronous step timed out
    td::XchgArgs xa;
    xa.peers = static_cast<float* const*>(ctx->x_ptrs.p);
    xa.p = ctx->nranks;
    xa.rank = ctx->rank;
    xa.epoch = ctx->x_epoch + 1;  // committed only once the launch is in: all ranks stay in step
    xa.max_rows = ctx->x_max_rows;
    // co-resident warp budget of the exchange kernel (TD_XCHG_WARPS_PER_SM, 8): its grid must
    // fit next to the next step's K1 (it only matters for the wide many-row launch: cfg4
    // at N=4 340.4 / 343.2 us with 8 vs 352.6 / 354.9 with 4, profiles/r2_k2_wide/);
    // workers sharing a GPU keep 4
    static const int xw = [] { const char* e = std::getenv("TD_XCHG_WARPS_PER_SM"); return e ? std::atoi(e) : 8; }();
    xa.max_blocks = std::min<int64_t>(td::kXchgBlocks, int64_t(ctx->shared_device ? 4 : std::max(1, xw)) * ctx->sm_count);
    xa.error = ctx->x_err;
    static const int pull = [] { const char* e = std::getenv("TD_XCHG_PULL"); return e ? std::atoi(e) : 0; }();
    xa.pull = pull;
    const CUtensorMap* pk = plan.kernel == 1 ? &ctx->tmk : nullptr;
    const CUtensorMap* pv = plan.kernel == 1 ? &ctx->tmv : nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (flags & TD_TIME_KERNELS) {
        cudaEvent_t* pr = next_timer(ctx);
        e0 = pr[0];
        e1 = pr[1];
    } else if (ctx->cur_phase) {
        e1 = (*ctx->cur_phase)[ctx->cur_mark++];
    }
    TD_CUDA(td::launch_decode_exchange(plan, tc.qd, ctx->k.p, ctx->v.p, static_cast<float>(scale), pk, pv,
                                       ctx->ws.p, xa, xdst, ctx->stream, e0, e1, parts));
    if (parts & 1) launched(ctx, plan);
    if (!(parts & 2)) return TD_OK;  // the exchange kernel follows (group, shared GPU)
    ctx->x_epoch = xa.epoch;
    ctx->kv_safe = plan.app_k ? plan.app_pos : ctx->len;  // later K1s run after this one's wait
    phase_mark(ctx);
    ctx->last_kernels = 2;  // K1 + K2x
    ctx->last_kv_bytes = 2.0 * double(ctx->b) * double(ctx->n_kv) * double(ctx->len) * double(d) *
                         td::dtype_bytes(ctx->dtype);
    ctx->last_split_kernel = plan.kernel;
    return TD_OK;
}

// TD_GRAPH (per call) or TD_NCCL_GRAPH=1 (process): replay the paper-literal NCCL
// step as a CUDA graph. Applies to device buffers with the static split (no pool
// counters to alternate) and no per-call instrumentation.
bool graph_mode(td_context* ctx, const SplitPlan& plan, int flags) {
    static const bool env = [] { const char* e = std::getenv("TD_NCCL_GRAPH"); return e && std::atoi(e) != 0; }();
    if (!(env || (flags & TD_GRAPH))) return false;
    if (flags & (TD_HOST_IO | TD_TIME_KERNELS | TD_TIME_PHASES | TD_BF16_OUT | TD_DEBUG_TS)) return false;
    return !plan.dbg && !plan.tl && !plan.app_k && ctx->comm;
}

// The NCCL tree step as a graph: captured on the first call of a shape and pool
// parity (the capture records the launches without running them; launches with a
// tile pool alternate two counter sets, hence two graphs), then launched; later calls
// with the same shape, buffers and scale only patch K1's claim epoch and relaunch.
int tree_nccl_graph(td_context* ctx, const SplitPlan& plan, const void* qd, double scale, int64_t rows, float* lse,
                    float* shift, float* nd, float* out) {
    auto& g = ctx->graph[plan.pool_tiles > 0 ? plan.parity & 1 : 0];
    const int64_t d = ctx->d;
    const bool same = g.exec && g.q == qd && g.out == out && g.scale == scale && g.rows == rows &&
                      g.total == plan.total_tiles && g.per_bh == plan.tiles_per_bh && g.len == ctx->len &&
                      g.cap == ctx->cap && g.ctas == plan.ctas && g.maxseg == plan.maxseg && g.kernel == plan.kernel &&
                      g.x_table == plan.x_table && g.k == ctx->k.p && g.lse == lse && g.t_safe == plan.t_safe &&
                      g.sflag == plan.sflag;
    if (same) {
        TD_CUDA(td::graph_set_k1_epoch(g.exec, g.k1, plan));
        if (g.k2s) TD_CUDA(td::graph_set_k2_epoch(g.exec, g.k2s, plan));
        launched(ctx, plan);  // (the capture path's run_partial does this)
    } else {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
        g = td_context::Graph{};
        TD_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        int rc = run_partial(ctx, plan, qd, ctx->k.p, ctx->v.p, ctx->len, scale, ctx->tm_ok, ctx->row_max, lse,
                             ctx->out_local, false);
        if (rc == TD_OK && nccl().AllReduce(lse, shift, size_t(rows), ncclFloat32, ncclMax, ctx->comm, ctx->stream) !=
                               ncclSuccess)
            rc = set_err(TD_ENCCL, "tree_decode (graph): allreduce(max) capture failed");
        if (rc == TD_OK && td::launch_to_numerator(lse, ctx->out_local, shift, rows, static_cast<int>(d), nd,
                                                   ctx->stream) != cudaSuccess)
            rc = set_err(TD_ECUDA, "tree_decode (graph): K3 capture failed");
        if (rc == TD_OK && nccl().AllReduce(nd, nd, size_t(rows * d + rows), ncclFloat32, ncclSum, ctx->comm,
                                            ctx->stream) != ncclSuccess)
            rc = set_err(TD_ENCCL, "tree_decode (graph): allreduce(sum) capture failed");
        if (rc == TD_OK &&
            td::launch_finalize(nd, rows, static_cast<int>(d), out, nullptr, ctx->stream) != cudaSuccess)
            rc = set_err(TD_ECUDA, "tree_decode (graph): K4 capture failed");
        cudaGraph_t graph = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(ctx->stream, &graph);
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        TD_CUDA(ec);
        g.graph = graph;
        TD_CUDA(cudaGraphInstantiate(&g.exec, graph, 0));
        size_t n = 0;
        TD_CUDA(cudaGraphGetNodes(graph, nullptr, &n));
        std::vector<cudaGraphNode_t> nodes(n);
        TD_CUDA(cudaGraphGetNodes(graph, nodes.data(), &n));
        const void* k1f = td::k1_function(plan);
        for (cudaGraphNode_t node : nodes) {
            cudaGraphNodeType t;
            if (cudaGraphNodeGetType(node, &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
            cudaKernelNodeParams kp{};
            if (cudaGraphKernelNodeGetParams(node, &kp) == cudaSuccess && kp.func == k1f) g.k1 = node;
            if (plan.sflag && kp.func == td::k2_stream_function()) g.k2s = node;
        }
        cudaGetLastError();
        if (!g.k1) return set_err(TD_ECUDA, "tree_decode (graph): split kernel node not found");
        if (td::stream_plan(plan) && !g.k2s) return set_err(TD_ECUDA, "tree_decode (graph): combine node not found");
        g.q = qd;
        g.out = out;
        g.scale = scale;
        g.rows = rows;
        g.total = plan.total_tiles;
        g.per_bh = plan.tiles_per_bh;
        g.len = ctx->len;
        g.cap = ctx->cap;
        g.ctas = plan.ctas;
        g.maxseg = plan.maxseg;
        g.kernel = plan.kernel;
        g.x_table = plan.x_table;
        g.k = ctx->k.p;
        g.lse = lse;
        g.t_safe = plan.t_safe;
        g.sflag = plan.sflag;
    }
    TD_CUDA(cudaGraphLaunch(g.exec, ctx->stream));
    ctx->kv_safe = ctx->len;
    ctx->last_kernels = 4;  // K1, K2, K3, K4 (+ two NCCL kernels)
    ctx->last_kv_bytes = 2.0 * double(ctx->b) * double(ctx->n_kv) * double(ctx->len) * double(d) *
                         td::dtype_bytes(ctx->dtype);
    ctx->last_split_kernel = plan.kernel;
    return note_table_use(ctx);
}

}  // namespace

extern "C" {

int td_tree_decode(td_context* ctx, const void* q, int64_t n_q, double scale, int strategy,
                   float* out, int flags) {
    TreeCall tc;
    if (int rc = tree_begin(ctx, q, n_q, strategy, flags, tc)) return rc;
    const SplitPlan& plan = tc.plan;
    const void* qd = tc.qd;
    const int64_t rows = tc.rows;
    const int64_t d = ctx->d;
    int rc = TD_OK;
    if ((flags & TD_P2P) && ctx->nranks > 1) {
        float* xdst = out;
        if ((flags & TD_HOST_IO) && !tc.fast) {
            float* m = (flags & TD_BF16_OUT) || !xchg_in_place(rows, d) ? nullptr : mapped_host(ctx, out);
            xdst = m ? m : ctx->out;
        }
        if (int rc2 = launch_tree_p2p(ctx, tc, scale, xdst, flags)) return rc2;
        if (tc.fast) {
            if (int rc2 = note_table_use(ctx)) return rc2;
            if (int rc2 = wait_done(ctx, plan.done_epoch)) return rc2;
        } else if (int rc2 = deliver_out(ctx, xdst, rows, out, flags)) {
            return rc2;
        }
        return (flags & TD_HOST_IO) ? exchange_failed(ctx) : TD_OK;  // synchronised: this step's verdict
    }
    if (ctx->nranks == 1) {
        // p = 1: the shard partial is the result (shift = lse, w = 1): one kernel,
        // written straight into the caller's buffer when it is on the device
        float* dst = out;
        if ((flags & TD_HOST_IO) && !tc.fast) {
            float* m = (flags & TD_BF16_OUT) ? nullptr : mapped_host(ctx, out);
            dst = m ? m : ctx->out;
        }
        const CUtensorMap* pk = plan.kernel == 1 ? &ctx->tmk : nullptr;
        const CUtensorMap* pv = plan.kernel == 1 ? &ctx->tmv : nullptr;
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (flags & TD_TIME_KERNELS) {
            cudaEvent_t* pr = next_timer(ctx);
            e0 = pr[0];
            e1 = pr[1];
        }
        unsigned long long* dbg = (flags & TD_DEBUG_TS) ? static_cast<unsigned long long*>(ctx->dbg.p) : nullptr;
        if (dbg) TD_CUDA(td::launch_stamp(dbg + 2, ctx->stream));
        TD_CUDA(td::launch_decode_final(plan, qd, ctx->k.p, ctx->v.p, static_cast<float>(scale), pk, pv,
                                        ctx->ws.p, dst, ctx->stream, e0, e1));
        launched(ctx, plan);
        if (dbg) TD_CUDA(td::launch_stamp(dbg + 3, ctx->stream));
        phase_mark(ctx);
        ctx->last_kernels = 2;  // K1 + K2
        ctx->last_kv_bytes = 2.0 * double(ctx->b) * double(ctx->n_kv) * double(ctx->len) * double(d) *
                             td::dtype_bytes(ctx->dtype);
        ctx->last_split_kernel = plan.kernel;
        if (!tc.fast) {
            if (int rc2 = deliver_out(ctx, dst, rows, out, flags)) return rc2;
            return (flags & TD_HOST_IO) ? stream_failed(ctx) : TD_OK;  // synchronised: this step's verdict
        }
        if (int rc2 = note_table_use(ctx)) return rc2;
        if (int rc2 = wait_done(ctx, plan.done_epoch)) return rc2;
        return stream_failed(ctx);
    }
    if (flags & TD_NCCL_DEVICE) {
        // K1 -> K2 (lse, out per row) -> K2n: allreduce(max), n/d numerators,
        // allreduce(sum), n/d in one kernel over the ranks' symmetric windows
        if (int rc2 = exchange_failed(ctx)) return rc2;
        if (int rc2 = nccl_dev_open(ctx, rows, d)) return rc2;
        float* dst = ctx->out;
        if (!(flags & TD_HOST_IO)) dst = out;
        else if (!(flags & TD_BF16_OUT) && xchg_in_place(rows, d)) if (float* m = mapped_host(ctx, out)) dst = m;
        td::XchgArgs xa;
        xa.peers = static_cast<float* const*>(ctx->nx_ptrs.p);
        xa.p = ctx->nranks;
        xa.rank = ctx->rank;
        xa.epoch = ctx->nx_epoch + 1;
        xa.max_rows = ctx->nx_rows;
        xa.max_blocks = std::min<int64_t>(td::kXchgBlocks, 4 * int64_t(ctx->sm_count));
        xa.error = ctx->x_err;
        // with the streamed combine the two rounds run inside the combine kernel
        // (TD_NCCL_FUSED=0: K2 then K2n, two kernels)
        static const bool fused = [] { const char* e = std::getenv("TD_NCCL_FUSED"); return !e || std::atoi(e) != 0; }();
        if (fused && td::stream_plan(plan) && rows * 4 <= std::min<int64_t>(plan.ctas, xa.max_blocks) &&
            !(flags & (TD_TIME_KERNELS | TD_TIME_PHASES))) {
            const CUtensorMap* pk = plan.kernel == 1 ? &ctx->tmk : nullptr;
            const CUtensorMap* pv = plan.kernel == 1 ? &ctx->tmv : nullptr;
            TD_CUDA(td::launch_decode_literal(plan, qd, ctx->k.p, ctx->v.p, static_cast<float>(scale), pk, pv,
                                              ctx->ws.p, xa, dst, ctx->stream));
            launched(ctx, plan);
            ctx->kv_safe = plan.app_k ? plan.app_pos : ctx->len;
            ctx->last_kernels = 2;  // K1 + the combine kernel
            ctx->last_kv_bytes = 2.0 * double(ctx->b) * double(ctx->n_kv) * double(ctx->len) * double(d) *
                                 td::dtype_bytes(ctx->dtype);
            ctx->last_split_kernel = plan.kernel;
        } else {
            if ((rc = run_partial(ctx, plan, qd, ctx->k.p, ctx->v.p, ctx->len, scale, ctx->tm_ok, ctx->row_max,
                                  ctx->lse, ctx->out_local, (flags & TD_TIME_KERNELS) != 0,
                                  ctx->cur_phase ? ctx : nullptr)))
                return rc;
            phase_mark(ctx);
            TD_CUDA(td::launch_literal_combine(ctx->lse, ctx->out_local, xa, rows, static_cast<int>(d), dst,
                                               ctx->stream));
            ctx->last_kernels += 1;
        }
        ctx->nx_epoch = xa.epoch;
        phase_mark(ctx);
        if (int rc2 = deliver_out(ctx, dst, rows, out, flags)) return rc2;
        return (flags & TD_HOST_IO) ? exchange_failed(ctx) : TD_OK;
    }
    // the allreduced buffers: in a symmetric NCCL window when available
    float *lse = ctx->lse, *shift = ctx->shift, *nd = ctx->nd;
    if (ctx->nranks > 1) {
        if (float* w = nccl_window(ctx, rows, d)) {
            const int64_t pr = (rows + 63) / 64 * 64;
            lse = w;
            shift = w + pr;
            nd = w + 2 * pr;
        }
    }
    if (ctx->nranks > 1 && graph_mode(ctx, plan, flags)) return tree_nccl_graph(ctx, plan, qd, scale, rows, lse, shift, nd, out);
    // 1. local partial (out, lse) of this shard
    if ((rc = run_partial(ctx, plan, qd, ctx->k.p, ctx->v.p, ctx->len, scale, ctx->tm_ok,
                          ctx->row_max, lse, ctx->out_local, (flags & TD_TIME_KERNELS) != 0,
                          ctx->cur_phase ? ctx : nullptr)))
        return rc;
    phase_mark(ctx);
    const float* result = ctx->out_local;
    if (ctx->nranks > 1) {
        // 2. allreduce(max) over lse -> common shift (decode.cpp:129-139)
        TD_NCCL(nccl().AllReduce(lse, shift, size_t(rows), ncclFloat32, ncclMax, ctx->comm, ctx->stream));
        phase_mark(ctx);
        // 3. n = o e^(lse-m), d = e^(lse-m) (decode.cpp:150-153)
        TD_CUDA(td::launch_to_numerator(lse, ctx->out_local, shift, rows, static_cast<int>(d), nd, ctx->stream));
        phase_mark(ctx);
        // 4. one fused sum-allreduce over [n|d] (decode.cpp:154-160); fp32 wire
        TD_NCCL(nccl().AllReduce(nd, nd, size_t(rows * d + rows), ncclFloat32, ncclSum, ctx->comm, ctx->stream));
        phase_mark(ctx);
        // 5. out = n / d (decode.cpp:165-173)
        TD_CUDA(td::launch_finalize(nd, rows, static_cast<int>(d), ctx->out, nullptr, ctx->stream));
        phase_mark(ctx);
        ctx->last_kernels += 2;
        result = ctx->out;
    }
    return deliver_out(ctx, result, rows, out, flags);
}

int td_local_partial(td_context* ctx, const void* q, int64_t n_q, double scale, float* row_max,
                     float* lse, float* out, int flags) {
    if (int rc = require_ctx(ctx)) return rc;
    ctx->det = call_deterministic(flags);
    if (int rc = debug_begin(ctx, flags)) return rc;
    if (!ctx->kv_ok) return set_err(TD_ESTATE, "local_partial: no KV shard placed");
    if (n_q % ctx->n_kv != 0) return set_err(TD_EINVAL, "local_partial: q/kv head mismatch");
    ctx->last_kernels = 0;
    ctx->last_kv_bytes = 0.0;
    const int64_t rows = ctx->b * n_q, d = ctx->d;
    if (int rc = ensure_rows(ctx, rows, d)) return rc;
    SplitPlan plan;
    if (int rc = plan_for(ctx, n_q, ctx->len, plan, ctx->cap)) return rc;
    int rc = TD_OK;
    const void* qd = stage_q(ctx, q, n_q, flags, &rc);
    if (rc) return rc;
    const bool host = (flags & TD_HOST_IO) != 0;
    if ((rc = run_partial(ctx, plan, qd, ctx->k.p, ctx->v.p, ctx->len, scale, ctx->tm_ok,
                          host ? ctx->r_max : row_max, host ? ctx->r_lse : lse,
                          host ? ctx->r_out : out, (flags & TD_TIME_KERNELS) != 0)))
        return rc;
    if ((rc = note_table_use(ctx))) return rc;
    if (host) {
        TD_CUDA(cudaMemcpyAsync(row_max, ctx->r_max, rows * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        TD_CUDA(cudaMemcpyAsync(lse, ctx->r_lse, rows * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        TD_CUDA(cudaMemcpyAsync(out, ctx->r_out, rows * d * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
        TD_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    return TD_OK;
}

// Alg. 1 (energy_forward_parallel over the ranks' shards): local (row_max,
// lse) of q.k + src.v -> allreduce(max) -> e^(lse - max) -> allreduce(sum) ->
// shifted = log(sum), value = max + shifted. Device pointers; q, src
// [b][h][nq][d] with h = the shard's kv heads.
int td_energy_forward(td_context* ctx, const void* q, const void* src, int64_t nq, float* value,
                      float* row_max, float* shifted, int flags) {
    if (int rc = require_ctx(ctx)) return rc;
    ctx->det = g_deterministic != 0;
    if (int rc = debug_begin(ctx, flags & ~TD_DEBUG_TS)) return rc;
    if (!ctx->kv_ok) return set_err(TD_ESTATE, "energy_forward: no KV shard placed");
    if (nq < 1) return set_err(TD_EINVAL, "energy_forward: need nq >= 1");
    if (ctx->nranks > ctx->seq_len) return set_err(TD_EINVAL, "energy_forward: more workers than keys");
    const int64_t n_q = ctx->n_kv * nq, rows = ctx->b * n_q, d = ctx->d;
    if (int rc = ensure_rows(ctx, rows, d)) return rc;
    SplitPlan plan;
    if (int rc = plan_for(ctx, n_q, ctx->len, plan, ctx->cap, true)) return rc;
    TD_CUDA(td::launch_decode_partial(plan, q, ctx->k.p, ctx->v.p, 1.0f, nullptr, nullptr, ctx->ws.p, ctx->r_max,
                                      ctx->r_lse, ctx->out_local, ctx->stream, nullptr, nullptr, src));
    if (ctx->nranks == 1) {
        TD_CUDA(td::launch_energy_combine(1, ctx->r_max, ctx->r_lse, rows, value, row_max, shifted, ctx->stream));
        ctx->last_kernels = 3;
        return TD_OK;
    }
    TD_NCCL(nccl().AllReduce(ctx->r_max, ctx->shift, size_t(rows), ncclFloat32, ncclMax, ctx->comm, ctx->stream));
    TD_CUDA(td::launch_energy_shift(ctx->r_lse, ctx->shift, rows, ctx->lse, ctx->stream));
    TD_NCCL(nccl().AllReduce(ctx->lse, ctx->lse, size_t(rows), ncclFloat32, ncclSum, ctx->comm, ctx->stream));
    TD_CUDA(td::launch_energy_finish(ctx->shift, ctx->lse, rows, value, row_max, shifted, ctx->stream));
    ctx->last_kernels = 4;
    return TD_OK;
}

// Alg. 2 (energy_grad_parallel): with the saved forward F = row_max + shifted,
// each rank's sum_a e^(s_a - F) v_a over its shard, then one allreduce(sum).
// No source (the gradient at zero source is the attention output).
int td_energy_grad(td_context* ctx, const void* q, int64_t nq, const float* row_max, const float* shifted,
                   float* grad, int flags) {
    if (int rc = require_ctx(ctx)) return rc;
    ctx->det = g_deterministic != 0;
    if (int rc = debug_begin(ctx, flags & ~TD_DEBUG_TS)) return rc;
    if (!ctx->kv_ok) return set_err(TD_ESTATE, "energy_grad: no KV shard placed");
    if (nq < 1) return set_err(TD_EINVAL, "energy_grad: need nq >= 1");
    if (ctx->nranks > ctx->seq_len) return set_err(TD_EINVAL, "energy_grad: more workers than keys");
    const int64_t n_q = ctx->n_kv * nq, rows = ctx->b * n_q, d = ctx->d;
    if (int rc = ensure_rows(ctx, rows, d)) return rc;
    SplitPlan plan;
    if (int rc = plan_for(ctx, n_q, ctx->len, plan, ctx->cap, true)) return rc;
    TD_CUDA(td::launch_decode_partial(plan, q, ctx->k.p, ctx->v.p, 1.0f, nullptr, nullptr, ctx->ws.p, ctx->r_max,
                                      ctx->r_lse, ctx->out_local, ctx->stream));
    TD_CUDA(td::launch_energy_logz(row_max, shifted, rows, ctx->shift, ctx->stream));
    // n = out * e^(lse - F): the partial_to_numerator kernel with shift F
    TD_CUDA(td::launch_to_numerator(ctx->r_lse, ctx->out_local, ctx->shift, rows, static_cast<int>(d), ctx->nd,
                                    ctx->stream));
    if (ctx->nranks > 1)
        TD_NCCL(nccl().AllReduce(ctx->nd, ctx->nd, size_t(rows * d), ncclFloat32, ncclSum, ctx->comm, ctx->stream));
    TD_CUDA(cudaMemcpyAsync(grad, ctx->nd, size_t(rows * d) * sizeof(float), cudaMemcpyDeviceToDevice, ctx->stream));
    ctx->last_kernels = 4;
    return TD_OK;
}

int td_ring_decode(td_context* ctx, const void* q, int64_t n_q, double scale, float* out,
                   int flags) {
    if (int rc = require_ctx(ctx)) return rc;
    ctx->det = call_deterministic(flags);
    if (int rc = debug_begin(ctx, flags)) return rc;
    if (!ctx->kv_ok) return set_err(TD_ESTATE, "ring_decode: no KV shard placed");
    if (int rc = flush_append(ctx)) return rc;  // the shard is sent as it sits in HBM
    if (ctx->nranks > ctx->seq_len) return set_err(TD_EINVAL, "ring_decode: more workers than keys");
    if (n_q % ctx->n_kv != 0) return set_err(TD_EINVAL, "ring_decode: q/kv head mismatch");
    ctx->last_kernels = 0;
    ctx->last_kv_bytes = 0.0;
    const int p = ctx->nranks, w = ctx->rank;
    const int64_t rows = ctx->b * n_q, d = ctx->d;
    if (int rc = ensure_rows(ctx, rows, d)) return rc;
    int rc = TD_OK;
    const void* qd = stage_q(ctx, q, n_q, flags, &rc);
    if (rc) return rc;
    const bool timed = (flags & TD_TIME_KERNELS) != 0;
    // shard lengths: chunk_extents at placement, grown by td_kv_append on rank p-1
    const std::vector<int64_t>& ext = ctx->lens;
    if (ext.size() != size_t(p) || ext[size_t(w)] != ctx->len)
        return set_err(TD_ESTATE, "ring_decode: shards are not the chunk_extents placement");
    const int64_t max_len = *std::max_element(ext.begin(), ext.end());
    const size_t esz = td::dtype_bytes(ctx->dtype);
    const size_t row_bytes = size_t(ctx->b) * size_t(ctx->n_kv) * size_t(d) * esz;

    // own chunk first: root = parts[w]
    SplitPlan plan;
    if ((rc = plan_for(ctx, n_q, ctx->len, plan, ctx->cap))) return rc;
    if ((rc = stream_setup(ctx, plan))) return rc;  // as tree_decode: bitwise the same partial
    if ((rc = run_partial(ctx, plan, qd, ctx->k.p, ctx->v.p, ctx->len, scale, ctx->tm_ok,
                          ctx->r_max, ctx->r_lse, ctx->r_out, timed)))
        return rc;
    if (p > 1) {
        for (auto& rb : ctx->ring)
            for (auto& x : rb) TD_CUDA(x.ensure(max_len * row_bytes > 0 ? max_len * row_bytes : 16));
        while (ctx->ring_ev.size() < 4) {  // start, recv-done, computed[buf 0], computed[buf 1]
            cudaEvent_t e;
            TD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ctx->ring_ev.push_back(e);
        }
        const int next = (w + 1) % p, prev = (w - 1 + p) % p;
        const void* cur_k = ctx->k.p;
        const void* cur_v = ctx->v.p;
        int64_t cur_len = ctx->len;
        if (ctx->cap != ctx->len) {  // appended shard: rows are cap apart, send them packed
            const size_t tok = size_t(d) * esz, nbh = size_t(ctx->b) * size_t(ctx->n_kv);
            for (int i = 0; i < 2; ++i) {
                TD_CUDA(ctx->ring_own[i].ensure(nbh * size_t(ctx->len) * tok + 16));
                TD_CUDA(cudaMemcpy2DAsync(ctx->ring_own[i].p, size_t(ctx->len) * tok, i ? ctx->v.p : ctx->k.p,
                                          size_t(ctx->cap) * tok, size_t(ctx->len) * tok, nbh,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
            }
            cur_k = ctx->ring_own[0].p;
            cur_v = ctx->ring_own[1].p;
        }
        // the transfer stream may start only once q/kv are ready on the compute stream
        TD_CUDA(cudaEventRecord(ctx->ring_ev[0], ctx->stream));
        TD_CUDA(cudaStreamWaitEvent(ctx->xfer, ctx->ring_ev[0], 0));
        for (int r = 0; r + 1 < p; ++r) {
            // worker w holds chunk (w - r) mod p, sends it to w+1, receives (w-1-r) mod p
            const int in_chunk = ((w - 1 - r) % p + p) % p;
            const int64_t in_len = ext[static_cast<size_t>(in_chunk)];
            DevBuf* dst = ctx->ring[r % 2];
            const size_t out_bytes = size_t(cur_len) * row_bytes, in_bytes = size_t(in_len) * row_bytes;
            // dst was last read by the partial of step r-2: wait for that compute only,
            // so this transfer overlaps the partial of step r-1 on the other buffer
            if (r >= 2) TD_CUDA(cudaStreamWaitEvent(ctx->xfer, ctx->ring_ev[2 + r % 2], 0));
            TD_NCCL(nccl().GroupStart());
            TD_NCCL(nccl().Send(cur_k, out_bytes, ncclUint8, next, ctx->comm, ctx->xfer));
            TD_NCCL(nccl().Send(cur_v, out_bytes, ncclUint8, next, ctx->comm, ctx->xfer));
            TD_NCCL(nccl().Recv(dst[0].p, in_bytes, ncclUint8, prev, ctx->comm, ctx->xfer));
            TD_NCCL(nccl().Recv(dst[1].p, in_bytes, ncclUint8, prev, ctx->comm, ctx->xfer));
            TD_NCCL(nccl().GroupEnd());
            TD_CUDA(cudaEventRecord(ctx->ring_ev[1], ctx->xfer));
            // compute on the received chunk once it lands, fold into the root
            TD_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ring_ev[1], 0));
            SplitPlan pl;
            if ((rc = plan_for(ctx, n_q, in_len, pl, 0))) return rc;
            if ((rc = run_partial(ctx, pl, qd, dst[0].p, dst[1].p, in_len, scale, false, ctx->row_max,
                                  ctx->lse, ctx->out_local, timed)))
                return rc;
            TD_CUDA(td::launch_combine_pair(ctx->r_max, ctx->r_lse, ctx->r_out, ctx->row_max,
                                            ctx->lse, ctx->out_local, rows, static_cast<int>(d),
                                            ctx->stream));
            ctx->last_kernels += 1;
            TD_CUDA(cudaEventRecord(ctx->ring_ev[2 + r % 2], ctx->stream));
            cur_k = dst[0].p;
            cur_v = dst[1].p;
            cur_len = in_len;
        }
    }
    if (p > 1) {  // the last transfer must be done before the next call reuses buffers
        TD_CUDA(cudaEventRecord(ctx->ring_ev[0], ctx->xfer));
        TD_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ring_ev[0], 0));
    }
    return deliver_out(ctx, ctx->r_out, rows, out, flags);
}

int td_output_bf16(td_context* ctx, const void** out_bf16) {
    if (int rc = require_ctx(ctx)) return rc;
    *out_bf16 = ctx->out_bf16.p;
    return TD_OK;
}

int td_calibration_info(td_context* ctx, double* gain, int* state) {
    if (int rc = require_ctx(ctx)) return rc;
    *gain = ctx->cal_gain;
    *state = ctx->cal_failed ? -1 : (ctx->cal_w.empty() ? 0 : (ctx->cal_gain > 0.005 ? 2 : 1));
    return TD_OK;
}

int td_kernel_time(td_context* ctx, double* mean_ms, int* calls) {
    if (int rc = require_ctx(ctx)) return rc;
    double total = 0.0;
    for (size_t i = 0; i < ctx->timers_used; ++i) {
        float ms = 0.f;
        TD_CUDA(cudaEventSynchronize(ctx->timers[i].second));
        TD_CUDA(cudaEventElapsedTime(&ms, ctx->timers[i].first, ctx->timers[i].second));
        total += ms;
    }
    *calls = static_cast<int>(ctx->timers_used);
    *mean_ms = ctx->timers_used ? total / double(ctx->timers_used) : 0.0;
    return TD_OK;
}

int td_reset_kernel_timer(td_context* ctx) {
    if (int rc = require_ctx(ctx)) return rc;
    ctx->timers_used = 0;
    ctx->phase_used = 0;
    return TD_OK;
}

int td_phase_times(td_context* ctx, double* phases, int max_phases, int* n, int* calls) {
    if (int rc = require_ctx(ctx)) return rc;
    int np = 0;
    for (int i = 0; i < max_phases; ++i) phases[i] = 0.0;
    // marks recorded per call are counted by querying each event's status
    for (size_t c = 0; c < ctx->phase_used; ++c) {
        auto& evs = ctx->phase_sets[c];
        int marks = 0;
        for (auto& e : evs) {
            if (cudaEventQuery(e) == cudaErrorNotReady) cudaEventSynchronize(e);
            float dummy;
            if (cudaEventElapsedTime(&dummy, evs[0], e) != cudaSuccess) break;
            ++marks;
        }
        cudaGetLastError();
        for (int i = 0; i + 1 < marks && i < max_phases; ++i) {
            float ms = 0.f;
            TD_CUDA(cudaEventElapsedTime(&ms, evs[size_t(i)], evs[size_t(i) + 1]));
            phases[i] += ms;
        }
        np = std::max(np, marks - 1);
    }
    for (int i = 0; i < max_phases; ++i) phases[i] /= ctx->phase_used ? double(ctx->phase_used) : 1.0;
    *n = np;
    *calls = static_cast<int>(ctx->phase_used);
    return TD_OK;
}

int td_last_launch_stats(td_context* ctx, int* kernels, double* kv_bytes, int* split_kernel) {
    if (int rc = require_ctx(ctx)) return rc;
    *kernels = ctx->last_kernels;
    *kv_bytes = ctx->last_kv_bytes;
    *split_kernel = ctx->last_split_kernel;
    return TD_OK;
}

int td_memory_bytes(td_context* ctx, size_t* bytes) {
    if (int rc = require_ctx(ctx)) return rc;
    size_t s = ctx->k.cap + ctx->v.cap + ctx->ws.cap + ctx->rows.cap + ctx->q_dev.cap +
               ctx->out_bf16.cap;
    for (auto& rb : ctx->ring)
        for (auto& x : rb) s += x.cap;
    *bytes = s;
    return TD_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- single-process worker group
// The reference runs its p workers in one process (decode.hpp:70-72; one
// std::thread per worker with parallel_workers, decode.cpp:37-41). A td_group
// is that: one context per worker, worker w on device devs[w * ndev / p]
// (contiguous placement, cluster.hpp:18-24), the exchange buffers of the
// one-shot combine addressed as plain device pointers (peer access over
// NVLink, or the same HBM when workers share a GPU) instead of CUDA IPC, and
// one host thread issuing every worker's launches asynchronously.
struct td_group {
    std::vector<td_context*> w;
    std::vector<int> dev;
    cudaEvent_t entry = nullptr;  // on worker 0's device: start of a call (orders the others after it)
    bool shared = false;          // some GPU hosts several workers
    std::vector<cudaEvent_t> k1_done;  // per worker (its device): K1 of the current call finished
};

extern "C" {

int td_group_create(int ndev, const int* devs, int workers, td_group** out) {
    if (!out) return set_err(TD_EINVAL, "td_group_create: null output");
    *out = nullptr;
    if (ndev < 1 || !devs || workers < 1) return set_err(TD_EINVAL, "td_group_create: need ndev >= 1 and workers >= 1");
    int n = 0;
    TD_CUDA(cudaGetDeviceCount(&n));
    for (int i = 0; i < ndev; ++i)
        if (devs[i] < 0 || devs[i] >= n) return set_err(TD_EINVAL, "td_group_create: no such device");
    auto* g = new td_group;
    auto fail = [&](int rc) {
        td_group_destroy(g);
        return rc;
    };
    for (int w = 0; w < workers; ++w) {
        const int dv = devs[int64_t(w) * ndev / workers];
        td_context* ctx = nullptr;
        if (int rc = td_create(dv, &ctx)) return fail(rc);
        ctx->nranks = workers;
        ctx->rank = w;
        g->w.push_back(ctx);
        g->dev.push_back(dv);
    }
    for (int w = 0; w < workers; ++w)
        for (int u = 0; u < workers; ++u)
            if (u != w && g->dev[size_t(u)] == g->dev[size_t(w)]) g->w[size_t(w)]->shared_device = true;
    // peer access between every pair of distinct devices (K2x stores into peers' HBM)
    for (int a = 0; a < workers; ++a)
        for (int b = 0; b < workers; ++b) {
            const int da = g->dev[size_t(a)], db = g->dev[size_t(b)];
            if (da == db) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, da, db);
            if (!can) return fail(set_err(TD_ECUDA, "td_group_create: no peer access between the devices"));
            cudaSetDevice(da);
            const cudaError_t e = cudaDeviceEnablePeerAccess(db, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                return fail(set_err(TD_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e)));
            cudaGetLastError();
        }
    cudaSetDevice(g->dev[0]);
    if (cudaEventCreateWithFlags(&g->entry, cudaEventDisableTiming) != cudaSuccess)
        return fail(set_err(TD_ECUDA, "td_group_create: event"));
    for (int w = 0; w < workers; ++w) {
        g->shared = g->shared || g->w[size_t(w)]->shared_device;
        cudaSetDevice(g->dev[size_t(w)]);
        cudaEvent_t e = nullptr;
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
            return fail(set_err(TD_ECUDA, "td_group_create: event"));
        g->k1_done.push_back(e);
    }
    *out = g;
    return TD_OK;
}

int td_group_destroy(td_group* g) {
    if (!g) return TD_OK;
    for (size_t w = 0; w < g->k1_done.size(); ++w) {
        cudaSetDevice(g->dev[w]);
        cudaEventDestroy(g->k1_done[w]);
    }
    for (td_context* ctx : g->w) td_destroy(ctx);
    if (g->entry) {
        cudaSetDevice(g->dev[0]);
        cudaEventDestroy(g->entry);
    }
    delete g;
    return TD_OK;
}

int td_group_context(td_group* g, int worker, td_context** ctx) {
    if (!g || !ctx || worker < 0 || worker >= int(g->w.size()))
        return set_err(TD_EINVAL, "td_group_context: no such worker");
    *ctx = g->w[size_t(worker)];
    return TD_OK;
}

int td_group_p2p_open(td_group* g, int64_t max_rows, int64_t d) {
    if (!g) return set_err(TD_EINVAL, "null td_group");
    std::vector<void*> base;
    for (td_context* ctx : g->w) {
        if (int rc = require_ctx(ctx)) return rc;
        if (int rc = xbuf_alloc(ctx, max_rows, d)) return rc;
        base.push_back(ctx->xbuf.p);
    }
    for (td_context* ctx : g->w) {
        if (int rc = require_ctx(ctx)) return rc;
        TD_CUDA(ctx->x_ptrs.ensure(base.size() * sizeof(void*)));
        TD_CUDA(cudaMemcpy(ctx->x_ptrs.p, base.data(), base.size() * sizeof(void*), cudaMemcpyHostToDevice));
        ctx->x_ready = true;
    }
    return TD_OK;
}

int td_group_tree_decode(td_group* g, const void* q, int64_t n_q, double scale, int strategy, float* out,
                         int flags) {
    if (!g) return set_err(TD_EINVAL, "null td_group");
    if (flags & (TD_BF16_OUT | TD_TIME_PHASES | TD_DEBUG_TS))
        return set_err(TD_EINVAL, "td_group_tree_decode: TD_BF16_OUT / TD_TIME_PHASES / TD_DEBUG_TS are per-context flags");
    flags &= ~TD_PINNED_IO;  // the group stages q and collects the output itself
    const int p = int(g->w.size());
    const bool host = (flags & TD_HOST_IO) != 0;
    td_context* c0 = g->w[0];
    if (int rc = require_ctx(c0)) return rc;
    // every worker's work is ordered after what the caller queued on worker 0's stream (a device q)
    TD_CUDA(cudaEventRecord(g->entry, c0->stream));
    for (int w = 1; w < p; ++w) {
        if (int rc = require_ctx(g->w[size_t(w)])) return rc;
        TD_CUDA(cudaStreamWaitEvent(g->w[size_t(w)]->stream, g->entry, 0));
    }
    if (p == 1) return td_tree_decode(c0, q, n_q, scale, strategy, out, flags);
    // 1. plans (and a first long decode's calibration) for every worker before any
    //    exchange is in flight; q onto every worker's device
    std::vector<TreeCall> tc(static_cast<size_t>(p));
    for (int w = 0; w < p; ++w) {
        td_context* ctx = g->w[size_t(w)];
        const void* qd = nullptr;
        if (!host) {
            if (g->dev[size_t(w)] == g->dev[0]) {
                qd = q;
            } else {
                if (int rc = require_ctx(ctx)) return rc;
                if (!ctx->kv_ok) return set_err(TD_ESTATE, "tree_decode: no KV shard placed");
                const size_t bytes = size_t(ctx->b) * size_t(n_q) * size_t(ctx->d) * td::dtype_bytes(ctx->dtype);
                TD_CUDA(ctx->q_dev.ensure(bytes));
                TD_CUDA(cudaMemcpyPeerAsync(ctx->q_dev.p, g->dev[size_t(w)], q, g->dev[0], bytes, ctx->stream));
                qd = ctx->q_dev.p;
            }
        }
        if (int rc = tree_begin(ctx, q, n_q, strategy, flags, tc[size_t(w)], qd)) return rc;
        if (ctx->b != c0->b || ctx->n_kv != c0->n_kv || ctx->d != c0->d || ctx->seq_len != c0->seq_len)
            return set_err(TD_EINVAL, "tree_decode: the workers' shards are not one cache");
    }
    // 2. K1 + K2x on every worker, back to back; worker 0 writes the caller's output
    float* dst0 = out;
    if (host) {
        require_ctx(c0);
        float* m = xchg_in_place(tc[0].rows, c0->d) ? mapped_host(c0, out) : nullptr;
        dst0 = m ? m : c0->out;
    }
    if (g->shared) {
        // Workers sharing a GPU: every worker's K1 first, then the exchange kernels,
        // each ordered after ALL the K1s. Exchange warps spin until their peers'
        // words arrive; resident before a peer's K1 has run, they could hold the
        // registers that K1's CTAs need and starve it (a deadlock the ~2 s timeout
        // ended: tests/cpp/shim_parity.cpp at p = 16 workers on one GPU).
        for (int w = 0; w < p; ++w) {
            td_context* ctx = g->w[size_t(w)];
            require_ctx(ctx);
            if (int rc = launch_tree_p2p(ctx, tc[size_t(w)], scale, w == 0 ? dst0 : ctx->out, flags, 1)) return rc;
            TD_CUDA(cudaEventRecord(g->k1_done[size_t(w)], ctx->stream));
        }
        for (int w = 0; w < p; ++w) {
            td_context* ctx = g->w[size_t(w)];
            require_ctx(ctx);
            for (int v = 0; v < p; ++v)
                if (v != w) TD_CUDA(cudaStreamWaitEvent(ctx->stream, g->k1_done[size_t(v)], 0));
            if (int rc = launch_tree_p2p(ctx, tc[size_t(w)], scale, w == 0 ? dst0 : ctx->out, flags, 2)) return rc;
            if (int rc = note_table_use(ctx)) return rc;
        }
    } else {
        for (int w = 0; w < p; ++w) {
            td_context* ctx = g->w[size_t(w)];
            require_ctx(ctx);
            if (int rc = launch_tree_p2p(ctx, tc[size_t(w)], scale, w == 0 ? dst0 : ctx->out, flags)) return rc;
            if (int rc = note_table_use(ctx)) return rc;
        }
    }
    if (!host) return TD_OK;
    require_ctx(c0);
    if (dst0 != c0->mapped_dev || c0->mapped_for != out)
        TD_CUDA(cudaMemcpyAsync(out, dst0, size_t(tc[0].rows) * size_t(c0->d) * sizeof(float), cudaMemcpyDeviceToHost,
                                c0->stream));
    int rc = TD_OK;
    for (int w = 0; w < p; ++w) {  // every worker's step is over: report any exchange timeout
        td_context* ctx = g->w[size_t(w)];
        require_ctx(ctx);
        TD_CUDA(cudaStreamSynchronize(ctx->stream));
        if (int e = exchange_failed(ctx)) rc = e;
    }
    return rc;
}

}  // extern "C"
