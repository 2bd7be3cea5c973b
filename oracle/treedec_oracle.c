/*
 * treedec_oracle.c -- CPU restatement of the reference tree-decode path.
 * TEST INFRASTRUCTURE ONLY (see treedec_oracle.h): the checker for the CUDA
 * product, never the product. Citations are relative to
 * /root/reference/proj/core. Build: oracle/Makefile (plain gcc, no -march
 * flags, so no FMA contraction; operation order follows the reference so
 * Float64 results are bitwise equal to it).
 */
#include "treedec_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define NEG_INF (-INFINITY)

/* ---- numerics.cpp:30-39 ------------------------------------------------ */
uint64_t orc_mix64(uint64_t seed, uint64_t counter) {
    uint64_t z = seed + (counter + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double orc_uniform01(uint64_t seed, uint64_t counter) {
    return (double)(orc_mix64(seed, counter) >> 11) * 0x1.0p-53;
}

/* ---- dtype.cpp:13-42 ----------------------------------------------------- */
static double round_bf16(double x) {
    if (x == 0.0 || !isfinite(x)) return x;
    int e = 0;
    (void)frexp(x, &e); /* |x| in [2^(e-1), 2^e) */
    int lsb = e - 8;
    if (lsb < -133) lsb = -133; /* bf16 subnormal quantum */
    const double y = ldexp(nearbyint(ldexp(x, -lsb)), lsb);
    if (fabs(y) >= 0x1p128) return copysign(INFINITY, x);
    return y;
}

static double round_f32(double x) {
    if (!isfinite(x)) return x;
    if (fabs(x) >= 0x1.ffffffp127) return copysign(INFINITY, x);
    return (double)(float)x;
}

double orc_round(double x, int dtype) {
    switch (dtype) {
    case ORC_F32: return round_f32(x);
    case ORC_BF16: return round_bf16(x);
    default: return x;
    }
}

int orc_stats_dtype(int dtype) { return dtype == ORC_BF16 ? ORC_F32 : dtype; }

/* ---- numerics.cpp:41-50 -------------------------------------------------- */
int orc_seeded_fill(uint64_t seed, double scale, int dtype, int64_t offset, int64_t n,
                    double* out) {
    if (!(scale > 0.0)) return -1;
    const double half_width = sqrt(3.0) * scale;
    for (int64_t i = 0; i < n; ++i) {
        const double u = orc_uniform01(seed, (uint64_t)(offset + i));
        out[i] = orc_round((2.0 * u - 1.0) * half_width, dtype);
    }
    return 0;
}

/* ---- attention.cpp:268-275 ----------------------------------------------- */
int orc_chunk_extents(int64_t n, int p, int64_t* out) {
    if (p < 1 || n < 0) return -1;
    const int64_t base = n / p, rem = n % p;
    for (int i = 0; i < p; ++i) out[i] = base + (i < rem ? 1 : 0);
    return 0;
}

/* ---- numerics.cpp:22-28 -------------------------------------------------- */
double orc_lse_combine(double a, double b) {
    if (isnan(a) || isnan(b)) return NAN;
    if (a == NEG_INF) return b;
    if (b == NEG_INF) return a;
    const double m = a > b ? a : b;
    return m + log(exp(a - m) + exp(b - m));
}

/* ---- attention.cpp:32-77: one (b, h) row of attention_chunk_partial ------- */
typedef struct {
    const double *q, *k, *v;
    int64_t b, n_q, n_kv, seq, start, len, d;
    double scale;
    int dtype;
    double *row_max, *lse, *out;
    int64_t row_begin, row_end;
} partial_job;

static void partial_rows(const partial_job* j) {
    const int sdt = orc_stats_dtype(j->dtype);
    const int64_t group = j->n_q / j->n_kv;
    double* scores = (double*)malloc(sizeof(double) * (size_t)(j->len > 0 ? j->len : 1));
    for (int64_t r = j->row_begin; r < j->row_end; ++r) {
        const int64_t ib = r / j->n_q, ih = r % j->n_q, kh = ih / group;
        const double* qr = j->q + r * j->d;
        const double* kb = j->k + ((ib * j->n_kv + kh) * j->seq + j->start) * j->d;
        const double* vb = j->v + ((ib * j->n_kv + kh) * j->seq + j->start) * j->d;
        double* orow = j->out + r * j->d;
        if (j->len == 0) { /* row_softmax_stats empty branch, :56-61 */
            j->row_max[r] = NEG_INF;
            j->lse[r] = NEG_INF;
            for (int64_t c = 0; c < j->d; ++c) orow[c] = 0.0;
            continue;
        }
        for (int64_t i = 0; i < j->len; ++i) { /* row_scores, :39-45 */
            double dot = 0.0;
            const double* kr = kb + i * j->d;
            for (int64_t c = 0; c < j->d; ++c) dot += qr[c] * kr[c];
            scores[i] = orc_round(dot * j->scale, j->dtype);
        }
        double m = scores[0]; /* :62-63 */
        for (int64_t i = 0; i < j->len; ++i) m = scores[i] > m ? scores[i] : m;
        double denom = 0.0;
        for (int64_t c = 0; c < j->d; ++c) orow[c] = 0.0;
        for (int64_t i = 0; i < j->len; ++i) { /* :67-72 */
            const double w = orc_round(exp(scores[i] - m), sdt);
            denom += w;
            const double* vr = vb + i * j->d;
            for (int64_t c = 0; c < j->d; ++c) orow[c] += w * vr[c];
        }
        for (int64_t c = 0; c < j->d; ++c) orow[c] = orc_round(orow[c] / denom, j->dtype);
        j->row_max[r] = m;
        j->lse[r] = orc_round(m + log(denom), sdt);
    }
    free(scores);
}

static void* partial_thread(void* arg) {
    partial_rows((const partial_job*)arg);
    return NULL;
}

int orc_chunk_partial(const double* q, const double* k, const double* v, int64_t b,
                      int64_t n_q, int64_t n_kv, int64_t seq, int64_t start, int64_t len,
                      int64_t d, double scale, int dtype, int nthreads, double* row_max,
                      double* lse, double* out) {
    if (b < 1 || n_q < 1 || n_kv < 1 || d < 1 || n_q % n_kv != 0) return -1;
    if (start < 0 || len < 0 || start + len > seq) return -1;
    const int64_t rows = b * n_q;
    partial_job base = {q, k, v, b, n_q, n_kv, seq, start, len, d, scale, dtype,
                        row_max, lse, out, 0, rows};
    if (nthreads <= 1 || rows == 1) {
        partial_rows(&base);
        return 0;
    }
    if (nthreads > rows) nthreads = (int)rows;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    partial_job* jobs = (partial_job*)malloc(sizeof(partial_job) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = base;
        jobs[t].row_begin = rows * t / nthreads;
        jobs[t].row_end = rows * (t + 1) / nthreads;
        pthread_create(&th[t], NULL, partial_thread, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    free(jobs);
    return 0;
}

/* ---- attention.cpp:178-205 ----------------------------------------------- */
int orc_combine_pair(const double* l_max, const double* l_lse, const double* l_out,
                     const double* r_max, const double* r_lse, const double* r_out, int64_t rows,
                     int64_t d, int dtype, double* o_max, double* o_lse, double* o_out) {
    const int sdt = orc_stats_dtype(dtype);
    for (int64_t r = 0; r < rows; ++r) {
        const double la = l_lse[r], lb = r_lse[r];
        const double lc = orc_lse_combine(la, lb);
        if (isnan(lc)) return -2;
        const double l = orc_round(lc, sdt);
        o_lse[r] = l;
        o_max[r] = l_max[r] > r_max[r] ? l_max[r] : r_max[r];
        const double wa = la == NEG_INF ? 0.0 : orc_round(exp(la - l), sdt);
        const double wb = lb == NEG_INF ? 0.0 : orc_round(exp(lb - l), sdt);
        for (int64_t c = 0; c < d; ++c)
            o_out[r * d + c] = orc_round(l_out[r * d + c] * wa + r_out[r * d + c] * wb, dtype);
    }
    return 0;
}

/* ---- attention.cpp:207-241 ----------------------------------------------- */
int orc_combine_partials(int P, const double* lse, const double* out, int64_t rows, int64_t d,
                         int dtype, double* result) {
    if (P < 1) return -1;
    const int sdt = orc_stats_dtype(dtype);
    double* num = (double*)malloc(sizeof(double) * (size_t)d);
    for (int64_t r = 0; r < rows; ++r) {
        double shift = NEG_INF;
        for (int p = 0; p < P; ++p) {
            const double l = lse[(int64_t)p * rows + r];
            shift = shift > l ? shift : l; /* std::max(shift, l) */
        }
        if (shift == NEG_INF) {
            free(num);
            return -1;
        }
        double denom = 0.0;
        for (int64_t c = 0; c < d; ++c) num[c] = 0.0;
        for (int p = 0; p < P; ++p) {
            const double l = lse[(int64_t)p * rows + r];
            if (l == NEG_INF) continue;
            const double w = orc_round(exp(l - shift), sdt);
            denom += w;
            const double* o = out + ((int64_t)p * rows + r) * d;
            for (int64_t c = 0; c < d; ++c) num[c] += o[c] * w;
        }
        for (int64_t c = 0; c < d; ++c) result[r * d + c] = orc_round(num[c] / denom, dtype);
    }
    free(num);
    return 0;
}

/* ---- attention.cpp:243-266 ----------------------------------------------- */
int orc_partial_to_numerator(const double* lse, const double* out, const double* shift,
                             int64_t rows, int64_t d, int dtype, double* num, double* den) {
    const int sdt = orc_stats_dtype(dtype);
    for (int64_t r = 0; r < rows; ++r) {
        const double l = lse[r];
        const double w = l == NEG_INF ? 0.0 : orc_round(exp(l - shift[r]), sdt);
        den[r] = w;
        for (int64_t c = 0; c < d; ++c) num[r * d + c] = orc_round(out[r * d + c] * w, dtype);
    }
    return 0;
}

/* ---- reduce.cpp:35-139: schedules as flat step lists ---------------------- */
typedef struct {
    int sender, receiver, combine;
} step_t;

typedef struct {
    step_t* steps;
    int* round_start; /* round r = steps[round_start[r], round_start[r+1]) */
    int n_steps, n_rounds, cap_steps, cap_rounds;
    int participants, reduce_rounds;
} schedule_t;

static void sched_init(schedule_t* s, int participants) {
    memset(s, 0, sizeof(*s));
    s->participants = participants;
    s->cap_steps = 64;
    s->cap_rounds = 64;
    s->steps = (step_t*)malloc(sizeof(step_t) * (size_t)s->cap_steps);
    s->round_start = (int*)malloc(sizeof(int) * (size_t)(s->cap_rounds + 1));
    s->round_start[0] = 0;
}

static void sched_free(schedule_t* s) {
    free(s->steps);
    free(s->round_start);
}

static void sched_push(schedule_t* s, int sender, int receiver, int combine) {
    if (s->n_steps == s->cap_steps) {
        s->cap_steps *= 2;
        s->steps = (step_t*)realloc(s->steps, sizeof(step_t) * (size_t)s->cap_steps);
    }
    s->steps[s->n_steps].sender = sender;
    s->steps[s->n_steps].receiver = receiver;
    s->steps[s->n_steps].combine = combine;
    s->n_steps++;
}

/* close the current round; empty rounds are kept only when keep_empty. */
static void sched_end_round(schedule_t* s, int keep_empty) {
    if (!keep_empty && s->n_steps == s->round_start[s->n_rounds]) return;
    if (s->n_rounds + 1 >= s->cap_rounds) {
        s->cap_rounds *= 2;
        s->round_start = (int*)realloc(s->round_start, sizeof(int) * (size_t)(s->cap_rounds + 1));
    }
    s->n_rounds++;
    s->round_start[s->n_rounds] = s->n_steps;
}

static int ceil_log2_int(int p) {
    int r = 0;
    while ((1 << r) < p) ++r;
    return r;
}

/* append_tree_reduce, reduce.cpp:37-44 (rounds always pushed) */
static void append_tree_reduce(schedule_t* s, int base, int count, int unit) {
    for (int stride = 1; stride < count; stride *= 2) {
        for (int i = 0; i + stride < count; i += 2 * stride)
            sched_push(s, base + (i + stride) * unit, base + i * unit, 1);
        sched_end_round(s, 1);
    }
}

/* append_tree_broadcast, reduce.cpp:47-56 (empty rounds skipped) */
static void append_tree_broadcast(schedule_t* s, int base, int count, int unit) {
    int top = 1;
    while (top < count) top *= 2;
    for (int stride = top / 2; stride >= 1; stride /= 2) {
        for (int i = 0; i + stride < count; i += 2 * stride)
            sched_push(s, base + i * unit, base + (i + stride) * unit, 0);
        sched_end_round(s, 0);
    }
}

static int build_schedule(int strategy, int nodes, int g, schedule_t* s) {
    if (nodes < 1 || g < 1) return -1;
    const int p = nodes * g;
    sched_init(s, p);
    if (strategy == ORC_TREE_BINARY) { /* reduce.cpp:60-72 */
        append_tree_reduce(s, 0, p, 1);
        s->reduce_rounds = s->n_rounds;
        append_tree_broadcast(s, 0, p, 1);
    } else if (strategy == ORC_RING) { /* reduce.cpp:74-84 */
        for (int r = 0; r + 1 < p; ++r) {
            sched_push(s, r, r + 1, 1);
            sched_end_round(s, 1);
        }
        s->reduce_rounds = p - 1;
        for (int r = 0; r + 1 < p; ++r) {
            sched_push(s, (p - 1 + r) % p, r, 0);
            sched_end_round(s, 1);
        }
    } else if (strategy == ORC_HIER) { /* reduce.cpp:86-130 */
        for (int r = 0; r + 1 < g; ++r) {
            for (int nd = 0; nd < nodes; ++nd) sched_push(s, nd * g + r, nd * g + r + 1, 1);
            sched_end_round(s, 1);
        }
        for (int stride = 1; stride < nodes; stride *= 2) {
            for (int i = 0; i + stride < nodes; i += 2 * stride)
                sched_push(s, (i + stride) * g + g - 1, i * g + g - 1, 1);
            sched_end_round(s, 1);
        }
        s->reduce_rounds = (g - 1) + ceil_log2_int(nodes);
        int top = 1;
        while (top < nodes) top *= 2;
        for (int stride = top / 2; stride >= 1; stride /= 2) {
            for (int i = 0; i + stride < nodes; i += 2 * stride)
                sched_push(s, i * g + g - 1, (i + stride) * g + g - 1, 0);
            sched_end_round(s, 0);
        }
        for (int r = 0; r + 1 < g; ++r) {
            for (int nd = 0; nd < nodes; ++nd) sched_push(s, nd * g + g - 1 - r, nd * g + g - 2 - r, 0);
            sched_end_round(s, 1);
        }
    } else {
        sched_free(s);
        return -1;
    }
    return 0;
}

int orc_schedule_rounds(int strategy, int nodes, int gpus_per_node, int* reduce_rounds,
                        int* total_rounds) {
    schedule_t s;
    if (build_schedule(strategy, nodes, gpus_per_node, &s) != 0) return -1;
    *reduce_rounds = s.reduce_rounds;
    *total_rounds = s.n_rounds;
    sched_free(&s);
    return 0;
}

/* execute_schedule, reduce.hpp:62-92, over p value slots of `width` doubles.
 * combine(lo, hi, dst) folds the lower-index operand on the left. */
typedef void (*combine_fn)(const double* lo, const double* hi, double* dst, int64_t width,
                           const void* ctx);

static void execute_schedule(const schedule_t* s, double* values, int64_t width,
                             combine_fn combine, const void* ctx) {
    double* results = NULL;
    size_t cap = 0;
    for (int r = 0; r < s->n_rounds; ++r) {
        const int a = s->round_start[r], e = s->round_start[r + 1];
        const size_t need = (size_t)(e - a) * (size_t)width;
        if (need > cap) {
            cap = need;
            results = (double*)realloc(results, sizeof(double) * cap);
        }
        for (int i = a; i < e; ++i) {
            const step_t* st = &s->steps[i];
            double* dst = results + (size_t)(i - a) * (size_t)width;
            if (!st->combine) {
                memcpy(dst, values + (size_t)st->sender * (size_t)width,
                       sizeof(double) * (size_t)width);
                continue;
            }
            const int lo = st->sender < st->receiver ? st->sender : st->receiver;
            const int hi = st->sender < st->receiver ? st->receiver : st->sender;
            combine(values + (size_t)lo * (size_t)width, values + (size_t)hi * (size_t)width,
                    dst, width, ctx);
        }
        for (int i = a; i < e; ++i)
            memcpy(values + (size_t)s->steps[i].receiver * (size_t)width,
                   results + (size_t)(i - a) * (size_t)width, sizeof(double) * (size_t)width);
    }
    free(results);
}

/* decode.cpp:133-138 */
static void combine_max(const double* a, const double* b, double* dst, int64_t width,
                        const void* ctx) {
    (void)ctx;
    for (int64_t i = 0; i < width; ++i) dst[i] = a[i] > b[i] ? a[i] : b[i];
}

typedef struct {
    int64_t num_width; /* rows * d, followed by rows denominators */
    int dtype, sdt;
} nd_ctx;

/* decode.cpp:154-160: num stored through dt, den through the stats grid. */
static void combine_nd(const double* a, const double* b, double* dst, int64_t width,
                       const void* vctx) {
    const nd_ctx* c = (const nd_ctx*)vctx;
    for (int64_t i = 0; i < c->num_width; ++i) dst[i] = orc_round(a[i] + b[i], c->dtype);
    for (int64_t i = c->num_width; i < width; ++i) dst[i] = orc_round(a[i] + b[i], c->sdt);
}

/* topology_for_workers, cluster.cpp:11-22 (default 8 GPUs per node) */
static int topology_for_workers(int p, int* nodes, int* g) {
    if (p < 1) return -1;
    if (p <= 8) {
        *nodes = 1;
        *g = p;
        return 0;
    }
    if (p % 8 != 0) return -1;
    *nodes = p / 8;
    *g = 8;
    return 0;
}

/* local_partials (decode.cpp:28-46) over shard_kv extents (decode.cpp:68-85).
 * parts: max [p][rows], lse [p][rows], out [p][rows][d]. */
static int local_partials(const double* q, const double* k, const double* v, int64_t b,
                          int64_t n_q, int64_t n_kv, int64_t seq, int64_t d, int p, double scale,
                          int dtype, int nthreads, double* pmax, double* plse, double* pout) {
    if (p < 1 || p > seq) return -1;
    int64_t* ext = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
    orc_chunk_extents(seq, p, ext);
    const int64_t rows = b * n_q;
    int64_t begin = 0;
    int rc = 0;
    for (int w = 0; w < p && rc == 0; ++w) {
        rc = orc_chunk_partial(q, k, v, b, n_q, n_kv, seq, begin, ext[w], d, scale, dtype,
                               nthreads, pmax + w * rows, plse + w * rows, pout + w * rows * d);
        begin += ext[w];
    }
    free(ext);
    return rc;
}

int orc_tree_decode(const double* q, const double* k, const double* v, int64_t b, int64_t n_q,
                    int64_t n_kv, int64_t seq, int64_t d, int p, int strategy, double scale,
                    int dtype, int nthreads, double* out) {
    int nodes = 0, g = 0;
    if (topology_for_workers(p, &nodes, &g) != 0) return -1;
    if (p > seq || n_q % n_kv != 0) return -1;
    const int64_t rows = b * n_q;
    const int sdt = orc_stats_dtype(dtype);
    double* pmax = (double*)malloc(sizeof(double) * (size_t)(p * rows));
    double* plse = (double*)malloc(sizeof(double) * (size_t)(p * rows));
    double* pout = (double*)malloc(sizeof(double) * (size_t)(p * rows * d));
    int rc = local_partials(q, k, v, b, n_q, n_kv, seq, d, p, scale, dtype, nthreads, pmax, plse,
                            pout);
    schedule_t s;
    if (rc == 0) rc = build_schedule(strategy, nodes, g, &s);
    if (rc != 0) {
        free(pmax);
        free(plse);
        free(pout);
        return rc;
    }
    /* allreduce(max) over lse -> shift (decode.cpp:129-139) */
    double* shift = (double*)malloc(sizeof(double) * (size_t)(p * rows));
    memcpy(shift, plse, sizeof(double) * (size_t)(p * rows));
    execute_schedule(&s, shift, rows, combine_max, NULL);
    /* partial_to_numerator per worker, fused sum-allreduce (decode.cpp:150-160) */
    const int64_t width = rows * d + rows;
    double* nd = (double*)malloc(sizeof(double) * (size_t)(p * width));
    for (int w = 0; w < p; ++w)
        orc_partial_to_numerator(plse + w * rows, pout + w * rows * d, shift, rows, d, dtype,
                                 nd + w * width, nd + w * width + rows * d);
    nd_ctx c = {rows * d, dtype, sdt};
    execute_schedule(&s, nd, width, combine_nd, &c);
    /* out = num / den (decode.cpp:165-173) */
    for (int64_t r = 0; r < rows; ++r) {
        const double den = nd[rows * d + r];
        for (int64_t j = 0; j < d; ++j) out[r * d + j] = orc_round(nd[r * d + j] / den, dtype);
    }
    sched_free(&s);
    free(shift);
    free(nd);
    free(pmax);
    free(plse);
    free(pout);
    return 0;
}

int orc_ring_decode(const double* q, const double* k, const double* v, int64_t b, int64_t n_q,
                    int64_t n_kv, int64_t seq, int64_t d, int p, double scale, int dtype,
                    int nthreads, double* out) {
    int nodes = 0, g = 0;
    if (topology_for_workers(p, &nodes, &g) != 0) return -1;
    if (p > seq || n_q % n_kv != 0) return -1;
    const int64_t rows = b * n_q;
    double* pmax = (double*)malloc(sizeof(double) * (size_t)(p * rows));
    double* plse = (double*)malloc(sizeof(double) * (size_t)(p * rows));
    double* pout = (double*)malloc(sizeof(double) * (size_t)(p * rows * d));
    int rc = local_partials(q, k, v, b, n_q, n_kv, seq, d, p, scale, dtype, nthreads, pmax, plse,
                            pout);
    if (rc == 0) {
        /* root = parts[0]; fold parts[(p-1-r) mod p] (decode.cpp:214-238) */
        double* rmax = (double*)malloc(sizeof(double) * (size_t)rows);
        double* rlse = (double*)malloc(sizeof(double) * (size_t)rows);
        double* rout = (double*)malloc(sizeof(double) * (size_t)(rows * d));
        double* tmax = (double*)malloc(sizeof(double) * (size_t)rows);
        double* tlse = (double*)malloc(sizeof(double) * (size_t)rows);
        double* tout = (double*)malloc(sizeof(double) * (size_t)(rows * d));
        memcpy(rmax, pmax, sizeof(double) * (size_t)rows);
        memcpy(rlse, plse, sizeof(double) * (size_t)rows);
        memcpy(rout, pout, sizeof(double) * (size_t)(rows * d));
        for (int r = 0; r + 1 < p && rc == 0; ++r) {
            const int inc = ((p - 1 - r) % p + p) % p;
            rc = orc_combine_pair(rmax, rlse, rout, pmax + inc * rows, plse + inc * rows,
                                  pout + inc * rows * d, rows, d, dtype, tmax, tlse, tout);
            memcpy(rmax, tmax, sizeof(double) * (size_t)rows);
            memcpy(rlse, tlse, sizeof(double) * (size_t)rows);
            memcpy(rout, tout, sizeof(double) * (size_t)(rows * d));
        }
        memcpy(out, rout, sizeof(double) * (size_t)(rows * d));
        free(rmax);
        free(rlse);
        free(rout);
        free(tmax);
        free(tlse);
        free(tout);
    }
    free(pmax);
    free(plse);
    free(pout);
    return rc;
}

/* attention_naive (attention.cpp:87-106) = chunk partial over the whole key
 * axis (row_softmax_stats is shared, so the outputs agree bitwise). */
int orc_attention_naive(const double* q, const double* k, const double* v, int64_t b,
                        int64_t n_q, int64_t n_kv, int64_t seq, int64_t d, double scale,
                        int dtype, int nthreads, double* out) {
    if (seq < 1) return -1;
    const int64_t rows = b * n_q;
    double* m = (double*)malloc(sizeof(double) * (size_t)rows);
    double* l = (double*)malloc(sizeof(double) * (size_t)rows);
    const int rc = orc_chunk_partial(q, k, v, b, n_q, n_kv, seq, 0, seq, d, scale, dtype,
                                     nthreads, m, l, out);
    free(m);
    free(l);
    return rc;
}

/* ---- energy.cpp: the energy formulation ------------------
 * Layouts: q, source [b][h][nq][d]; k, v [b][h][n][d]; per-row stats [b][h][nq];
 * grad [b][h][nq][d]. The reference requires k.extent(1) == q.extent(1): no GQA
 * (energy.cpp:15-25). */

/* energy_scores, energy.cpp:27-47: one dot per key, q.k then source.v into the
 * same accumulator, rounded to dt once. */
static void energy_scores(const double* q, const double* k, const double* v, const double* src,
                          int64_t qo, int64_t kvrow0, int64_t k0, int64_t k1, int64_t d, int dtype,
                          double* scores) {
    for (int64_t i = k0; i < k1; ++i) {
        double dot = 0.0;
        const int64_t ko = (kvrow0 + i) * d;
        for (int64_t j = 0; j < d; ++j) dot += q[qo + j] * k[ko + j];
        if (src)
            for (int64_t j = 0; j < d; ++j) dot += src[qo + j] * v[ko + j];
        scores[i - k0] = orc_round(dot, dtype);
    }
}

static void combine_max1(const double* a, const double* b, double* dst, int64_t width, const void* ctx) {
    (void)ctx;
    for (int64_t i = 0; i < width; ++i) dst[i] = a[i] > b[i] ? a[i] : b[i];
}

typedef struct {
    int sdt;
} sdt_ctx;

/* energy.cpp:189-191: round(lse_combine(a, b), sdt) */
static void combine_lse1(const double* a, const double* b, double* dst, int64_t width, const void* vctx) {
    const sdt_ctx* c = (const sdt_ctx*)vctx;
    for (int64_t i = 0; i < width; ++i) dst[i] = orc_round(orc_lse_combine(a[i], b[i]), c->sdt);
}

typedef struct {
    int dtype;
} dt_ctx;

/* energy.cpp:244-249: elementwise round(a + b, dt) */
static void combine_sum_dt(const double* a, const double* b, double* dst, int64_t width, const void* vctx) {
    const dt_ctx* c = (const dt_ctx*)vctx;
    for (int64_t i = 0; i < width; ++i) dst[i] = orc_round(a[i] + b[i], c->dtype);
}

/* tree_reduce (reduce.hpp:97-104): the reduce-only tree schedule
 * (reduce.cpp:60-66); the result is participant 0's slot. */
static void tree_reduce_slots(double* values, int participants, int64_t width, combine_fn f,
                              const void* ctx) {
    schedule_t s;
    sched_init(&s, participants);
    append_tree_reduce(&s, 0, participants, 1);
    execute_schedule(&s, values, width, f, ctx);
    sched_free(&s);
}

int orc_energy_forward_parallel(const double* q, const double* k, const double* v, const double* src,
                                int64_t b, int64_t h, int64_t nq, int64_t n, int64_t d, int chunks,
                                int dtype, double* value, double* row_max, double* shifted) {
    if (chunks < 1 || chunks > n || b < 1 || h < 1 || nq < 0 || d < 1) return -1;
    const int sdt = orc_stats_dtype(dtype);
    int64_t* ext = (int64_t*)malloc(sizeof(int64_t) * (size_t)chunks);
    orc_chunk_extents(n, chunks, ext);
    double* scores = (double*)malloc(sizeof(double) * (size_t)n);
    double* lmax = (double*)malloc(sizeof(double) * (size_t)chunks);
    double* llse = (double*)malloc(sizeof(double) * (size_t)chunks);
    sdt_ctx sc = {sdt};
    for (int64_t ib = 0; ib < b; ++ib)
        for (int64_t ih = 0; ih < h; ++ih)
            for (int64_t iq = 0; iq < nq; ++iq) {
                const int64_t r = (ib * h + ih) * nq + iq;
                const int64_t qo = r * d, kvrow0 = (ib * h + ih) * n;
                /* energy.cpp:169-180: all chunk scores, per-chunk maxima */
                energy_scores(q, k, v, src, qo, kvrow0, 0, n, d, dtype, scores);
                int64_t begin = 0;
                for (int c = 0; c < chunks; ++c) {
                    double m = NEG_INF;
                    for (int64_t a = begin; a < begin + ext[c]; ++a) m = scores[a] > m ? scores[a] : m;
                    lmax[c] = m;
                    begin += ext[c];
                }
                tree_reduce_slots(lmax, chunks, 1, combine_max1, NULL); /* :181-183 */
                const double m = lmax[0];
                begin = 0;
                for (int c = 0; c < chunks; ++c) { /* :185-193 */
                    double sum = 0.0;
                    for (int64_t a = begin; a < begin + ext[c]; ++a) {
                        scores[a] = orc_round(scores[a] - m, dtype);
                        sum += exp(scores[a]);
                    }
                    llse[c] = ext[c] == 0 ? NEG_INF : orc_round(log(sum), sdt);
                    begin += ext[c];
                }
                tree_reduce_slots(llse, chunks, 1, combine_lse1, &sc); /* :194-198 */
                row_max[r] = m;
                shifted[r] = llse[0];
                value[r] = orc_round(llse[0] + m, sdt); /* store into an sdt tensor */
            }
    free(ext);
    free(scores);
    free(lmax);
    free(llse);
    return 0;
}

int orc_energy_grad_parallel(const double* q, const double* k, const double* v, const double* row_max,
                             const double* shifted, int64_t b, int64_t h, int64_t nq, int64_t n,
                             int64_t d, int chunks, int dtype, double* grad) {
    if (chunks < 1 || chunks > n || b < 1 || h < 1 || nq < 0 || d < 1) return -1;
    const int sdt = orc_stats_dtype(dtype);
    int64_t* ext = (int64_t*)malloc(sizeof(int64_t) * (size_t)chunks);
    orc_chunk_extents(n, chunks, ext);
    double* scores = (double*)malloc(sizeof(double) * (size_t)n);
    double* acc = (double*)malloc(sizeof(double) * (size_t)(chunks * d));
    dt_ctx dc = {dtype};
    for (int64_t ib = 0; ib < b; ++ib)
        for (int64_t ih = 0; ih < h; ++ih)
            for (int64_t iq = 0; iq < nq; ++iq) {
                const int64_t r = (ib * h + ih) * nq + iq;
                const int64_t qo = r * d, kvrow0 = (ib * h + ih) * n;
                const double m = row_max[r], sh = shifted[r];
                energy_scores(q, k, v, NULL, qo, kvrow0, 0, n, d, dtype, scores);
                int64_t begin = 0;
                for (int c = 0; c < chunks; ++c) { /* energy.cpp:232-243 */
                    double* ac = acc + (size_t)c * (size_t)d;
                    for (int64_t j = 0; j < d; ++j) ac[j] = 0.0;
                    for (int64_t a = begin; a < begin + ext[c]; ++a) {
                        const double rr = orc_round(scores[a] - m, dtype);
                        const double w = orc_round(exp(rr - sh), sdt);
                        const int64_t vo = (kvrow0 + a) * d;
                        for (int64_t j = 0; j < d; ++j) ac[j] += w * v[vo + j];
                    }
                    for (int64_t j = 0; j < d; ++j) ac[j] = orc_round(ac[j], dtype);
                    begin += ext[c];
                }
                tree_reduce_slots(acc, chunks, d, combine_sum_dt, &dc); /* :244-251 */
                for (int64_t j = 0; j < d; ++j) grad[qo + j] = orc_round(acc[j], dtype);
            }
    free(ext);
    free(scores);
    free(acc);
    return 0;
}
