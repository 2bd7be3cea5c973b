/* capi_c_demo.c -- the C-ABI (include/treedec_b200.h) from plain C, no C++ and no
 * Python: what a cgo / JNI / N-API binding would call. Built and run by
 * tests/test_gpu_capi_c.py on a GPU box.
 *
 *   capi_c_demo 1   one rank: exact decode of a seeded 1M-token cache
 *   capi_c_demo 2   two ranks (fork + pipes for the NCCL id and the CUDA IPC
 *                   handles, i.e. no launcher at all): NCCL path and one-shot
 *                   NVLink exchange, checked against a one-rank decode of the
 *                   whole cache on rank 0
 *
 * Prints "ok" and exits 0 when every check holds. */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/wait.h>
#include <unistd.h>

#include "treedec_b200.h"

enum { B = 1, NQ = 32, NKV = 8, D = 128 };
static const int64_t N = 1 << 20;

#define CHECK(call)                                                                  \
    do {                                                                             \
        int rc_ = (call);                                                            \
        if (rc_ != TD_OK) {                                                          \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, td_last_error());   \
            exit(2);                                                                 \
        }                                                                            \
    } while (0)

static void make_q(uint16_t* q) { /* seeded_random_tensor([1, 32, 128], 7, 1, bf16) */
    void* dq = NULL;
    if (cudaMalloc(&dq, sizeof(uint16_t) * B * NQ * D) != cudaSuccess) exit(3);
    CHECK(td_seeded_fill(TD_BF16, dq, 7, 1.0, B * NQ, 1, 0, 1, D, NULL));
    if (cudaMemcpy(q, dq, sizeof(uint16_t) * B * NQ * D, cudaMemcpyDeviceToHost) != cudaSuccess) exit(3);
    cudaFree(dq);
}

static double max_rel(const float* a, const float* b, int n) {
    double m = 0.0, e = 0.0;
    for (int i = 0; i < n; ++i) {
        if (!isfinite(a[i]) || !isfinite(b[i])) return INFINITY;
        if (fabs(b[i]) > m) m = fabs(b[i]);
        if (fabs(a[i] - b[i]) > e) e = fabs(a[i] - b[i]);
    }
    return m > 0 ? e / m : e;
}

static int one_rank(void) {
    td_context* ctx = NULL;
    CHECK(td_create(0, &ctx));
    CHECK(td_kv_generate(ctx, TD_BF16, B, NKV, N, D, 11, 12, 1.0));
    uint16_t q[B * NQ * D];
    float out[B * NQ * D], again[B * NQ * D];
    make_q(q);
    CHECK(td_tree_decode(ctx, q, NQ, 1.0, TD_HIERARCHICAL, out, TD_HOST_IO));
    CHECK(td_tree_decode(ctx, q, NQ, 1.0, TD_HIERARCHICAL, again, TD_HOST_IO));
    const double e = max_rel(out, again, B * NQ * D);
    printf("one rank: repeat rel diff %.3g\n", e);
    CHECK(td_destroy(ctx));
    return e <= 1e-5 ? 0 : 1;
}

static void xfer(int fd, void* p, size_t n, int writing) {
    char* c = (char*)p;
    while (n) {
        const ssize_t k = writing ? write(fd, c, n) : read(fd, c, n);
        if (k <= 0) exit(4);
        c += k;
        n -= (size_t)k;
    }
}

static int two_ranks(void) {
    int to_child[2], to_parent[2];
    if (pipe(to_child) || pipe(to_parent)) return 5;
    const pid_t pid = fork(); /* before any CUDA call */
    const int rank = pid == 0 ? 1 : 0;
    const int tx = rank == 0 ? to_child[1] : to_parent[1], rx = rank == 0 ? to_parent[0] : to_child[0];
    unsigned char id[128];
    if (rank == 0) {
        CHECK(td_comm_unique_id(id));
        xfer(tx, id, sizeof id, 1);
    } else {
        xfer(rx, id, sizeof id, 0);
    }
    td_context* ctx = NULL;
    CHECK(td_create(rank, &ctx));
    CHECK(td_comm_init(ctx, 2, rank, id));
    CHECK(td_kv_generate(ctx, TD_BF16, B, NKV, N, D, 11, 12, 1.0)); /* this rank's chunk */
    unsigned char handles[2 * 64];
    CHECK(td_p2p_handle(ctx, B * NQ, D, handles + 64 * rank));
    xfer(tx, handles + 64 * rank, 64, 1);
    xfer(rx, handles + 64 * (1 - rank), 64, 0);
    CHECK(td_p2p_open(ctx, handles));
    uint16_t q[B * NQ * D];
    float nccl[B * NQ * D], p2p[B * NQ * D];
    make_q(q);
    CHECK(td_tree_decode(ctx, q, NQ, 1.0, TD_HIERARCHICAL, nccl, TD_HOST_IO));
    CHECK(td_tree_decode(ctx, q, NQ, 1.0, TD_HIERARCHICAL, p2p, TD_HOST_IO | TD_P2P));
    int err = 0;
    CHECK(td_p2p_status(ctx, &err));
    int bad = err != 0;
    if (rank == 0) { /* the whole cache on one rank, in a second context */
        td_context* one = NULL;
        CHECK(td_create(0, &one));
        CHECK(td_kv_generate(one, TD_BF16, B, NKV, N, D, 11, 12, 1.0));
        float ref[B * NQ * D];
        CHECK(td_tree_decode(one, q, NQ, 1.0, TD_HIERARCHICAL, ref, TD_HOST_IO));
        const double e1 = max_rel(nccl, ref, B * NQ * D), e2 = max_rel(p2p, ref, B * NQ * D);
        printf("two ranks: nccl vs one rank %.3g, p2p vs one rank %.3g\n", e1, e2);
        bad |= !(e1 <= 1e-5 && e2 <= 1e-5);
        CHECK(td_destroy(one));
    }
    CHECK(td_destroy(ctx));
    if (rank == 1) exit(bad);
    int status = 0;
    waitpid(pid, &status, 0);
    return bad || !WIFEXITED(status) || WEXITSTATUS(status) != 0;
}

int main(int argc, char** argv) {
    const int ranks = argc > 1 ? atoi(argv[1]) : 1;
    printf("td_version %d\n", td_version());
    const int rc = ranks == 2 ? two_ranks() : one_rank();
    if (rc == 0) printf("ok\n");
    return rc;
}
