// NCCL device API: the addresses of every rank's copy of a symmetric window.
//
// ncclCommWindowRegister(..., NCCL_WIN_COLL_SYMMETRIC) maps the ranks of one
// NVLink domain (NCCL's "LSA" team: load/store accessible) into each other's
// address space; ncclGetLsaPointer(win, offset, k) is the device-side address of
// rank k's copy. K2n (td_kernels.cu) stores into and polls those copies directly,
// so the paper-literal allreduces of decode.cpp:129-173 run inside one kernel.
// The header is NCCL's (>= 2.28); without it this unit builds a stub and the
// combine reports that it is unavailable.
#include <cuda_runtime.h>

#include "td_internal.h"

#if defined(TD_HAVE_NCCL_DEVICE)
#include <nccl.h>
#include <nccl_device.h>

namespace {
__global__ void k_lsa_peers(ncclWindow_t win, int p, void** ptrs, int* ok) {
    for (int k = threadIdx.x; k < p; k += blockDim.x) ptrs[k] = ncclGetLsaPointer(win, 0, k);
    if (threadIdx.x == 0) *ok = win->lsaRank == win->worldRank ? 1 : 0;
}
}  // namespace

namespace td {
cudaError_t launch_lsa_peers(void* win, int p, void** ptrs, int* ok, cudaStream_t stream) {
    k_lsa_peers<<<1, 32, 0, stream>>>(static_cast<ncclWindow_t>(win), p, ptrs, ok);
    return cudaGetLastError();
}
}  // namespace td
#else
namespace td {
cudaError_t launch_lsa_peers(void*, int, void**, int*, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace td
#endif
