// Multi-GPU update over peer memory: reduce-scatter of
// the AoS-12 gradient + Adam on the rank's shard + all-gather of the updated
// parameters, in ONE kernel that reads the peers' gradient rows and writes
// the peers' parameter rows directly through NVLink (CUDA IPC mappings).
//
// Every rank owns an "arena" (one cudaMalloc, exported with cudaIpcGetMemHandle)
// holding its parameter SoA, AoS-12 gradient and moments and the densify
// statistics; each process maps every peer's arena.  A training step is
//   backward -> own arena gradient        (ugs_backward, pad slot = touched)
//   barrier                               (stream-ordered collective)
//   ugs_peer_update on shard [lo, hi):    sum the W gradient rows in rank
//        order (deterministic, identical on every rank), densify statistics,
//        bit-compatible Adam on the owned rows, then store the new parameter
//        row into EVERY rank's arena; the 2 background parameters are
//        reduced and updated identically by every rank
//   barrier
// so the NCCL all-reduce of the full gradient and the replicated Adam of the
// all-reduce design are replaced by 1/W of the Adam work plus the minimum
// NVLink traffic (each gradient row is read once by its owner, each
// parameter row written once per peer).
#include <cstring>

#include "ugs_adam.cuh"

namespace ugs {
namespace {

constexpr int kMaxPeers = 8;

struct PeerViews {
    ugs_peer_view v[kMaxPeers];
};

__global__ void __launch_bounds__(256)
peer_update_kernel(PeerViews pv, int world, int rank, int64_t n, int64_t lo, int64_t hi,
                   AdamConst k, int stats) {
    const int64_t g = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const ugs_peer_view &me = pv.v[rank];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // background: every rank reduces and updates identically (replicated)
        float gb[2] = {0.f, 0.f};
        for (int q = 0; q < world; ++q) {
            gb[0] += pv.v[q].grad[kG * n];
            gb[1] += pv.v[q].grad[kG * n + 1];
        }
        adam_bg(me.bg_raw, gb, me.m + kG * n, me.v + kG * n, k);
    }
    if (g >= hi) return;
    float gr[kG];
#pragma unroll
    for (int j = 0; j < kG; ++j) gr[j] = 0.f;
    for (int q = 0; q < world; ++q) {   // rank order: the same sum on every rank
        const float4 *src = reinterpret_cast<const float4 *>(pv.v[q].grad + kG * g);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float4 a = src[c];
            gr[4 * c] += a.x;
            gr[4 * c + 1] += a.y;
            gr[4 * c + 2] += a.z;
            gr[4 * c + 3] += a.w;
        }
    }
    const bool touched = gr[11] > 0.f;   // any rank's slice accepted g
    const CloudMut p{me.means, me.l_raw, me.intensity_raw, me.opacity_raw};
    adam_gaussian(g, gr, me.m + kG * g, me.v + kG * g, p, k, touched,
                  stats ? me.grad_sum : nullptr, stats ? me.grad_cnt : nullptr);
    // all-gather: the owner writes the new row into every peer's arena
    float row[11];
#pragma unroll
    for (int c = 0; c < 3; ++c) row[c] = me.means[3 * g + c];
#pragma unroll
    for (int c = 0; c < 6; ++c) row[3 + c] = me.l_raw[6 * g + c];
    row[9] = me.intensity_raw[g];
    row[10] = me.opacity_raw[g];
    for (int q = 0; q < world; ++q) {
        if (q == rank) continue;
        const ugs_peer_view &d = pv.v[q];
#pragma unroll
        for (int c = 0; c < 3; ++c) d.means[3 * g + c] = row[c];
#pragma unroll
        for (int c = 0; c < 6; ++c) d.l_raw[6 * g + c] = row[3 + c];
        d.intensity_raw[g] = row[9];
        d.opacity_raw[g] = row[10];
    }
    // the remote (NVLink) stores are performed system-wide before the thread
    // retires, so the barrier that follows the kernel publishes them
    __threadfence_system();
}

// Before densify: the rows of m, v, grad_sum, grad_cnt this rank does not
// own are fetched from their owners, so every rank holds the full state.
__global__ void peer_gather_kernel(PeerViews pv, int world, int rank, int64_t n) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    int owner = 0;
    while (owner + 1 < world && (n * (owner + 1)) / world <= g) ++owner;
    if (owner == rank) return;
    const ugs_peer_view &src = pv.v[owner], &me = pv.v[rank];
    const float4 *ms = reinterpret_cast<const float4 *>(src.m + kG * g);
    const float4 *vs = reinterpret_cast<const float4 *>(src.v + kG * g);
    float4 *md = reinterpret_cast<float4 *>(me.m + kG * g);
    float4 *vd = reinterpret_cast<float4 *>(me.v + kG * g);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        md[c] = ms[c];
        vd[c] = vs[c];
    }
    me.grad_sum[g] = src.grad_sum[g];
    me.grad_cnt[g] = src.grad_cnt[g];
}

int load_views(const ugs_peer_view *views, int world, int rank, PeerViews &pv) {
    if (!views || world < 1 || world > kMaxPeers || rank < 0 || rank >= world) {
        set_error("peer views: need 1 <= world <= 8 and 0 <= rank < world");
        return UGS_ERR_INVALID;
    }
    std::memset(&pv, 0, sizeof(pv));
    for (int q = 0; q < world; ++q) {
        const ugs_peer_view &v = views[q];
        if (!v.means || !v.l_raw || !v.intensity_raw || !v.opacity_raw || !v.grad || !v.m ||
            !v.v || !v.grad_sum || !v.grad_cnt || !v.bg_raw) {
            set_error("peer views: NULL arena pointer");
            return UGS_ERR_INVALID;
        }
        if ((((uintptr_t)v.grad | (uintptr_t)v.m | (uintptr_t)v.v) & 15) != 0) {
            set_error("peer views: grad, m, v must be 16-byte aligned");
            return UGS_ERR_INVALID;
        }
        pv.v[q] = v;
    }
    return UGS_OK;
}

}  // namespace
}  // namespace ugs

using namespace ugs;

extern "C" int ugs_ipc_alloc(size_t bytes, void **ptr, void *handle) {
    if (!ptr || !handle || bytes == 0) {
        set_error("ugs_ipc_alloc: invalid arguments");
        return UGS_ERR_INVALID;
    }
    *ptr = nullptr;
    UGS_CUDA(cudaMalloc(ptr, bytes));
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, *ptr);
    if (e != cudaSuccess) {
        cudaFree(*ptr);
        *ptr = nullptr;
        return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    std::memcpy(handle, &h, sizeof(h));
    return UGS_OK;
}

extern "C" int ugs_ipc_open(const void *handle, void **ptr) {
    if (!handle || !ptr) {
        set_error("ugs_ipc_open: invalid arguments");
        return UGS_ERR_INVALID;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    *ptr = nullptr;
    UGS_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return UGS_OK;
}

extern "C" int ugs_ipc_close(void *ptr) {
    if (ptr) UGS_CUDA(cudaIpcCloseMemHandle(ptr));
    return UGS_OK;
}

extern "C" int ugs_ipc_free(void *ptr) {
    if (ptr) UGS_CUDA(cudaFree(ptr));
    return UGS_OK;
}

extern "C" int ugs_peer_update(const ugs_peer_view *views, int world, int rank, int64_t n,
                               int64_t lo, int64_t hi, int64_t t, const double *lr,
                               double beta1, double beta2, double eps, int stats,
                               void *stream) {
    PeerViews pv;
    int rc = load_views(views, world, rank, pv);
    if (rc) return rc;
    if (!lr || t < 1 || n < 0 || lo < 0 || hi < lo || hi > n) {
        set_error("ugs_peer_update: invalid shard / step / lr");
        return UGS_ERR_INVALID;
    }
    const AdamConst k = make_adam_const(t, lr, beta1, beta2, eps);
    const int64_t rows = hi - lo;
    const unsigned blocks = (unsigned)((rows + 255) / 256 > 0 ? (rows + 255) / 256 : 1);
    peer_update_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(pv, world, rank, n, lo, hi, k,
                                                                  stats);
    UGS_LAUNCH_CHECK("peer_update_kernel");
    return UGS_OK;
}

extern "C" int ugs_peer_gather(const ugs_peer_view *views, int world, int rank, int64_t n,
                               void *stream) {
    PeerViews pv;
    int rc = load_views(views, world, rank, pv);
    if (rc) return rc;
    if (n <= 0) return UGS_OK;
    peer_gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        pv, world, rank, n);
    UGS_LAUNCH_CHECK("peer_gather_kernel");
    return UGS_OK;
}
