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
constexpr int kSyncReady = 0, kSyncDone = 8, kSyncCount = 16;
constexpr int kPeerThreads = 256;

struct PeerViews {
    ugs_peer_view v[kMaxPeers];
};

__host__ __device__ inline int64_t shard_bound(int64_t n, int world, int q) {
    if (q >= world) return n;
    const int64_t b = (n * q / world) / 32 * 32;
    return b < n ? b : n;
}

__device__ __forceinline__ unsigned ld_acquire_sys(const uint32_t *p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t *p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// bounded spin until flag >= epoch (wrap-safe); a peer that never arrives
// traps the kernel (a loud CUDA error) instead of hanging the device
__device__ void spin_until(const uint32_t *flag, uint32_t epoch) {
    const unsigned long long t0 = globaltimer();
    while ((int)(ld_acquire_sys(flag) - epoch) < 0) {
        if (globaltimer() - t0 > 20000000000ull) __trap();
        __nanosleep(256);
    }
}

__global__ void peer_signal_kernel(PeerViews pv, int world, int rank, uint32_t epoch,
                                   int slot) {
    const int q = threadIdx.x;
    if (q >= world) return;
    // this rank's writes from earlier kernels on the stream happen-before
    // this thread; the system-scope release makes them visible to peer q
    // before it can observe the flag
    __threadfence_system();
    st_release_sys(pv.v[q].sync + slot + rank, epoch);
}

__global__ void peer_wait_kernel(PeerViews pv, int world, int rank, uint32_t epoch) {
    const int q = threadIdx.x;
    if (q < world) spin_until(pv.v[rank].sync + kSyncDone + q, epoch);
}

// One thread per owned Gaussian, one warp per 32 consecutive rows (shard
// bounds are multiples of 32).
__global__ void __launch_bounds__(kPeerThreads)
peer_update_kernel(PeerViews pv, int world, int rank, int64_t n, int64_t lo, int64_t hi,
                   AdamConst k, int stats, uint32_t epoch) {
    __shared__ float4 stage[kPeerThreads / 32][88];   // a warp's 32 updated rows
    const ugs_peer_view &me = pv.v[rank];
    if (epoch) {   // every rank's gradient of this step is written
        if (threadIdx.x < world) spin_until(me.sync + kSyncReady + threadIdx.x, epoch);
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        // background: every rank reduces and updates identically (replicated)
        float gb[2] = {0.f, 0.f};
        for (int q = 0; q < world; ++q) {
            gb[0] += pv.v[q].grad[kG * n];
            gb[1] += pv.v[q].grad[kG * n + 1];
        }
        adam_bg(me.bg_raw, gb, me.m + kG * n, me.v + kG * n, k);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t g0 = lo + ((int64_t)blockIdx.x * (kPeerThreads / 32) + warp) * 32;
    const int64_t g = g0 + lane;
    if (g0 < hi) {
        float row[11];
        if (g < hi) {
            float gr[kG];
#pragma unroll
            for (int j = 0; j < kG; ++j) gr[j] = 0.f;
            for (int q = 0; q < world; ++q) {   // rank order: the same sum everywhere
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
#pragma unroll
            for (int c = 0; c < 3; ++c) row[c] = me.means[3 * g + c];
#pragma unroll
            for (int c = 0; c < 6; ++c) row[3 + c] = me.l_raw[6 * g + c];
            row[9] = me.intensity_raw[g];
            row[10] = me.opacity_raw[g];
        }
        if (g0 + 32 <= hi) {
            // all-gather of a full warp: stage the 32 rows as the arena's SoA
            // segments (means 24 | l_raw 48 | intensity 8 | opacity 8 float4)
            // and push each segment to every peer as coalesced 16-byte stores
            float *sf = reinterpret_cast<float *>(stage[warp]);
#pragma unroll
            for (int c = 0; c < 3; ++c) sf[3 * lane + c] = row[c];
#pragma unroll
            for (int c = 0; c < 6; ++c) sf[96 + 6 * lane + c] = row[3 + c];
            sf[288 + lane] = row[9];
            sf[320 + lane] = row[10];
            __syncwarp();
            for (int q = 0; q < world; ++q) {
                if (q == rank) continue;
                const ugs_peer_view &d = pv.v[q];
                float4 *dm = reinterpret_cast<float4 *>(d.means + 3 * g0);
                float4 *dl = reinterpret_cast<float4 *>(d.l_raw + 6 * g0);
                float4 *dc = reinterpret_cast<float4 *>(d.intensity_raw + g0);
                float4 *da = reinterpret_cast<float4 *>(d.opacity_raw + g0);
                if (lane < 24) dm[lane] = stage[warp][lane];
                dl[lane] = stage[warp][24 + lane];
                if (lane < 16) dl[32 + lane] = stage[warp][56 + lane];
                if (lane < 8) dc[lane] = stage[warp][72 + lane];
                else if (lane < 16) da[lane - 8] = stage[warp][80 + lane - 8];
            }
        } else if (g < hi) {   // the shard's tail (last rank only): per row
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
        }
    }
    // the remote (NVLink) stores are performed system-wide before the
    // completion signal (or the caller's barrier) publishes them
    __threadfence_system();
    if (epoch) {
        __syncthreads();
        __shared__ bool last;
        if (threadIdx.x == 0) {
            const unsigned prev = atomicAdd(me.sync + kSyncCount, 1u);
            last = prev == gridDim.x - 1;
        }
        __syncthreads();
        if (last && threadIdx.x < world) {
            if (threadIdx.x == 0) me.sync[kSyncCount] = 0u;   // next step's count
            __threadfence_system();
            st_release_sys(pv.v[threadIdx.x].sync + kSyncDone + rank, epoch);
        }
    }
}

// Before densify: the rows of m, v, grad_sum, grad_cnt this rank does not
// own are fetched from their owners, so every rank holds the full state.
__global__ void peer_gather_kernel(PeerViews pv, int world, int rank, int64_t n) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    int owner = 0;
    while (owner + 1 < world && shard_bound(n, world, owner + 1) <= g) ++owner;
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
            !v.v || !v.grad_sum || !v.grad_cnt || !v.bg_raw || !v.sync) {
            set_error("peer views: NULL arena pointer");
            return UGS_ERR_INVALID;
        }
        if ((((uintptr_t)v.grad | (uintptr_t)v.m | (uintptr_t)v.v | (uintptr_t)v.means |
              (uintptr_t)v.l_raw | (uintptr_t)v.intensity_raw | (uintptr_t)v.opacity_raw) &
             15) != 0) {
            set_error("peer views: arena arrays must be 16-byte aligned");
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

extern "C" int ugs_peer_shard(int64_t n, int world, int q, int64_t *lo, int64_t *hi) {
    if (!lo || !hi || world < 1 || q < 0 || q >= world || n < 0) {
        set_error("ugs_peer_shard: invalid arguments");
        return UGS_ERR_INVALID;
    }
    *lo = shard_bound(n, world, q);
    *hi = shard_bound(n, world, q + 1);
    return UGS_OK;
}

extern "C" int ugs_peer_update(const ugs_peer_view *views, int world, int rank, int64_t n,
                               int64_t lo, int64_t hi, int64_t t, const double *lr,
                               double beta1, double beta2, double eps, int stats,
                               uint32_t epoch, void *stream) {
    PeerViews pv;
    int rc = load_views(views, world, rank, pv);
    if (rc) return rc;
    if (!lr || t < 1 || n < 0 || lo < 0 || hi < lo || hi > n) {
        set_error("ugs_peer_update: invalid shard / step / lr");
        return UGS_ERR_INVALID;
    }
    if (lo != shard_bound(n, world, rank) || hi != shard_bound(n, world, rank + 1)) {
        set_error("ugs_peer_update: [lo, hi) must be this rank's ugs_peer_shard");
        return UGS_ERR_INVALID;
    }
    const AdamConst k = make_adam_const(t, lr, beta1, beta2, eps);
    const int64_t warps = (hi - lo + 31) / 32;
    const int64_t per = kPeerThreads / 32;
    const unsigned blocks = (unsigned)(warps > 0 ? (warps + per - 1) / per : 1);
    peer_update_kernel<<<blocks, kPeerThreads, 0, (cudaStream_t)stream>>>(pv, world, rank, n,
                                                                           lo, hi, k, stats,
                                                                           epoch);
    UGS_LAUNCH_CHECK("peer_update_kernel");
    return UGS_OK;
}

extern "C" int ugs_peer_signal(const ugs_peer_view *views, int world, int rank, uint32_t epoch,
                               void *stream) {
    PeerViews pv;
    int rc = load_views(views, world, rank, pv);
    if (rc) return rc;
    peer_signal_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(pv, world, rank, epoch, kSyncReady);
    UGS_LAUNCH_CHECK("peer_signal_kernel");
    return UGS_OK;
}

extern "C" int ugs_peer_wait(const ugs_peer_view *views, int world, int rank, uint32_t epoch,
                             void *stream) {
    PeerViews pv;
    int rc = load_views(views, world, rank, pv);
    if (rc) return rc;
    peer_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(pv, world, rank, epoch);
    UGS_LAUNCH_CHECK("peer_wait_kernel");
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
