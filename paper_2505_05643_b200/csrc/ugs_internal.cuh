// Internal declarations shared by the libugs translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <string>
#include <vector>

#include "../../include/ugs.h"

namespace ugs {

constexpr int kTile = UGS_TILE;        // 16x16 pixel tiles
constexpr int kPrepThreads = 256;      // phase-1 block size (one Gaussian per thread)
constexpr int kSortThreads = 256;      // radix sort block size
constexpr int kSortItems = 16;         // keys per thread per sort block
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr int kPartial = 8;          // floats per backward tile-instance partial

// Per accepted (slice, Gaussian) record: two float4 = 32 B.
//   r0 = (A, B2, C, color): quadratic part of the plane-conditioned exponent
//        (log2 domain, ugs_geometry.cuh PlaneForm), pixel units
//   r1 = (bits(iu0 | iu1 << 16), bits(iv0 | iv1 << 16), alpha,
//         bits(ui | vi << 16)): inclusive pixel window and the record's
//        reference pixel (rounded in-plane centre clamped to the window)
struct Rec {
    float4 r0, r1;
};

// Per tile instance (32 B), written by the build in instance order (a
// record's instances consecutive, row-major tiles): everything the raster
// kernels need, so a tile's staging is one 32-byte gather per instance
// (cp.async, sorted id -> Frag) instead of a dependent chain through the
// record.
//   q0 = (A, B2, C, color)   the record's quadratic and colour
//   q1 = (D, E, F, bits)     the exponent re-expanded EXACTLY (float64, then
//        float32) around the instance's own expansion pixel (pu, pv) = the
//        record's reference pixel (ui, vi) clamped to the instance's clipped
//        tile rectangle:
//          log2 w = A x^2 + B2 x y + C y^2 + D x + E y + F,  x = u - pu, y = v - pv
//        so pixel offsets never exceed the tile (|x|, |y| <= 15) whatever the
//        Gaussian's extent; and the clipped rectangle + expansion pixel
//        relative to the tile origin:
//        x0 | x1 << 4 | y0 << 8 | y1 << 12 | pu << 16 | pv << 20
struct Frag {
    float4 q0, q1;
};

// Per-slice parameters of the single-pass bin sort (ugs_sort.cu).
struct SortSlice {
    int inst_base, k;        // the slice's instance segment
    int tile_base, ntile;    // its bins
    int nb, bpre;            // sort blocks of the segment, and of earlier slices
    int hoff, pad;           // offset of its (tile-major) histogram table
};

// Per-batch binning state (device pointers are owned by the plan).
struct PlanBuffers {
    // phase 1
    uint2 *blk_cnt = nullptr;       // [S][nblk] (accepted, tiles) -> exclusive offsets
    size_t blk_cnt_cap = 0;
    unsigned *blk_pairs = nullptr;  // [S][nblk] (window pixel pairs)
    size_t blk_pairs_cap = 0;
    uint32_t *amask = nullptr;      // [S][nblk*8] accept ballots of the count pass
    size_t amask_cap = 0;
    uint2 *wcnt = nullptr;          // [S][nblk*8] (accepted, tiles) per warp of Gaussians
    size_t wcnt_cap = 0;
    int32_t *warp_inst = nullptr;   // [S][nblk*8] first instance of each warp
    size_t warp_inst_cap = 0;
    int32_t *warp_rec = nullptr;    // [S][nblk*8] record index of each warp's first
    size_t warp_rec_cap = 0;        //   accepted Gaussian (emit pass)
    int32_t *rec_bucket = nullptr;  // [m/32 + 1] flattened warp holding record 32 b
    size_t rec_bucket_cap = 0;
    uint2 *win_sparse = nullptr;    // [S][n] packed windows of accepted pairs
    size_t win_sparse_cap = 0;
    unsigned long long *slice_tot = nullptr; // [S][2] totals (accepted, tiles)
    int64_t *slice_base = nullptr;  // [S][2] record base, instance base
    ugs_slice *slices = nullptr;    // [S] device copy
    int slices_cap = 0;
    // records
    Rec *rec = nullptr;             // [M]
    int32_t *rec_gid = nullptr;     // [M]
    int32_t *rec_inst = nullptr;    // [M+1] first instance of each record
    size_t rec_cap = 0, rec_gid_cap = 0, rec_inst_cap = 0;
    float *rgrad = nullptr;         // [M][12] per-record raw gradients (backward)
    size_t rgrad_cap = 0;
    double2 *bg_sums = nullptr;     // [64] per-slice background gradient sums
    // instances
    Frag *frag = nullptr;           // [K] every (unsorted) instance's raster data
    uint32_t *keys = nullptr, *vals = nullptr;     // sorted (key, instance)
    uint32_t *keys2 = nullptr, *vals2 = nullptr;   // ping-pong
    float *partial = nullptr;       // [K][8] backward per-instance partial sums
    size_t inst_cap = 0;
    // sort scratch
    uint32_t *hist = nullptr;       // [kRadix][nblk_sort]
    uint32_t *scan_tmp = nullptr;
    size_t hist_cap = 0, scan_tmp_cap = 0;
    SortSlice *sort_slices = nullptr;   // [S] device copy
    int sort_slices_cap = 0;
    // bins
    int2 *bin_range = nullptr;      // [n_bins] [start, end) into sorted arrays
    float2 *bin_bg = nullptr;       // [n_bins] per-tile (sum G, sum G*chat)
    int32_t *tile_order = nullptr;  // [S * max_tiles] raster CTA -> (slice, tile), heaviest first
    size_t tile_order_cap = 0;
    size_t bin_cap = 0;
};

}  // namespace ugs

struct ugs_plan {
    ugs::PlanBuffers b;
    int S = 0;
    int n_bins = 0;
    int64_t m_total = 0;
    int64_t k_total = 0;
    int64_t n = 0;                 // cloud size the plan was binned for
    int max_tiles = 0;
    int64_t *h_slice_base = nullptr; // host copy [S][2]
    int64_t *h_m = nullptr;          // host [S]
    // pinned staging, a ring of kRing slots so a sync-free call never
    // overwrites a slot whose copy may still be queued: slice structs (H2D)
    // and the per-slice totals + plan header (D2H), each with its event
    unsigned long long *h_plan = nullptr;   // pinned [kRing][kPlanWords]
    ugs_slice *h_slices = nullptr;          // pinned [kRing][64]
    cudaEvent_t ev_slices[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_counts[4] = {nullptr, nullptr, nullptr, nullptr};
    int slot = 0;                    // ring slot of the last ugs_bin / ugs_bin_async
    bool counts_pending = false;     // the last call's counts not yet harvested
    // capacities of the record / instance / sort-table buffers (what a
    // sync-free call may use; the device flags an overflow against them)
    int64_t m_cap = 0, k_cap = 0, hist_cap = 0, nblk_cap = 0;
    bool sized = false;              // capacities set by a synchronous ugs_bin
    int64_t m_grid = 0, k_grid = 0, nblk_grid = 0;   // launch extents of this batch
    int64_t p_total = 0;             // (Gaussian, pixel) pairs of the batch
    int32_t *h_tile_base = nullptr;  // host [S]
    int32_t *h_ntile = nullptr;      // host [S]
    int h_cap = 0;
    uint32_t *sorted_keys = nullptr; // point into b.keys/b.keys2
    uint32_t *sorted_vals = nullptr;
    bool ordered = false;            // strict per-pixel ascending-index forward
    bool slice_sort = false;         // single-pass per-slice bin sort in use
    int64_t hist_n = 0;              // its histogram table entries
    int nblk_sort = 0;               // and sort blocks
    // side stream for the background-gradient kernels, which overlap the
    // per-record finalize + update (forked and joined with events)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // optional per-stage CUDA-event timing (ugs_plan_set_timing)
    bool timing = false;
    bool ev_ready = false;
    cudaEvent_t ev[8][2];
    bool pending[8] = {false, false, false, false, false, false, false, false};
    double ms_total[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t calls[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    std::string err;
    // ugs_render_batch: the sync-free bin chain as a CUDA graph, replayed
    // while its key (plan buffers, capacities, cloud, batch shape) repeats
    cudaEvent_t ev_ofork = nullptr, ev_ojoin = nullptr;   // tile order fork / join
    cudaEvent_t ev_tot = nullptr;    // totals ready: their D2H copy goes on the side stream
    cudaGraphExec_t rgraph = nullptr;
    cudaStream_t cap = nullptr;      // capture stream (the legacy default stream cannot be)
    std::vector<unsigned long long> rgraph_key;
    long long rgraph_kernels = 0;    // kernels per replay (launch counter)
};

namespace ugs {

void set_error(const std::string &msg);

// Per-device one-time setup (function attributes, constant memory): one
// process may drive several devices, so "done" is a bit per device.  The
// setups are idempotent, so two threads racing on one device at most
// repeat one.
inline bool device_setup_done(const std::atomic<unsigned long long> &mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    return (mask.load() >> (dev & 63)) & 1ull;
}
inline void mark_device_setup(std::atomic<unsigned long long> &mask) {
    int dev = 0;
    cudaGetDevice(&dev);
    mask.fetch_or(1ull << (dev & 63));
}
int cuda_fail(cudaError_t e, const char *what);

#define UGS_CUDA(call)                                              \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return ::ugs::cuda_fail(e_, #call);  \
    } while (0)

// every kernel launch is followed by exactly one UGS_LAUNCH_CHECK, which
// also feeds the diagnostic launch counter (ugs_launch_count)
#define UGS_LAUNCH_CHECK(what)                                      \
    do {                                                            \
        ::ugs::note_launch();                                       \
        cudaError_t e_ = cudaGetLastError();                        \
        if (e_ != cudaSuccess) return ::ugs::cuda_fail(e_, what);   \
    } while (0)

void note_launch();

// Programmatic dependent launch (sm_90+): the kernels of a plan's chain are
// launched with programmatic stream serialization, so each one's CTAs can be
// scheduled while its predecessor's last wave drains (hiding the launch gap);
// every kernel starts with pdl_entry(), which waits for its prerequisite
// grids to complete (and their memory to be visible) before touching any
// memory, then lets its own dependent launch.  A kernel launched without the
// attribute passes the wait at once.
#ifndef UGS_V8
#define UGS_V8 1
#endif
#ifndef UGS_V8_BWD
#define UGS_V8_BWD 1   // the backward's partial as one 32-byte store per instance
#endif
// 32-byte global accesses as ONE instruction (sm_100 STG/LDG .256): a Frag,
// a Rec or an instance partial is one full sector per access instead of two
// half-sector requests.  The address must be 32-byte aligned (every buffer is
// its own cudaMalloc and these records are 32 B each).
__device__ __forceinline__ void st_v8(void *p, float4 a, float4 b) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p),
                 "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z),
                 "f"(b.w)
                 : "memory");
}
__device__ __forceinline__ void ld_v8(const void *p, float4 &a, float4 &b) {
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
          "=f"(b.w)
        : "l"(p));
}

__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// The two halves, for kernels with work that only reads data of EARLIER
// stages (complete before the immediate predecessor started): they trigger
// first, do that work while the predecessor drains, then wait.
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_opt(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                                  size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
#ifdef UGS_NO_PDL
    cfg.numAttrs = 0;   // experiment: plain stream-ordered launches
#else
    cfg.numAttrs = pdl ? 1 : 0;
#endif
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}
// Tuning knob: UGS_PDL_OFF="name1,name2" launches those kernels without the
// programmatic attribute (read once per process).
bool pdl_enabled(const char *kernel_name);
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
    return launch_pdl_opt(true, kernel, grid, block, smem, st, args...);
}

// launch without the programmatic attribute (a plain stream-ordered launch)
#define UGS_LAUNCH_EX(pdl, kernel, grid, block, smem, st, ...)                   \
    do {                                                                         \
        cudaError_t e_ = ::ugs::launch_pdl_opt((pdl) && ::ugs::pdl_enabled(#kernel), \
                                               kernel, dim3(grid), dim3(block),  \
                                               (size_t)(smem), st, __VA_ARGS__); \
        if (e_ != cudaSuccess) return ::ugs::cuda_fail(e_, #kernel);             \
    } while (0)

// kernel<<<grid, block, smem, st>>>(args...) as a programmatic dependent
// launch, followed by the usual launch check
#define UGS_PDL(kernel, grid, block, smem, st, ...)                              \
    do {                                                                         \
        cudaError_t e_ = ::ugs::launch_pdl_opt(::ugs::pdl_enabled(#kernel), kernel, \
                                               dim3(grid), dim3(block),          \
                                               (size_t)(smem), st, __VA_ARGS__); \
        if (e_ != cudaSuccess) return ::ugs::cuda_fail(e_, #kernel);             \
    } while (0)

enum Stage {
    kStageCount = 0,   // prepare_count + prepare_scan (+ the host read)
    kStageEmit,        // prepare_emit: records + tile instances
    kStageSort,        // radix sort
    kStageRanges,      // bin ranges
    kStageForward,     // forward_kernel
    kStageBackward,    // backward_kernel
    kStageFinalize,    // finalize_records (the bg kernels run on the side stream)
    kStageUpdate,      // update_gather (accumulate + stats + Adam)
    kNumStages
};
void stage_begin(ugs_plan *p, int stage, cudaStream_t st);
void stage_end(ugs_plan *p, int stage, cudaStream_t st);

// phase 1 (ugs_prepare.cu)
int launch_prepare_count(const ugs_cloud &c, const ugs_slice *slices, int S,
                         uint2 *blk_cnt, unsigned *blk_pairs, int nblk,
                         uint2 *win_sparse, uint32_t *amask, uint2 *wcnt, cudaStream_t st);
// per-slice bases + sort tables on the device; slice_tot holds [3*64] per-slice
// (accepted, tiles, pairs) then the plan header: 5 totals (m, k, pairs, sort
// entries, sort blocks) and the overflow flag
constexpr int kPlanWords = 3 * 64 + 8;
constexpr int kHdr = 3 * 64;
constexpr int kRing = 4;
struct PlanHdr {
    unsigned long long m, k, pairs, hist_n, nblk, ovf;
};
// ovf != 0: the batch does not fit the plan's capacities (a sync-free call);
// every later kernel of the plan returns at entry, the host grows and retries
__device__ __forceinline__ bool plan_overflow(const PlanHdr *h) {
    return h != nullptr && *(volatile const unsigned long long *)&h->ovf != 0ull;
}
inline const PlanHdr *plan_hdr(const PlanBuffers &b) {
    return reinterpret_cast<const PlanHdr *>(b.slice_tot + kHdr);
}
struct PlanCaps {
    unsigned long long m, k, hist, nblk;
};
int launch_plan_slices(unsigned long long *slice_tot, const ugs_slice *slices, int S,
                       int64_t *slice_base, SortSlice *ss, PlanCaps caps, cudaStream_t st);
int launch_prepare_scan(uint2 *blk_cnt, const unsigned *blk_pairs, int S, int nblk,
                        unsigned long long *slice_tot, cudaStream_t st);
// m_grid: records the build grid covers (the exact count after a
// synchronous plan, the capacity in a sync-free one); the kernels read the
// batch's true totals from the plan header
int launch_prepare_emit(const ugs_cloud &c, const ugs_slice *slices, int S,
                        const uint2 *blk_off, int nblk, const int64_t *slice_base,
                        Rec *rec, int32_t *rec_gid, int32_t *rec_inst,
                        Frag *frag, uint32_t *keys, const PlanHdr *hdr, int64_t m_grid,
                        const uint2 *win_sparse, const uint32_t *amask,
                        const uint2 *wcnt, int32_t *warp_rec, int32_t *warp_inst,
                        int32_t *rec_bucket, cudaStream_t st);

// radix sort (ugs_sort.cu): sorts (keys, identity values) by the low `bits`
// bits, stable.  On return *keys_out/*vals_out point at the sorted arrays
// (one of the two ping-pong buffers).
int radix_sort_pairs(uint32_t *keys, uint32_t *vals, uint32_t *keys2,
                     uint32_t *vals2, int64_t n, int bits, uint32_t *hist,
                     uint32_t *scan_tmp, cudaStream_t st, uint32_t **keys_out,
                     uint32_t **vals_out);
size_t radix_hist_entries(int64_t n);
size_t scan_tmp_entries(size_t n);
// single-pass per-slice counting sort of slice-major instances; tiles per
// slice <= 1024 (else the LSD radix sort above is used)
constexpr int kSliceSortMaxTiles = 1024;
// hist_grid / nblk_grid: table entries and sort blocks the launches cover
// (exact, or capacities); the true counts come from the plan header
// work launched between the bin ranges and the scatter (ugs_api: the raster
// CTA order, forked onto a side stream)
struct SortHook {
    int (*fn)(void *ctx, cudaStream_t st);
    void *ctx;
};
int slice_sort_bins(const uint32_t *keys, const SortSlice *d_ss, int S, const PlanHdr *hdr,
                    int64_t hist_grid, int max_tiles, int n_bins, int nblk_grid,
                    uint32_t *hist, uint32_t *scan_tmp, uint32_t *vals_out,
                    int2 *bin_range, cudaStream_t st,
                    const SortHook *after_ranges = nullptr);
int launch_bin_ranges(const uint32_t *keys, int64_t n, int2 *bin_range,
                      int n_bins, cudaStream_t st);

// raster (ugs_raster.cu)
// raster CTA order of the batch: (slice, tile) by instance count, heaviest
// first (after the bin sort; both raster kernels read it)
int launch_tile_order(const ugs_plan &p, cudaStream_t st);
int launch_forward(const ugs_plan &p, const ugs_cloud &c, const uint32_t *vals,
                   float *num, float *den, cudaStream_t st);
struct AdamArgs;   // ugs_adam.cuh
int launch_backward(const ugs_plan &p, const ugs_cloud &c, const uint32_t *vals,
                    const float *num, const float *den, const float *dpix,
                    float *grad, uint8_t *touched, float scale, const AdamArgs *adam,
                    cudaStream_t st, bool dense = false);

}  // namespace ugs
