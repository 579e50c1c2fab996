// C ABI entry points (include/ugs.h): plan lifetime, batch binning, forward,
// backward, exports.  Error reporting: negative ugs_status + thread-local
// message (ugs_last_error), the reference raises InvalidParameterError at
// its API layer for the same conditions (gradients.py:43-52).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <vector>

#include "ugs_adam.cuh"
#include "ugs_internal.cuh"

namespace ugs {

static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

bool pdl_enabled(const char *kernel_name) {
    static const std::string off = [] {
        const char *e = getenv("UGS_PDL_OFF");
        return e ? "," + std::string(e) + "," : std::string();
    }();
    if (off.empty()) return true;
    return off.find("," + std::string(kernel_name) + ",") == std::string::npos;
}

static void harvest(ugs_plan *p, int stage) {
    if (!p->pending[stage]) return;
    float ms = 0.f;
    if (cudaEventSynchronize(p->ev[stage][1]) == cudaSuccess &&
        cudaEventElapsedTime(&ms, p->ev[stage][0], p->ev[stage][1]) == cudaSuccess) {
        p->ms_total[stage] += ms;
        p->calls[stage] += 1;
    }
    p->pending[stage] = false;
}

void stage_begin(ugs_plan *p, int stage, cudaStream_t st) {
    if (!p->timing) return;
    if (!p->ev_ready) {
        for (int i = 0; i < kNumStages; ++i)
            for (int j = 0; j < 2; ++j) cudaEventCreate(&p->ev[i][j]);
        p->ev_ready = true;
    }
    harvest(p, stage);
    cudaEventRecord(p->ev[stage][0], st);
}

void stage_end(ugs_plan *p, int stage, cudaStream_t st) {
    if (!p->timing || !p->ev_ready) return;
    cudaEventRecord(p->ev[stage][1], st);
    p->pending[stage] = true;
}

void set_error(const std::string &msg) { g_err = msg; }

int cuda_fail(cudaError_t e, const char *what) {
    g_err = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? UGS_ERR_OOM : UGS_ERR_CUDA;
}

namespace {

// Capacity for `need` elements: 25 % headroom (counts drift per batch), and
// when a buffer outgrows its capacity at least double it -- footprints
// that grow during training (time to SSIM: ~9x in the first steps) then
// cost a handful of re-allocations and re-issued batches, not one per step.
inline size_t grow_cap(size_t need, size_t old_cap) {
    const size_t a = need + need / 4 + 64;
    return old_cap && 2 * old_cap > a ? 2 * old_cap : a;
}

template <typename T>
int ensure(T **ptr, size_t *cap, size_t need, const char *what) {
    if (need <= *cap && *ptr) return UGS_OK;
    const size_t alloc = grow_cap(need, *ptr ? *cap : 0);
    if (*ptr) {
        cudaError_t e = cudaFree(*ptr);
        *ptr = nullptr;
        *cap = 0;
        if (e != cudaSuccess) return cuda_fail(e, what);
    }
    cudaError_t e = cudaMalloc((void **)ptr, alloc * sizeof(T));
    if (e != cudaSuccess) {
        *ptr = nullptr;
        return cuda_fail(e, what);
    }
    *cap = alloc;
    return UGS_OK;
}

int ensure_host(ugs_plan *p, int S) {
    if (!p->h_plan) {
        cudaError_t e = cudaMallocHost((void **)&p->h_plan,
                                       sizeof(unsigned long long) * kPlanWords * kRing);
        if (e != cudaSuccess) { p->h_plan = nullptr; return cuda_fail(e, "alloc h_plan"); }
        e = cudaMallocHost((void **)&p->h_slices, sizeof(ugs_slice) * 64 * kRing);
        if (e != cudaSuccess) { p->h_slices = nullptr; return cuda_fail(e, "alloc h_slices"); }
        for (int i = 0; i < kRing; ++i) {
            UGS_CUDA(cudaEventCreateWithFlags(&p->ev_slices[i], cudaEventDisableTiming));
            UGS_CUDA(cudaEventCreateWithFlags(&p->ev_counts[i], cudaEventDisableTiming));
        }
    }
    if (S <= p->h_cap) return UGS_OK;
    delete[] p->h_slice_base;
    delete[] p->h_m;
    delete[] p->h_tile_base;
    delete[] p->h_ntile;
    p->h_slice_base = new int64_t[2 * S];
    p->h_m = new int64_t[S];
    p->h_tile_base = new int32_t[S];
    p->h_ntile = new int32_t[S];
    p->h_cap = S;
    return UGS_OK;
}

int check_cloud(const ugs_cloud *c) {
    if (!c) { set_error("cloud is NULL"); return UGS_ERR_INVALID; }
    if (!(c->beta > 0)) { set_error("beta must be > 0"); return UGS_ERR_INVALID; }
    if (c->n < 0 || c->n > 0x7fffffffLL) {
        set_error("cloud size out of range (0 <= n < 2^31)");
        return UGS_ERR_RANGE;
    }
    if (c->n > 0 && (!c->means || !c->l_raw || !c->intensity_raw || !c->opacity_raw)) {
        set_error("cloud has NULL parameter arrays");
        return UGS_ERR_INVALID;
    }
    if (!c->bg_raw) { set_error("cloud bg_raw is NULL"); return UGS_ERR_INVALID; }
    return UGS_OK;
}

int bits_for(int64_t n) {
    int b = 0;
    while (((int64_t)1 << b) < n) ++b;
    return b;
}

}  // namespace
}  // namespace ugs

using namespace ugs;

extern "C" const char *ugs_last_error(void) { return g_err.c_str(); }

extern "C" int ugs_abi_version(void) { return UGS_ABI_VERSION; }

extern "C" int ugs_plan_create(ugs_plan **out) {
    if (!out) { set_error("ugs_plan_create: out is NULL"); return UGS_ERR_INVALID; }
    *out = new ugs_plan();
    return UGS_OK;
}

extern "C" int ugs_plan_destroy(ugs_plan *p) {
    if (!p) return UGS_OK;
    PlanBuffers &b = p->b;
    void *bufs[] = {b.blk_cnt, b.blk_pairs, b.amask, b.wcnt, b.warp_rec, b.warp_inst, b.rec_bucket, b.win_sparse, b.slice_tot,
                    b.slice_base, b.slices, b.rec,
                    b.rec_gid, b.rec_inst, b.frag, b.keys, b.vals, b.keys2,
                    b.vals2, b.partial, b.rgrad, b.bg_sums, b.tile_order,
                    b.hist,
                    b.scan_tmp, b.sort_slices, b.bin_range,
                    b.bin_bg};
    for (void *q : bufs)
        if (q) cudaFree(q);
    if (p->ev_ofork) cudaEventDestroy(p->ev_ofork);
    if (p->ev_tot) cudaEventDestroy(p->ev_tot);
    if (p->ev_ojoin) cudaEventDestroy(p->ev_ojoin);
    if (p->rgraph) cudaGraphExecDestroy(p->rgraph);
    if (p->cap) cudaStreamDestroy(p->cap);
    delete[] p->h_slice_base;
    delete[] p->h_m;
    delete[] p->h_tile_base;
    delete[] p->h_ntile;
    if (p->h_plan) cudaFreeHost(p->h_plan);
    for (int i = 0; i < kRing; ++i) {
        if (p->ev_slices[i]) cudaEventDestroy(p->ev_slices[i]);
        if (p->ev_counts[i]) cudaEventDestroy(p->ev_counts[i]);
    }
    if (p->h_slices) cudaFreeHost(p->h_slices);
    if (p->ev_ready)
        for (int i = 0; i < kNumStages; ++i)
            for (int j = 0; j < 2; ++j) cudaEventDestroy(p->ev[i][j]);
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    if (p->side) cudaStreamDestroy(p->side);
    delete p;
    return UGS_OK;
}

namespace ugs {
namespace {

constexpr int64_t kHistCapMax = ((int64_t)1 << 24) - 1;   // one exclusive_scan

PlanCaps caps_of(const ugs_plan *p) {
    return PlanCaps{(unsigned long long)p->m_cap, (unsigned long long)p->k_cap,
                    (unsigned long long)p->hist_cap, (unsigned long long)p->nblk_cap};
}

// Record / instance / sort-table buffers for m records and k instances (with
// the headroom of ensure(): counts drift from batch to batch); the plan's
// capacities are what later sync-free calls may use.
int grow_to(ugs_plan *p, int64_t m_need, int64_t k_need, int max_tiles, int S) {
    PlanBuffers &b = p->b;
    int rc;
    if ((rc = ensure(&b.rec, &b.rec_cap, (size_t)m_need + 1, "alloc rec"))) return rc;
    if ((rc = ensure(&b.rec_gid, &b.rec_gid_cap, (size_t)m_need + 2, "alloc rec_gid")))
        return rc;
    if ((rc = ensure(&b.rec_inst, &b.rec_inst_cap, (size_t)m_need + 2, "alloc rec_inst")))
        return rc;
    if ((rc = ensure(&b.rgrad, &b.rgrad_cap, 12 * ((size_t)m_need + 1), "alloc rgrad")))
        return rc;
    if ((rc = ensure(&b.rec_bucket, &b.rec_bucket_cap, (size_t)m_need / 32 + 2,
                     "alloc rec_bucket")))
        return rc;
    const size_t kneed = (size_t)k_need + 1;
    if (kneed > b.inst_cap || !b.frag) {
        const size_t old_cap = b.frag ? b.inst_cap : 0;
        // all-or-nothing: every pointer is nulled when freed and the capacity
        // is published only after every allocation succeeded, so a failed
        // (OOM) grow leaves no dangling pointer and no stale capacity
        void **bufs[] = {(void **)&b.frag, (void **)&b.keys, (void **)&b.vals,
                         (void **)&b.keys2, (void **)&b.vals2, (void **)&b.partial};
        const size_t elem[] = {sizeof(Frag), sizeof(uint32_t), sizeof(uint32_t),
                               sizeof(uint32_t), sizeof(uint32_t), sizeof(float) * kPartial};
        for (void **q : bufs) {
            if (*q) cudaFree(*q);
            *q = nullptr;
        }
        b.inst_cap = 0;
        const size_t cap = grow_cap(kneed, old_cap);
        for (int i = 0; i < 6; ++i) {
            cudaError_t e = cudaMalloc(bufs[i], elem[i] * cap);
            if (e != cudaSuccess) {
                for (void **q : bufs) {
                    if (*q) cudaFree(*q);
                    *q = nullptr;
                }
                return cuda_fail(e, "alloc tile instances");
            }
        }
        b.inst_cap = cap;
    }
    // capacities (each buffer's own, minus its +1/+2 sentinels)
    int64_t mc = (int64_t)b.rec_cap - 1;
    mc = std::min(mc, (int64_t)b.rec_gid_cap - 2);
    mc = std::min(mc, (int64_t)b.rec_inst_cap - 2);
    mc = std::min(mc, (int64_t)(b.rgrad_cap / 12) - 1);
    mc = std::min(mc, ((int64_t)b.rec_bucket_cap - 2) * 32);
    const int64_t kc = (int64_t)b.inst_cap - 1;
    // sort tables: blocks <= k/kSortTile + S, entries <= tiles x blocks
    const int64_t nb_cap = kc / kSortTile + S + 1;
    int64_t hcap = std::min((int64_t)std::max(max_tiles, 1) * nb_cap, kHistCapMax);
    const size_t hn = std::max((size_t)hcap, radix_hist_entries(kc)) + 1;
    if ((rc = ensure(&b.hist, &b.hist_cap, hn, "alloc hist"))) return rc;
    if ((rc = ensure(&b.scan_tmp, &b.scan_tmp_cap, scan_tmp_entries(hn) + 1, "alloc scan_tmp")))
        return rc;
    p->m_cap = mc;
    p->k_cap = kc;
    p->hist_cap = hcap;
    p->nblk_cap = nb_cap;
    return UGS_OK;
}

// Harvests the counts of the last call (waits on its D2H event only).
void read_counts(ugs_plan *p, int S, int64_t *m_out, int64_t *k_out, int64_t *p_out) {
    const unsigned long long *tot = p->h_plan + (size_t)p->slot * kPlanWords;
    const unsigned long long *tt = tot + kHdr;
    for (int s = 0; s < S; ++s) {
        if (m_out) m_out[s] = (int64_t)tot[3 * s];
        if (k_out) k_out[s] = (int64_t)tot[3 * s + 1];
        if (p_out) p_out[s] = (int64_t)tot[3 * s + 2];
    }
    p->m_total = (int64_t)tt[0];
    p->k_total = (int64_t)tt[1];
    p->p_total = (int64_t)tt[2];
    p->hist_n = (int64_t)tt[3];
    p->nblk_sort = (int)tt[4];
}

// ugs_bin / ugs_bin_async.  Synchronous: the per-slice totals come back to
// the host before the record / instance buffers are sized, so the launches
// are exact.  Sync-free (after one synchronous call sized the plan): the
// launches cover the plan's capacities, the device compares the batch's
// totals against them (plan_slices) and, if the batch does not fit, every
// later kernel of the plan returns at entry; ugs_plan_poll reports it.
struct BinPrep {
    int nblk = 0, max_tiles = 0, n_bins = 0, slot = 0;
    unsigned long long *hp = nullptr;   // this call's pinned totals slot
};

// The raster CTA order of the batch, forked onto the plan's side stream
// between the bin ranges and the scatter (it needs only the ranges): it runs
// while the scatter does; bin_join_order makes the stream wait for it.
int order_hook(void *ctx, cudaStream_t st) {
    ugs_plan *p = static_cast<ugs_plan *>(ctx);
    if (!p->side) UGS_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
    if (!p->ev_ofork) {
        UGS_CUDA(cudaEventCreateWithFlags(&p->ev_ofork, cudaEventDisableTiming));
        UGS_CUDA(cudaEventCreateWithFlags(&p->ev_ojoin, cudaEventDisableTiming));
    }
    UGS_CUDA(cudaEventRecord(p->ev_ofork, st));
    UGS_CUDA(cudaStreamWaitEvent(p->side, p->ev_ofork, 0));
    int rc = launch_tile_order(*p, p->side);
    if (rc) return rc;
    UGS_CUDA(cudaEventRecord(p->ev_ojoin, p->side));
    return UGS_OK;
}

int bin_join_order(ugs_plan *p, cudaStream_t st) {
    UGS_CUDA(cudaStreamWaitEvent(st, p->ev_ojoin, 0));
    return UGS_OK;
}

// Host side of a bin call: validation, tile layout, buffers, the ring slot
// and the slice constants' H2D copy.  `async` is cleared when the call must
// be synchronous (unsized plan, radix fallback).
int bin_prepare(ugs_plan *p, const ugs_cloud *c, ugs_slice *slices, int S, cudaStream_t st,
                bool &async, BinPrep &bp) {
    if (!p || !slices || S < 1 || S > 64) {
        set_error("ugs_bin: need a plan and 1 <= S <= 64 slices");
        return UGS_ERR_INVALID;
    }
    int rc = check_cloud(c);
    if (rc) return rc;
    PlanBuffers &b = p->b;
    // tiles and bin ids
    int tile_base = 0, max_tiles = 0;
    for (int s = 0; s < S; ++s) {
        ugs_slice &sl = slices[s];
        if (sl.width < 1 || sl.height < 1 || sl.width > 32767 || sl.height > 32767 ||
            !(sl.s > 0)) {
            set_error("ugs_bin: slice width/height must be in [1, 32767], spacing > 0");
            return UGS_ERR_INVALID;
        }
        sl.tiles_x = (sl.width + kTile - 1) / kTile;
        sl.tiles_y = (sl.height + kTile - 1) / kTile;
        sl.tile_base = tile_base;
        const int nt = sl.tiles_x * sl.tiles_y;
        tile_base += nt;
        if (nt > max_tiles) max_tiles = nt;
    }
    const int n_bins = tile_base;
    // sync-free only on a sized plan and with the single-pass bin sort
    // (the LSD radix fallback for > 1024 tiles per slice sizes its passes
    // on the host)
    if (async && (!p->sized || max_tiles > kSliceSortMaxTiles)) async = false;
    if ((rc = ensure_host(p, S))) return rc;
    p->S = S;
    p->n_bins = n_bins;
    p->max_tiles = max_tiles;
    p->n = c->n;
    for (int s = 0; s < S; ++s) {
        p->h_tile_base[s] = slices[s].tile_base;
        p->h_ntile[s] = slices[s].tiles_x * slices[s].tiles_y;
    }
    size_t cap_sl = (size_t)b.slices_cap;
    if ((rc = ensure(&b.slices, &cap_sl, (size_t)S, "alloc slices"))) return rc;
    b.slices_cap = (int)cap_sl;
    const int nblk = (int)((c->n + kPrepThreads - 1) / kPrepThreads);
    if ((int64_t)S * nblk * (kPrepThreads / 32) >= 0x7fffffffLL) {
        // the flattened (slice, warp) index of the record search is 32-bit
        set_error("ugs_bin: slices x Gaussians exceeds the 2^36 plan budget; use fewer slices");
        return UGS_ERR_RANGE;
    }
    const size_t nb1 = (size_t)S * (nblk > 0 ? nblk : 1);
    if ((rc = ensure(&b.blk_cnt, &b.blk_cnt_cap, nb1, "alloc blk_cnt"))) return rc;
    if ((rc = ensure(&b.blk_pairs, &b.blk_pairs_cap, nb1, "alloc blk_pairs"))) return rc;
    // accept bits per (slice, warp) and the windows of accepted pairs,
    // written by the count pass and read back by the emit pass
    const size_t nw1 = nb1 * (kPrepThreads / 32);
    if ((rc = ensure(&b.amask, &b.amask_cap, nw1, "alloc amask"))) return rc;
    if ((rc = ensure(&b.wcnt, &b.wcnt_cap, nw1, "alloc wcnt"))) return rc;
    if ((rc = ensure(&b.warp_inst, &b.warp_inst_cap, nw1, "alloc warp_inst"))) return rc;
    if ((rc = ensure(&b.warp_rec, &b.warp_rec_cap, nw1, "alloc warp_rec"))) return rc;
    if ((rc = ensure(&b.win_sparse, &b.win_sparse_cap, (size_t)S * (c->n > 0 ? c->n : 1),
                     "alloc win_sparse")))
        return rc;
    {
        static_assert(sizeof(unsigned long long) == 8, "");
        size_t cap = b.slice_tot ? (size_t)kPlanWords : 0;
        if ((rc = ensure(&b.slice_tot, &cap, (size_t)kPlanWords, "alloc slice_tot"))) return rc;
        size_t cap2 = b.slice_base ? 128 : 0;
        if ((rc = ensure(&b.slice_base, &cap2, (size_t)128, "alloc slice_base"))) return rc;
        size_t cap3 = (size_t)b.sort_slices_cap;
        if ((rc = ensure(&b.sort_slices, &cap3, (size_t)64, "alloc sort_slices"))) return rc;
        b.sort_slices_cap = (int)cap3;
        size_t cap4 = b.bg_sums ? 64 : 0;
        if ((rc = ensure(&b.bg_sums, &cap4, (size_t)64, "alloc bg_sums"))) return rc;
    }
    if (b.bin_cap < (size_t)n_bins || !b.bin_range) {
        if (b.bin_range) cudaFree(b.bin_range);
        if (b.bin_bg) cudaFree(b.bin_bg);
        b.bin_range = nullptr;
        b.bin_bg = nullptr;
        b.bin_cap = 0;
        const size_t cap = (size_t)n_bins + 64;
        cudaError_t e = cudaMalloc(&b.bin_range, sizeof(int2) * cap);
        if (e == cudaSuccess) e = cudaMalloc(&b.bin_bg, sizeof(float2) * cap);
        if (e != cudaSuccess) {
            if (b.bin_range) cudaFree(b.bin_range);
            b.bin_range = nullptr;
            b.bin_bg = nullptr;
            return cuda_fail(e, "alloc bins");
        }
        b.bin_cap = cap;
    }
    if ((rc = ensure(&b.tile_order, &b.tile_order_cap, (size_t)S * max_tiles,
                     "alloc tile_order")))
        return rc;
    // the next ring slot: its previous copies (kRing calls ago) are done
    p->slot = (p->slot + 1) % kRing;
    const int slot = p->slot;
    UGS_CUDA(cudaEventSynchronize(p->ev_slices[slot]));
    UGS_CUDA(cudaEventSynchronize(p->ev_counts[slot]));
    ugs_slice *hs = p->h_slices + (size_t)slot * 64;
    unsigned long long *hp = p->h_plan + (size_t)slot * kPlanWords;
    // through pinned staging: an async DMA (a pageable copy would block the
    // host until the stream drains)
    std::memcpy(hs, slices, sizeof(ugs_slice) * S);
    UGS_CUDA(cudaMemcpyAsync(b.slices, hs, sizeof(ugs_slice) * S, cudaMemcpyHostToDevice, st));
    UGS_CUDA(cudaEventRecord(p->ev_slices[slot], st));
    bp.nblk = nblk;
    bp.max_tiles = max_tiles;
    bp.n_bins = n_bins;
    bp.slot = slot;
    bp.hp = hp;
    return UGS_OK;
}

// The sync-free kernel chain of a bin call (count -> scan -> plan -> emit ->
// bin sort) over the plan's capacities; the device flags a batch that does
// not fit and every later kernel of the plan returns at entry.
int bin_async_chain(ugs_plan *p, const ugs_cloud *c, int S, const BinPrep &bp,
                    cudaStream_t st) {
    PlanBuffers &b = p->b;
    int rc;
    const int nblk = bp.nblk, max_tiles = bp.max_tiles, n_bins = bp.n_bins;
    stage_begin(p, kStageCount, st);
    if (c->n > 0) {
        if ((rc = launch_prepare_count(*c, b.slices, S, b.blk_cnt, b.blk_pairs, nblk,
                                       b.win_sparse, b.amask, b.wcnt, st)))
            return rc;
        if ((rc = launch_prepare_scan(b.blk_cnt, b.blk_pairs, S, nblk, b.slice_tot, st)))
            return rc;
    } else {
        UGS_CUDA(cudaMemsetAsync(b.slice_tot, 0, sizeof(unsigned long long) * 3 * S, st));
    }
    if ((rc = launch_plan_slices(b.slice_tot, b.slices, S, b.slice_base, b.sort_slices,
                                 caps_of(p), st)))
        return rc;
    stage_end(p, kStageCount, st);
    p->counts_pending = true;
    p->slice_sort = true;
    p->m_grid = p->m_cap;
    p->k_grid = p->k_cap;
    p->nblk_grid = p->nblk_cap;
    const PlanHdr *hdr = plan_hdr(b);
    stage_begin(p, kStageEmit, st);
    if (c->n > 0) {
        if ((rc = launch_prepare_emit(*c, b.slices, S, b.blk_cnt, nblk, b.slice_base,
                                      b.rec, b.rec_gid, b.rec_inst, b.frag, b.keys, hdr,
                                      p->m_grid, b.win_sparse, b.amask, b.wcnt, b.warp_rec,
                                      b.warp_inst, b.rec_bucket, st)))
            return rc;
    } else {
        // an empty cloud: no records, rec_inst[0] = 0 (the buffer may not
        // exist yet -- a plan that never needed records)
        if ((rc = ensure(&b.rec_inst, &b.rec_inst_cap, (size_t)2, "alloc rec_inst"))) return rc;
        UGS_CUDA(cudaMemsetAsync(b.rec_inst, 0, sizeof(int32_t), st));
    }
    stage_end(p, kStageEmit, st);
    stage_begin(p, kStageSort, st);
    const SortHook hook{order_hook, p};
    if ((rc = slice_sort_bins(b.keys, b.sort_slices, S, hdr, p->hist_cap, max_tiles, n_bins,
                              (int)p->nblk_grid, b.hist, b.scan_tmp, b.vals, b.bin_range, st,
                              &hook)))
        return rc;
    if ((rc = bin_join_order(p, st))) return rc;
    p->sorted_keys = nullptr;
    p->sorted_vals = b.vals;
    stage_end(p, kStageSort, st);
    return UGS_OK;
}

// the totals of a sync-free call to its pinned slot (read by ugs_plan_poll),
// copied on the plan's side stream: the launch stream goes straight on to
// the forward (no copy between the sort and it)
int bin_async_totals(ugs_plan *p, const BinPrep &bp, cudaStream_t st) {
    if (!p->side) UGS_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking));
    if (!p->ev_tot) UGS_CUDA(cudaEventCreateWithFlags(&p->ev_tot, cudaEventDisableTiming));
    UGS_CUDA(cudaEventRecord(p->ev_tot, st));
    UGS_CUDA(cudaStreamWaitEvent(p->side, p->ev_tot, 0));
    UGS_CUDA(cudaMemcpyAsync(bp.hp, p->b.slice_tot, sizeof(unsigned long long) * kPlanWords,
                             cudaMemcpyDeviceToHost, p->side));
    UGS_CUDA(cudaEventRecord(p->ev_counts[bp.slot], p->side));
    return UGS_OK;
}

// The synchronous remainder of a bin call: count, read the totals back, size
// the buffers, then emit and sort exactly.
int bin_sync_rest(ugs_plan *p, const ugs_cloud *c, int S, const BinPrep &bp, cudaStream_t st,
                  int64_t *m_out, int64_t *k_out, int64_t *p_out) {
    int rc;
    PlanBuffers &b = p->b;
    const int nblk = bp.nblk, max_tiles = bp.max_tiles, n_bins = bp.n_bins, slot = bp.slot;
    unsigned long long *hp = bp.hp;
    stage_begin(p, kStageCount, st);
    if (c->n > 0) {
        if ((rc = launch_prepare_count(*c, b.slices, S, b.blk_cnt, b.blk_pairs, nblk,
                                       b.win_sparse, b.amask, b.wcnt, st)))
            return rc;
        if ((rc = launch_prepare_scan(b.blk_cnt, b.blk_pairs, S, nblk, b.slice_tot, st)))
            return rc;
    } else {
        UGS_CUDA(cudaMemsetAsync(b.slice_tot, 0, sizeof(unsigned long long) * 3 * S, st));
    }
    // bases, sort tables and the overflow flag on the device; the totals go
    // to pinned memory now: a synchronous call sizes its buffers from them
    // (the sync-free chain copies them after the sort instead, so its
    // kernels stay back to back -- programmatic dependent launches overlap
    // consecutive kernels only)
    if ((rc = launch_plan_slices(b.slice_tot, b.slices, S, b.slice_base, b.sort_slices,
                                 caps_of(p), st)))
        return rc;
    UGS_CUDA(cudaMemcpyAsync(hp, b.slice_tot, sizeof(unsigned long long) * kPlanWords,
                             cudaMemcpyDeviceToHost, st));
    UGS_CUDA(cudaEventRecord(p->ev_counts[slot], st));
    stage_end(p, kStageCount, st);
    p->counts_pending = true;
    {
        UGS_CUDA(cudaEventSynchronize(p->ev_counts[slot]));
        read_counts(p, S, m_out, k_out, p_out);
        p->counts_pending = false;
        if (p->k_total >= 0x7fffffffLL || p->m_total >= 0x7fffffffLL) {
            set_error("ugs_bin: batch exceeds 2^31 tile instances; use fewer slices");
            return UGS_ERR_RANGE;
        }
        p->slice_sort = max_tiles <= kSliceSortMaxTiles && p->hist_n < kHistCapMax;
        const bool fits = p->m_total <= p->m_cap && p->k_total <= p->k_cap &&
                          (!p->slice_sort || (p->hist_n <= p->hist_cap &&
                                              p->nblk_sort <= p->nblk_cap));
        if (!fits && (rc = grow_to(p, p->m_total, p->k_total, max_tiles, S))) return rc;
        if (hp[kHdr + 5] != 0ull) {
            // re-derive the device flag against the new capacities (the
            // radix fallback sizes its sort tables here, not from the caps)
            PlanCaps caps = caps_of(p);
            if (!p->slice_sort) caps.hist = caps.nblk = ~0ull;
            if ((rc = launch_plan_slices(b.slice_tot, b.slices, S, b.slice_base,
                                         b.sort_slices, caps, st)))
                return rc;
        }
        p->sized = true;
        p->m_grid = p->m_total;
        p->k_grid = p->k_total;
        p->nblk_grid = p->nblk_sort;
    }
    const PlanHdr *hdr = plan_hdr(b);
    stage_begin(p, kStageEmit, st);
    if (c->n > 0) {
        if ((rc = launch_prepare_emit(*c, b.slices, S, b.blk_cnt, nblk, b.slice_base,
                                      b.rec, b.rec_gid, b.rec_inst, b.frag, b.keys, hdr,
                                      p->m_grid, b.win_sparse, b.amask, b.wcnt, b.warp_rec,
                                      b.warp_inst, b.rec_bucket, st)))
            return rc;
    } else {
        // an empty cloud: no records, rec_inst[0] = 0 (the buffer may not
        // exist yet -- a plan that never needed records)
        if ((rc = ensure(&b.rec_inst, &b.rec_inst_cap, (size_t)2, "alloc rec_inst"))) return rc;
        UGS_CUDA(cudaMemsetAsync(b.rec_inst, 0, sizeof(int32_t), st));
    }
    stage_end(p, kStageEmit, st);
    stage_begin(p, kStageSort, st);
    if (p->slice_sort) {
        const SortHook hook{order_hook, p};
        if ((rc = slice_sort_bins(b.keys, b.sort_slices, S, hdr, p->hist_n, max_tiles, n_bins,
                                  (int)p->nblk_grid, b.hist, b.scan_tmp, b.vals,
                                  b.bin_range, st, &hook)))
            return rc;
        if ((rc = bin_join_order(p, st))) return rc;
        p->sorted_keys = nullptr;
        p->sorted_vals = b.vals;
        stage_end(p, kStageSort, st);
        return UGS_OK;
    } else {
        if ((rc = radix_sort_pairs(b.keys, b.vals, b.keys2, b.vals2, p->k_total,
                                   bits_for(n_bins), b.hist, b.scan_tmp, st,
                                   &p->sorted_keys, &p->sorted_vals)))
            return rc;
        stage_end(p, kStageSort, st);
        stage_begin(p, kStageRanges, st);
        if ((rc = launch_bin_ranges(p->sorted_keys, p->k_total, b.bin_range, n_bins, st)))
            return rc;
        stage_end(p, kStageRanges, st);
    }
    return launch_tile_order(*p, st);   // the radix path: after its ranges
}

int bin_impl(ugs_plan *p, const ugs_cloud *c, ugs_slice *slices, int S, cudaStream_t st,
             bool async, int64_t *m_out, int64_t *k_out, int64_t *p_out) {
    BinPrep bp;
    int rc = bin_prepare(p, c, slices, S, st, async, bp);
    if (rc) return rc;
    if (async) {
        if ((rc = bin_async_chain(p, c, S, bp, st))) return rc;
        return bin_async_totals(p, bp, st);
    }
    return bin_sync_rest(p, c, S, bp, st, m_out, k_out, p_out);
}

// The key of ugs_render_batch's graph: everything its kernels' arguments and
// launch extents are made of (buffer addresses, capacities, cloud, batch
// shape); a different key re-captures.
std::vector<unsigned long long> render_graph_key(const ugs_plan *p, const ugs_cloud *c, int S,
                                                 const BinPrep &bp) {
    const PlanBuffers &b = p->b;
    auto u = [](const void *q) { return (unsigned long long)(uintptr_t)q; };
    double beta = c->beta;
    unsigned long long beta_bits;
    std::memcpy(&beta_bits, &beta, sizeof(beta_bits));
    return {u(b.blk_cnt), u(b.blk_pairs), u(b.amask), u(b.wcnt), u(b.warp_rec),
            u(b.warp_inst), u(b.rec_bucket), u(b.win_sparse), u(b.slice_tot),
            u(b.slice_base), u(b.slices), u(b.rec), u(b.rec_gid), u(b.rec_inst),
            u(b.frag), u(b.keys), u(b.vals), u(b.hist), u(b.scan_tmp),
            u(b.sort_slices), u(b.bin_range), u(b.tile_order),
            u(c->means), u(c->l_raw), u(c->intensity_raw), u(c->opacity_raw),
            u(c->bg_raw), (unsigned long long)c->n, beta_bits,
            (unsigned long long)S, (unsigned long long)bp.nblk,
            (unsigned long long)bp.max_tiles, (unsigned long long)bp.n_bins,
            (unsigned long long)p->m_cap, (unsigned long long)p->k_cap,
            (unsigned long long)p->hist_cap, (unsigned long long)p->nblk_cap};
}

}  // namespace
}  // namespace ugs

extern "C" int ugs_bin(ugs_plan *p, const ugs_cloud *c, ugs_slice *slices,
                       int S, void *stream, int64_t *m_out, int64_t *k_out,
                       int64_t *p_out) {
    return bin_impl(p, c, slices, S, (cudaStream_t)stream, false, m_out, k_out, p_out);
}

extern "C" int ugs_bin_async(ugs_plan *p, const ugs_cloud *c, ugs_slice *slices, int S,
                             void *stream) {
    return bin_impl(p, c, slices, S, (cudaStream_t)stream, true, nullptr, nullptr, nullptr);
}

extern "C" int ugs_plan_poll(ugs_plan *p, int *overflowed, int64_t *m_out, int64_t *k_out,
                             int64_t *p_out) {
    if (!p) { set_error("ugs_plan_poll: NULL plan"); return UGS_ERR_INVALID; }
    if (overflowed) *overflowed = 0;
    if (!p->h_plan || p->S == 0) return UGS_OK;
    UGS_CUDA(cudaEventSynchronize(p->ev_counts[p->slot]));
    const unsigned long long *hp = p->h_plan + (size_t)p->slot * kPlanWords;
    const bool ovf = hp[kHdr + 5] != 0ull;
    read_counts(p, p->S, m_out, k_out, p_out);
    if (p->counts_pending && ovf) {
        if (p->k_total >= 0x7fffffffLL || p->m_total >= 0x7fffffffLL) {
            set_error("ugs_bin_async: batch exceeds 2^31 tile instances; use fewer slices");
            return UGS_ERR_RANGE;
        }
        // the batch's kernels were no-ops: grow so that a retry fits
        int rc = grow_to(p, p->m_total, p->k_total, p->max_tiles, p->S);
        if (rc) return rc;
        if (overflowed) *overflowed = 1;
    }
    p->counts_pending = false;
    return UGS_OK;
}

extern "C" int ugs_forward(ugs_plan *p, const ugs_cloud *c, float *num,
                           float *den, void *stream) {
    if (!p || !num || !den) { set_error("ugs_forward: NULL argument"); return UGS_ERR_INVALID; }
    int rc = check_cloud(c);
    if (rc) return rc;
    if (c->n != p->n) {
        set_error("ugs_forward: cloud size differs from the binned cloud");
        return UGS_ERR_INVALID;
    }
    return launch_forward(*p, *c, p->sorted_vals, num, den, (cudaStream_t)stream);
}

extern "C" int ugs_render(ugs_plan *p, const ugs_cloud *c, float *pixels, void *stream) {
    if (!p || !pixels) { set_error("ugs_render: NULL argument"); return UGS_ERR_INVALID; }
    int rc = check_cloud(c);
    if (rc) return rc;
    if (c->n != p->n) {
        set_error("ugs_render: cloud size differs from the binned cloud");
        return UGS_ERR_INVALID;
    }
    if (p->ordered) {
        set_error("ugs_render: the strict-order forward has no render mode");
        return UGS_ERR_INVALID;
    }
    return launch_forward(*p, *c, p->sorted_vals, pixels, nullptr, (cudaStream_t)stream);
}

extern "C" int ugs_render_batch(ugs_plan *p, const ugs_cloud *c, ugs_slice *slices, int S,
                                float *pixels, void *stream) {
    if (!p || !pixels) { set_error("ugs_render_batch: NULL argument"); return UGS_ERR_INVALID; }
    int rc = check_cloud(c);
    if (rc) return rc;
    if (p->ordered) {
        set_error("ugs_render_batch: the strict-order forward has no render mode");
        return UGS_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    bool async = true;
    BinPrep bp;
    if ((rc = bin_prepare(p, c, slices, S, st, async, bp))) return rc;
    if (!async) {   // unsized plan / radix fallback: the synchronous bin
        if ((rc = bin_sync_rest(p, c, S, bp, st, nullptr, nullptr, nullptr))) return rc;
        return launch_forward(*p, *c, p->sorted_vals, pixels, nullptr, st);
    }
    if (p->timing || c->n == 0) {   // per-stage events / empty cloud: plain launches
        if ((rc = bin_async_chain(p, c, S, bp, st))) return rc;
        if ((rc = launch_forward(*p, *c, p->sorted_vals, pixels, nullptr, st))) return rc;
        return bin_async_totals(p, bp, st);
    }
    // the graph is the bin chain (count -> ... -> sort); the totals' copy
    // and the render follow it as plain stream work, so ugs_plan_poll can
    // return while the forward runs (and the output pointer is free)
    std::vector<unsigned long long> key = render_graph_key(p, c, S, bp);
    if (!p->rgraph || key != p->rgraph_key) {
        if (p->rgraph) {
            cudaGraphExecDestroy(p->rgraph);
            p->rgraph = nullptr;
        }
        if (!p->cap) UGS_CUDA(cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking));
        const long long l0 = g_launches.load();
        UGS_CUDA(cudaStreamBeginCapture(p->cap, cudaStreamCaptureModeThreadLocal));
        rc = bin_async_chain(p, c, S, bp, p->cap);
        cudaGraph_t g = nullptr;
        const cudaError_t ec = cudaStreamEndCapture(p->cap, &g);
        if (!rc && ec != cudaSuccess) rc = cuda_fail(ec, "ugs_render_batch capture");
        if (!rc) {
            const cudaError_t ei = cudaGraphInstantiate(&p->rgraph, g, 0);
            if (ei != cudaSuccess) {
                p->rgraph = nullptr;
                rc = cuda_fail(ei, "ugs_render_batch instantiate");
            }
        }
        if (g) cudaGraphDestroy(g);
        if (rc) return rc;
        p->rgraph_key = key;
        p->rgraph_kernels = g_launches.load() - l0;
    } else {
        // host state the captured chain sets
        p->counts_pending = true;
        p->slice_sort = true;
        p->m_grid = p->m_cap;
        p->k_grid = p->k_cap;
        p->nblk_grid = p->nblk_cap;
        p->sorted_keys = nullptr;
        p->sorted_vals = p->b.vals;
        g_launches.fetch_add(p->rgraph_kernels, std::memory_order_relaxed);
    }
    UGS_CUDA(cudaGraphLaunch(p->rgraph, st));
    if ((rc = bin_async_totals(p, bp, st))) return rc;
    return launch_forward(*p, *c, p->sorted_vals, pixels, nullptr, st);
}

extern "C" int ugs_backward(ugs_plan *p, const ugs_cloud *c, const float *num,
                            const float *den, const float *d_pixels, float *grad,
                            uint8_t *touched, float scale, void *stream) {
    if (!p || !num || !den || !d_pixels || !grad) {
        set_error("ugs_backward: NULL argument");
        return UGS_ERR_INVALID;
    }
    int rc = check_cloud(c);
    if (rc) return rc;
    if (c->n != p->n) {
        set_error("ugs_backward: buffers do not match this cloud");
        return UGS_ERR_INVALID;
    }
    return launch_backward(*p, *c, p->sorted_vals, num, den, d_pixels, grad, touched,
                           scale, nullptr, (cudaStream_t)stream);
}

extern "C" int ugs_backward_dense(ugs_plan *p, const ugs_cloud *c, const float *num,
                                  const float *den, const float *d_pixels, float *grad,
                                  float scale, void *stream) {
    if (!p || !num || !den || !d_pixels || !grad) {
        set_error("ugs_backward_dense: NULL argument");
        return UGS_ERR_INVALID;
    }
    int rc = check_cloud(c);
    if (rc) return rc;
    if (c->n != p->n) {
        set_error("ugs_backward_dense: buffers do not match this cloud");
        return UGS_ERR_INVALID;
    }
    if (((uintptr_t)grad & 15) != 0) {
        set_error("ugs_backward_dense: grad must be 16-byte aligned");
        return UGS_ERR_INVALID;
    }
    return launch_backward(*p, *c, p->sorted_vals, num, den, d_pixels, grad, nullptr, scale,
                           nullptr, (cudaStream_t)stream, true);
}

extern "C" int ugs_backward_adam(ugs_plan *p, const ugs_cloud *c, const float *num,
                                 const float *den, const float *d_pixels, float scale,
                                 float *m, float *v, int64_t t, const double *lr,
                                 double beta1, double beta2, double eps,
                                 float *grad_sum, int32_t *grad_cnt, void *stream) {
    if (!p || !num || !den || !d_pixels || !m || !v || !lr || t < 1) {
        set_error("ugs_backward_adam: invalid arguments");
        return UGS_ERR_INVALID;
    }
    if ((grad_sum == nullptr) != (grad_cnt == nullptr)) {
        set_error("ugs_backward_adam: grad_sum and grad_cnt go together");
        return UGS_ERR_INVALID;
    }
    int rc = check_cloud(c);
    if (rc) return rc;
    if (c->n != p->n) {
        set_error("ugs_backward_adam: buffers do not match this cloud");
        return UGS_ERR_INVALID;
    }
    if ((((uintptr_t)m | (uintptr_t)v) & 15) != 0) {
        set_error("ugs_backward_adam: m, v must be 16-byte aligned");
        return UGS_ERR_INVALID;
    }
    AdamArgs a{m, v, make_adam_const(t, lr, beta1, beta2, eps), grad_sum, grad_cnt};
    return launch_backward(*p, *c, p->sorted_vals, num, den, d_pixels, nullptr, nullptr,
                           scale, &a, (cudaStream_t)stream);
}

namespace ugs {
namespace {
__global__ void export_accepted_kernel(const Rec *__restrict__ rec,
                                       const int32_t *__restrict__ gid, int64_t m,
                                       int32_t *__restrict__ acc,
                                       int32_t *__restrict__ win) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    if (acc) acc[r] = gid[r];
    if (win) {
        const int wu = __float_as_int(rec[r].r1.x), wv = __float_as_int(rec[r].r1.y);
        win[4 * r + 0] = wu & 0xffff;
        win[4 * r + 1] = wu >> 16;
        win[4 * r + 2] = wv & 0xffff;
        win[4 * r + 3] = wv >> 16;
    }
}

__global__ void export_sorted_kernel(const uint32_t *__restrict__ vals,
                                     const int32_t *__restrict__ rec_inst, int64_t m,
                                     const int32_t *__restrict__ gid, int64_t k,
                                     int32_t *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    // the instance's record: the last r with rec_inst[r] <= instance
    const int32_t inst = (int32_t)vals[i];
    int64_t lo = 0, hi = m - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (rec_inst[mid] <= inst) lo = mid; else hi = mid - 1;
    }
    out[i] = gid[lo];
}
}  // namespace
}  // namespace ugs

extern "C" int ugs_export_accepted(const ugs_plan *p, int32_t *accepted,
                                   int32_t *windows, void *stream) {
    if (!p) { set_error("ugs_export_accepted: NULL plan"); return UGS_ERR_INVALID; }
    if (p->m_total == 0) return UGS_OK;
    const int th = 256;
    export_accepted_kernel<<<(unsigned)((p->m_total + th - 1) / th), th, 0,
                             (cudaStream_t)stream>>>(p->b.rec, p->b.rec_gid,
                                                     p->m_total, accepted, windows);
    UGS_LAUNCH_CHECK("export_accepted_kernel");
    return UGS_OK;
}

extern "C" int ugs_export_bins(const ugs_plan *p, int32_t *bin_range,
                               int32_t *sorted_gauss, int32_t *n_bins_out,
                               int64_t *k_total_out, void *stream) {
    if (!p) { set_error("ugs_export_bins: NULL plan"); return UGS_ERR_INVALID; }
    if (n_bins_out) *n_bins_out = p->n_bins;
    if (k_total_out) *k_total_out = p->k_total;
    cudaStream_t st = (cudaStream_t)stream;
    if (bin_range && p->n_bins > 0)
        UGS_CUDA(cudaMemcpyAsync(bin_range, p->b.bin_range, sizeof(int2) * p->n_bins,
                                 cudaMemcpyDeviceToDevice, st));
    if (sorted_gauss && p->k_total > 0) {
        const int th = 256;
        export_sorted_kernel<<<(unsigned)((p->k_total + th - 1) / th), th, 0, st>>>(
            p->sorted_vals, p->b.rec_inst, p->m_total, p->b.rec_gid, p->k_total, sorted_gauss);
        UGS_LAUNCH_CHECK("export_sorted_kernel");
    }
    return UGS_OK;
}

extern "C" long long ugs_launch_count(void) { return g_launches.load(); }

// Host: the batch's ugs_slice constants from float64 poses, with the
// reference's own operation order (ProbePose.inverse geometry.py:61-64,
// plane_axes :107-120, the window bounds rasterizer.py:126-135), every
// product and sum rounded separately (this translation unit's host code is
// not contracted to FMA), then cast to float32 -- byte-identical to the
// numpy fill_slice / fill_slices (tests/test_capi_cpu.py), without numpy's
// per-call overhead on the serving path.
extern "C" int ugs_fill_slices(const double *rot, const double *trans, const double *spacing,
                               const int32_t *width, const int32_t *height, int S, double cut,
                               ugs_slice *out) {
    if (S < 0 || (S > 0 && (!rot || !trans || !spacing || !width || !height || !out)) ||
        !(cut > 0.0)) {
        set_error("ugs_fill_slices: invalid arguments");
        return UGS_ERR_INVALID;
    }
    const float sqrt_cut = std::sqrt((float)cut);
    int64_t pix = 0;
    for (int s = 0; s < S; ++s) {
        const double *R = rot + 9 * s, *t = trans + 3 * s;
        const double sp = spacing[s];
        const int W = width[s], H = height[s];
        ugs_slice &o = out[s];
        std::memset(&o, 0, sizeof(o));
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) o.rw[3 * i + j] = (float)R[3 * j + i];   // R^T
        for (int i = 0; i < 3; ++i) {
            // -(R^T t)_i, the inner product in order
            volatile double acc = R[0 + i] * t[0];
            acc = acc + R[3 + i] * t[1];
            acc = acc + R[6 + i] * t[2];
            o.tw[i] = (float)(-acc);
        }
        const double cxw = (double)(W - 1) / 2.0, cyh = (double)(H - 1) / 2.0;
        for (int k = 0; k < 3; ++k) {
            const double du = R[3 * k + 0] * sp, dv = R[3 * k + 1] * sp;
            volatile double a = cxw * du;
            volatile double b = cyh * dv;
            volatile double org = t[k] - a;
            org = org - b;
            o.origin[k] = (float)org;
            o.du[k] = (float)du;
            o.dv[k] = (float)dv;
        }
        o.sqrt_cut = sqrt_cut;
        o.s = (float)sp;
        o.cx = (float)cxw;
        o.cy = (float)cyh;
        o.x1h = (float)(cxw * sp);
        o.x2h = (float)(cyh * sp);
        o.width = W;
        o.height = H;
        o.pix_base = pix;
        pix += (int64_t)W * H;
    }
    return UGS_OK;
}

extern "C" int ugs_plan_set_ordered(ugs_plan *p, int ordered) {
    if (!p) { set_error("ugs_plan_set_ordered: NULL plan"); return UGS_ERR_INVALID; }
    p->ordered = ordered != 0;
    return UGS_OK;
}

extern "C" int ugs_plan_set_timing(ugs_plan *p, int enabled) {
    if (!p) { set_error("ugs_plan_set_timing: NULL plan"); return UGS_ERR_INVALID; }
    p->timing = enabled != 0;
    return UGS_OK;
}

extern "C" int ugs_plan_timings(ugs_plan *p, double *ms_total, int64_t *calls,
                                int n, int reset) {
    if (!p) { set_error("ugs_plan_timings: NULL plan"); return UGS_ERR_INVALID; }
    for (int s = 0; s < kNumStages; ++s) harvest(p, s);
    for (int s = 0; s < n && s < kNumStages; ++s) {
        if (ms_total) ms_total[s] = p->ms_total[s];
        if (calls) calls[s] = p->calls[s];
    }
    if (reset)
        for (int s = 0; s < kNumStages; ++s) { p->ms_total[s] = 0; p->calls[s] = 0; }
    return kNumStages;
}
