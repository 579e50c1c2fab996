// Hand-written stable LSD radix sort of (slice, tile) bin keys with the
// original instance index as payload, plus the bin-range scan.
//
// The instance array is produced in ascending (slice, Gaussian, tile) order,
// so a STABLE sort by bin key yields per-(slice, tile) lists in ascending
// Gaussian index -- exactly the accumulation order of the reference's
// sequential forward loop (ref _kernels.py:23) -- and the tile assignment is
// bit-exact by construction.
//
// Per 8-bit digit pass: histogram (smem atomics, order-free) -> exclusive
// scan of the digit-major [256][nblk] table -> scatter with a stable in-block
// rank (warp match.any + per-warp running digit counters).
#include "ugs_internal.cuh"

namespace ugs {

namespace {

// ---------------------------------------------------------------- scan ----
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t x,
                                                         uint32_t *total) {
    __shared__ uint32_t ws[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    __syncthreads();
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t a = lane < nw ? ws[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t t = __shfl_up_sync(0xffffffffu, a, o);
            if (lane >= o) a += t;
        }
        ws[lane] = a;
    }
    __syncthreads();
    uint32_t pre = (warp ? ws[warp - 1] : 0u) + inc - x;
    if (total) *total = ws[nw - 1];
    return pre;
}

// n_dev (optional): the true entry count on the device, clamped to the
// launch extent n (a sync-free plan sizes the grid by capacity)
__device__ __forceinline__ size_t scan_count(size_t n, const unsigned long long *n_dev) {
    return n_dev ? (size_t)min((unsigned long long)n, *n_dev) : n;
}

__global__ void __launch_bounds__(kScanThreads)
scan_reduce_kernel(const uint32_t *__restrict__ in, size_t n,
                   const unsigned long long *__restrict__ n_dev,
                   uint32_t *__restrict__ sums) {
    pdl_entry();
    n = scan_count(n, n_dev);
    const size_t base = (size_t)blockIdx.x * kScanTile;
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        size_t i = base + (size_t)j * kScanThreads + threadIdx.x;
        if (i < n) acc += in[i];
    }
    acc = __reduce_add_sync(0xffffffffu, acc);
    __shared__ uint32_t ws[kScanThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kScanThreads / 32; ++w) t += ws[w];
        sums[blockIdx.x] = t;
    }
}

// single block, exclusive scan of up to 1024*8 entries in place
__global__ void __launch_bounds__(1024)
scan_sums_kernel(uint32_t *__restrict__ sums, int n) {
    pdl_entry();
    uint32_t v[8];
    const int base = threadIdx.x * 8;
    uint32_t local = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        v[j] = (base + j < n) ? sums[base + j] : 0u;
        local += v[j];
    }
    uint32_t pre = block_exclusive_scan(local, nullptr);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        if (base + j < n) sums[base + j] = pre;
        pre += v[j];
    }
}

__global__ void __launch_bounds__(kScanThreads)
scan_down_kernel(const uint32_t *__restrict__ in, uint32_t *__restrict__ out,
                 size_t n, const unsigned long long *__restrict__ n_dev,
                 const uint32_t *__restrict__ sums) {
    pdl_entry();
    n = scan_count(n, n_dev);
    // each thread scans kScanItems consecutive entries (blocked layout)
    __shared__ uint32_t tile[kScanTile];
    const size_t base = (size_t)blockIdx.x * kScanTile;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        size_t i = base + (size_t)j * kScanThreads + threadIdx.x;
        tile[j * kScanThreads + threadIdx.x] = i < n ? in[i] : 0u;
    }
    __syncthreads();
    uint32_t v[kScanItems], local = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        v[j] = tile[threadIdx.x * kScanItems + j];
        local += v[j];
    }
    uint32_t pre = block_exclusive_scan(local, nullptr) + sums[blockIdx.x];
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        tile[threadIdx.x * kScanItems + j] = pre;
        pre += v[j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        size_t i = base + (size_t)j * kScanThreads + threadIdx.x;
        if (i < n) out[i] = tile[j * kScanThreads + threadIdx.x];
    }
}

// Exclusive scan in place or out of place.  Up to 8192 tiles of block sums
// are scanned by one block; larger inputs scan their block sums recursively
// (tmp holds every level: scan_tmp_entries()).
int exclusive_scan(const uint32_t *in, uint32_t *out, size_t n,
                   uint32_t *tmp, cudaStream_t st,
                   const unsigned long long *n_dev = nullptr) {
    if (n == 0) return UGS_OK;
    const size_t nb = (n + kScanTile - 1) / kScanTile;
    UGS_PDL(scan_reduce_kernel, (unsigned)nb, kScanThreads, 0, st,
        in, n, n_dev, tmp);
    UGS_LAUNCH_CHECK("scan_reduce_kernel");
    if (nb > 8192) {
        int rc = exclusive_scan(tmp, tmp, nb, tmp + nb, st);
        if (rc) return rc;
    } else {
        UGS_PDL(scan_sums_kernel, 1, 1024, 0, st,
        tmp, (int)nb);
        UGS_LAUNCH_CHECK("scan_sums_kernel");
    }
    UGS_PDL(scan_down_kernel, (unsigned)nb, kScanThreads, 0, st,
        in, out, n, n_dev, tmp);
    UGS_LAUNCH_CHECK("scan_down_kernel");
    return UGS_OK;
}

// ---------------------------------------------------------- radix sort ----
__global__ void __launch_bounds__(kSortThreads)
radix_hist_kernel(const uint32_t *__restrict__ keys, int64_t n, int shift,
                  uint32_t *__restrict__ hist, int nblk) {
    pdl_entry();
    __shared__ uint32_t h[kRadix];
    for (int i = threadIdx.x; i < kRadix; i += kSortThreads) h[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSortTile;
#pragma unroll 4
    for (int j = 0; j < kSortItems; ++j) {
        int64_t i = base + (int64_t)j * kSortThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(__ldg(keys + i) >> shift) & (kRadix - 1)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kSortThreads)
        hist[(size_t)d * nblk + blockIdx.x] = h[d];
}

__global__ void __launch_bounds__(kSortThreads)
radix_scatter_kernel(const uint32_t *__restrict__ keys_in,
                     const uint32_t *__restrict__ vals_in,  // null: identity
                     uint32_t *__restrict__ keys_out,
                     uint32_t *__restrict__ vals_out, int64_t n, int shift,
                     const uint32_t *__restrict__ offs, int nblk) {
    pdl_entry();
    constexpr int kWarps = kSortThreads / 32;
    constexpr int kPerWarp = kSortItems * 32;
    __shared__ uint32_t wcnt[kWarps][kRadix];
    __shared__ uint32_t gofs[kRadix];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kSortThreads)
        (&wcnt[0][0])[i] = 0;
    for (int d = threadIdx.x; d < kRadix; d += kSortThreads)
        gofs[d] = offs[(size_t)d * nblk + blockIdx.x];
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)warp * kPerWarp;
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t k[kSortItems], v[kSortItems], dr[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const int64_t i = base + j * 32 + lane;
        const bool ok = i < n;
        k[j] = ok ? keys_in[i] : 0u;
        v[j] = ok ? (vals_in ? vals_in[i] : (uint32_t)i) : 0u;
        const uint32_t d = ok ? ((k[j] >> shift) & (kRadix - 1)) : (uint32_t)kRadix;
        // lanes with the same digit: 9 ballots (8 digit bits + the invalid
        // flag) -- constant cost, unlike match.any on many distinct values
        unsigned peers = 0xffffffffu;
#pragma unroll
        for (int bit = 0; bit <= kRadixBits; ++bit) {
            const unsigned bal = __ballot_sync(0xffffffffu, (d >> bit) & 1u);
            peers &= ((d >> bit) & 1u) ? bal : ~bal;
        }
        const uint32_t rank = __popc(peers & lt_mask);
        uint32_t cnt_before = 0;
        if (ok) cnt_before = wcnt[warp][d];
        __syncwarp();
        if (ok && rank == 0) wcnt[warp][d] = cnt_before + __popc(peers);
        __syncwarp();
        dr[j] = ok ? ((d << 16) | (cnt_before + rank)) : 0xffffffffu;
    }
    __syncthreads();
    // exclusive prefix of the per-warp digit counts across warps
    for (int d = threadIdx.x; d < kRadix; d += kSortThreads) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            uint32_t t = wcnt[w][d];
            wcnt[w][d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        if (dr[j] == 0xffffffffu) continue;
        const uint32_t d = dr[j] >> 16, r = dr[j] & 0xffffu;
        const uint32_t pos = gofs[d] + wcnt[warp][d] + r;
        keys_out[pos] = k[j];
        vals_out[pos] = v[j];
    }
}

// ------------------------------------------- single-pass slice bin sort ----
// The instances of a batch are emitted slice-major (records in slice order),
// so a stable sort by (slice, tile) only has to sort each slice's segment by
// its tile id.  One counting pass per segment does it: per-block tile
// histograms (tile-major, block-minor table per slice), one exclusive scan of
// the concatenated tables -- whose entries are then the global output
// positions -- and a stable scatter of the instance ids.  Half the traffic
// and a third of the launches of the two-pass LSD sort, and the per-tile
// ranges fall out of the scan.

// The slice of sort block b: the block stages the slices' first-block
// indices in shared memory (one parallel load) and binary-searches them,
// instead of a chain of dependent global loads per block.
__device__ __forceinline__ int sort_slice_of(const SortSlice *__restrict__ ss, int S, int b) {
    __shared__ int s_bpre[64];
    for (int q = threadIdx.x; q < S; q += blockDim.x) s_bpre[q] = ss[q].bpre;
    __syncthreads();
    int s = 0;
#pragma unroll
    for (int step = 32; step > 0; step >>= 1)   // last slice whose bpre <= b
        if (s + step < S && s_bpre[s + step] <= b) s += step;
    return s;
}

__global__ void __launch_bounds__(kSortThreads)
slice_hist_kernel(const uint32_t *__restrict__ keys, const SortSlice *__restrict__ ss, int S,
                  const PlanHdr *__restrict__ hdr, uint32_t *__restrict__ hist) {
    pdl_entry();
    extern __shared__ uint32_t sh[];
    if (plan_overflow(hdr) || blockIdx.x >= hdr->nblk) return;   // whole block
    const int s = sort_slice_of(ss, S, blockIdx.x);
    const SortSlice q = ss[s];
    const int lb = blockIdx.x - q.bpre;
    for (int t = threadIdx.x; t < q.ntile; t += kSortThreads) sh[t] = 0;
    __syncthreads();
    const int start = q.inst_base + lb * kSortTile;
    const int end = min(start + kSortTile, q.inst_base + q.k);
    // all of a thread's key loads are in flight before the first atomic
    uint32_t d[kSortItems];
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const int i = start + j * kSortThreads + threadIdx.x;
        d[j] = i < end ? __ldg(keys + i) - (uint32_t)q.tile_base : 0xffffffffu;
    }
#pragma unroll
    for (int j = 0; j < kSortItems; ++j)
        if (d[j] != 0xffffffffu) atomicAdd(&sh[d[j]], 1u);
    __syncthreads();
    for (int t = threadIdx.x; t < q.ntile; t += kSortThreads)
        hist[(size_t)q.hoff + (size_t)t * q.nb + lb] = sh[t];
}

template <int kBits>
#ifndef UGS_SCATTER_STAGE
#define UGS_SCATTER_STAGE 1
#endif
#ifndef UGS_SCATTER_MINB
#define UGS_SCATTER_MINB (UGS_SCATTER_STAGE ? 5 : 6)
#endif
__global__ void __launch_bounds__(kSortThreads, UGS_SCATTER_MINB)
slice_scatter_kernel(const uint32_t *__restrict__ keys, const SortSlice *__restrict__ ss,
                     int S, const PlanHdr *__restrict__ hdr, const uint32_t *__restrict__ offs,
                     uint32_t *__restrict__ vals_out) {
    pdl_entry();
    constexpr int kWarpsS = kSortThreads / 32;
    constexpr int kPerWarp = kSortItems * 32;
    constexpr int kT = 1 << kBits;
    extern __shared__ uint32_t wcnt[];   // [kWarpsS][kT]
    if (plan_overflow(hdr) || blockIdx.x >= hdr->nblk) return;   // whole block
    const int s = sort_slice_of(ss, S, blockIdx.x);
    const SortSlice q = ss[s];
    const int lb = blockIdx.x - q.bpre;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kWarpsS * kT; i += kSortThreads) wcnt[i] = 0;
    __syncthreads();
    const int start = q.inst_base + lb * kSortTile + warp * kPerWarp;
    const int end = min(q.inst_base + lb * kSortTile + kSortTile, q.inst_base + q.k);
    const unsigned lt_mask = (1u << lane) - 1u;
    uint32_t dr[kSortItems];
    uint32_t *my = wcnt + warp * kT;
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        const int i = start + j * 32 + lane;
        const bool ok = i < end;
        const uint32_t d = ok ? __ldg(keys + i) - (uint32_t)q.tile_base : (uint32_t)kT;
        // lanes with the same tile: kBits + 1 ballots (tile bits + invalid)
        unsigned peers = 0xffffffffu;
#pragma unroll
        for (int bit = 0; bit <= kBits; ++bit) {
            const unsigned bal = __ballot_sync(0xffffffffu, (d >> bit) & 1u);
            peers &= ((d >> bit) & 1u) ? bal : ~bal;
        }
        const uint32_t rank = __popc(peers & lt_mask);
        uint32_t before = 0;
        if (ok) before = my[d];
        __syncwarp();
        if (ok && rank == 0) my[d] = before + __popc(peers);
        __syncwarp();
        dr[j] = ok ? ((d << 16) | (before + rank)) : 0xffffffffu;
    }
    __syncthreads();
#if UGS_SCATTER_STAGE
    // the block's ids are staged in shared memory in output order (tile,
    // then rank), each with its destination, and written out by consecutive
    // threads: a tile's run of the block (~16 ids) becomes one coalesced
    // store instead of ~16 scattered 4-byte ones
    __shared__ uint32_t s_val[kSortTile], s_dst[kSortTile];
    __shared__ uint32_t s_gbase[kT], s_lbase[kT], s_wsum[kWarpsS];
    constexpr int TPT = (kT + kSortThreads - 1) / kSortThreads;   // tiles per thread
    uint32_t tot[TPT], sum = 0u;
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
        const int d = threadIdx.x * TPT + k;
        uint32_t run = 0u;
        if (d < q.ntile) {
            s_gbase[d] = __ldg(offs + (size_t)q.hoff + (size_t)d * q.nb + lb);
#pragma unroll
            for (int w = 0; w < kWarpsS; ++w) {   // within-tile prefix over warps
                const uint32_t t = wcnt[w * kT + d];
                wcnt[w * kT + d] = run;
                run += t;
            }
        }
        tot[k] = run;
        sum += run;
    }
    // block-wide exclusive scan of the per-thread tile sums (tile order)
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_wsum[warp] = incl;
    __syncthreads();
    uint32_t base = incl - sum;
    for (int w = 0; w < warp; ++w) base += s_wsum[w];
#pragma unroll
    for (int k = 0; k < TPT; ++k) {
        const int d = threadIdx.x * TPT + k;
        if (d < q.ntile) {
            s_lbase[d] = base;
#pragma unroll
            for (int w = 0; w < kWarpsS; ++w) wcnt[w * kT + d] += base;
        }
        base += tot[k];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        if (dr[j] == 0xffffffffu) continue;
        const uint32_t d = dr[j] >> 16, r = dr[j] & 0xffffu;
        const uint32_t loc = my[d] + r;
        s_val[loc] = (uint32_t)(start + j * 32 + lane);
        s_dst[loc] = s_gbase[d] + (loc - s_lbase[d]);
    }
    __syncthreads();
    const int nloc = end - (q.inst_base + lb * kSortTile);
    for (int i = threadIdx.x; i < nloc; i += kSortThreads) vals_out[s_dst[i]] = s_val[i];
#else
    // per tile: this block's global offset (scanned histogram, one load per
    // tile) plus the exclusive prefix of the per-warp counts across warps
    for (int d = threadIdx.x; d < q.ntile; d += kSortThreads) {
        uint32_t run = __ldg(offs + (size_t)q.hoff + (size_t)d * q.nb + lb);
#pragma unroll
        for (int w = 0; w < kWarpsS; ++w) {
            const uint32_t t = wcnt[w * kT + d];
            wcnt[w * kT + d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kSortItems; ++j) {
        if (dr[j] == 0xffffffffu) continue;
        const uint32_t d = dr[j] >> 16, r = dr[j] & 0xffffu;
        vals_out[my[d] + r] = (uint32_t)(start + j * 32 + lane);
    }
#endif
}

// Per-(slice, tile) [start, end) straight from the scanned tables.
__global__ void slice_ranges_kernel(const SortSlice *__restrict__ ss, int S,
                                    const PlanHdr *__restrict__ hdr,
                                    const uint32_t *__restrict__ offs, int n_bins,
                                    int2 *__restrict__ range) {
    pdl_entry();
    __shared__ int s_tb[64];
    if (plan_overflow(hdr)) return;
    for (int q = threadIdx.x; q < S; q += blockDim.x) s_tb[q] = ss[q].tile_base;
    __syncthreads();
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n_bins) return;
    int s = 0;
#pragma unroll
    for (int step = 32; step > 0; step >>= 1)   // last slice whose tile_base <= b
        if (s + step < S && s_tb[s + step] <= b) s += step;
    const SortSlice q = ss[s];
    const int t = b - q.tile_base;
    if (q.nb == 0) {
        range[b] = make_int2(q.inst_base, q.inst_base);
        return;
    }
    const int lo = (int)offs[(size_t)q.hoff + (size_t)t * q.nb];
    const int hi = (t + 1 < q.ntile) ? (int)offs[(size_t)q.hoff + (size_t)(t + 1) * q.nb]
                                     : q.inst_base + q.k;
    range[b] = make_int2(lo, hi);
}

__global__ void bin_ranges_kernel(const uint32_t *__restrict__ keys, int64_t n,
                                  int2 *__restrict__ range) {
    pdl_entry();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t k = keys[i];
    if (i == 0 || keys[i - 1] != k) range[k].x = (int)i;
    if (i == n - 1 || keys[i + 1] != k) range[k].y = (int)(i + 1);
}

}  // namespace

size_t radix_hist_entries(int64_t n) {
    const size_t nblk = (size_t)((n + kSortTile - 1) / kSortTile);
    return nblk * kRadix;
}

size_t scan_tmp_entries(size_t n) {
    size_t total = 1;
    for (size_t nb = (n + kScanTile - 1) / kScanTile; nb > 0;
         nb = nb > 8192 ? (nb + kScanTile - 1) / kScanTile : 0)
        total += nb + 1;
    return total;
}

int radix_sort_pairs(uint32_t *keys, uint32_t *vals, uint32_t *keys2,
                     uint32_t *vals2, int64_t n, int bits, uint32_t *hist,
                     uint32_t *scan_tmp, cudaStream_t st, uint32_t **keys_out,
                     uint32_t **vals_out) {
    *keys_out = keys;
    *vals_out = vals;
    if (n <= 0) return UGS_OK;
    const int nblk = (int)((n + kSortTile - 1) / kSortTile);
    const size_t hn = (size_t)nblk * kRadix;
    uint32_t *kin = keys, *vin = nullptr, *kout = keys2, *vout = vals2;
    const int passes = bits <= 0 ? 1 : (bits + kRadixBits - 1) / kRadixBits;
    for (int p = 0; p < passes; ++p) {
        const int shift = p * kRadixBits;
        UGS_PDL(radix_hist_kernel, nblk, kSortThreads, 0, st,
        kin, n, shift, hist, nblk);
        UGS_LAUNCH_CHECK("radix_hist_kernel");
        int rc = exclusive_scan(hist, hist, hn, scan_tmp, st);
        if (rc) return rc;
        UGS_PDL(radix_scatter_kernel, nblk, kSortThreads, 0, st,
        kin, vin, kout, vout,
                                                            n, shift, hist, nblk);
        UGS_LAUNCH_CHECK("radix_scatter_kernel");
        // ping-pong: first pass reads identity values, writes vals2
        uint32_t *tk = kin, *tv = vin;
        kin = kout;
        vin = vout;
        kout = tk;
        vout = (tv == nullptr) ? vals : tv;
    }
    *keys_out = kin;
    *vals_out = vin;
    return UGS_OK;
}

int slice_sort_bins(const uint32_t *keys, const SortSlice *d_ss, int S, const PlanHdr *hdr,
                    int64_t hist_grid, int max_tiles, int n_bins, int nblk_grid,
                    uint32_t *hist, uint32_t *scan_tmp, uint32_t *vals_out,
                    int2 *bin_range, cudaStream_t st, const SortHook *after_ranges) {
    // the per-tile ranges come straight from the scanned histogram, so they
    // are launched before the scatter: a hook (the raster CTA order) can run
    // on a side stream while the scatter runs
    const size_t hsm = sizeof(uint32_t) * (size_t)max_tiles;
    if (nblk_grid > 0) {
        UGS_PDL(slice_hist_kernel, nblk_grid, kSortThreads, hsm, st,
        keys, d_ss, S, hdr, hist);
        UGS_LAUNCH_CHECK("slice_hist_kernel");
        int rc = exclusive_scan(hist, hist, (size_t)hist_grid, scan_tmp, st, &hdr->hist_n);
        if (rc) return rc;
    }
    // an empty batch (no sort blocks) still gets its ranges: slice_ranges
    // writes [inst_base, inst_base) for every tile of a slice without blocks
    const int th = 256;
    if (n_bins > 0) {
        UGS_PDL(slice_ranges_kernel, (n_bins + th - 1) / th, th, 0, st,
        d_ss, S, hdr, hist, n_bins,
                                                                   bin_range);
        UGS_LAUNCH_CHECK("slice_ranges_kernel");
    }
    if (after_ranges) {
        int rc = after_ranges->fn(after_ranges->ctx, st);
        if (rc) return rc;
    }
    if (nblk_grid > 0) {
        const int bits = max_tiles <= 256 ? 8 : 10;
        const size_t ssm = sizeof(uint32_t) * (kSortThreads / 32) * ((size_t)1 << bits);
        if (bits == 8) {
            UGS_PDL(slice_scatter_kernel<8>, nblk_grid, kSortThreads, ssm, st,
        keys, d_ss, S, hdr,
                                                                          hist, vals_out);
        } else {
            static std::atomic<unsigned long long> attr{0};
            if (!device_setup_done(attr)) {
                UGS_CUDA(cudaFuncSetAttribute(slice_scatter_kernel<10>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)ssm));
                mark_device_setup(attr);
            }
            UGS_PDL(slice_scatter_kernel<10>, nblk_grid, kSortThreads, ssm, st,
        keys, d_ss, S, hdr,
                                                                           hist, vals_out);
        }
        UGS_LAUNCH_CHECK("slice_scatter_kernel");
    }
    return UGS_OK;
}

int launch_bin_ranges(const uint32_t *keys, int64_t n, int2 *bin_range,
                      int n_bins, cudaStream_t st) {
    UGS_CUDA(cudaMemsetAsync(bin_range, 0, sizeof(int2) * (size_t)n_bins, st));
    if (n <= 0) return UGS_OK;
    const int th = 256;
    UGS_PDL(bin_ranges_kernel, (unsigned)((n + th - 1) / th), th, 0, st,
        keys, n,
                                                                    bin_range);
    UGS_LAUNCH_CHECK("bin_ranges_kernel");
    return UGS_OK;
}

}  // namespace ugs
