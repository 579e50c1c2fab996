// Phase 1 for a batch of slices: per-Gaussian factor + chi^2 box + cull +
// compact + clamped windows (ref rasterizer.py:109-137), fused with the
// per-(slice, Gaussian) record build and the tile-instance expansion.
//
//   count        : one thread per Gaussian, loops over the S slices of the
//                  batch: accept ballots, windows, per-warp and per-block
//                  (accepted, tiles) counts
//   scan, plan   : exclusive scan of the block counts per slice (ascending
//                  Gaussian order = the reference's compact() order), slice
//                  bases and bin-sort tables on the device
//   warp_offsets : first record / instance of every (slice, warp)
//   build        : one thread per record: finds its Gaussian from the record
//                  index, float64 plane conditioning, tile instances
#include "ugs_geometry.cuh"

namespace ugs {

namespace {

constexpr int kMaxSlicesSmem = 64;
constexpr int kBuildThreads = 128;   // records per build block
constexpr int kBucket = 32;          // records per rec_bucket entry (one build warp)

__device__ __forceinline__ void load_slices_smem(ugs_slice *dst,
                                                 const ugs_slice *src, int S) {
    const int words = S * (int)(sizeof(ugs_slice) / 4);
    const uint32_t *s = reinterpret_cast<const uint32_t *>(src);
    uint32_t *d = reinterpret_cast<uint32_t *>(dst);
    for (int i = threadIdx.x; i < words; i += blockDim.x) d[i] = s[i];
}

__global__ void __launch_bounds__(kPrepThreads)
prepare_count_kernel(const float *__restrict__ means,
                     const float *__restrict__ l_raw, int64_t n, float beta,
                     const ugs_slice *__restrict__ slices, int S,
                     uint2 *__restrict__ blk_cnt, unsigned *__restrict__ blk_pairs,
                     int nblk, uint2 *__restrict__ win_sparse,
                     uint32_t *__restrict__ amask, uint2 *__restrict__ wcnt) {
    pdl_entry();
    constexpr int kW = kPrepThreads / 32;
    __shared__ ugs_slice sl[kMaxSlicesSmem];
    __shared__ unsigned s_tiles[kMaxSlicesSmem], s_pairs[kMaxSlicesSmem];
    __shared__ unsigned s_wt[kMaxSlicesSmem][kW], s_bal[kMaxSlicesSmem][kW];
    __shared__ uint32_t s_acc[kMaxSlicesSmem][kW];   // accept bits per (slice, warp)
    __shared__ float s_fac[kW][9][32];                // L^-T (6) + mean (3) per lane
    __shared__ uint16_t s_list[kW][32 * 32];          // candidate (slice << 5 | lane)
    load_slices_smem(sl, slices, S);
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
        s_tiles[s] = 0;
        s_pairs[s] = 0;
    }
    for (int i = threadIdx.x; i < S * kW; i += blockDim.x) (&s_wt[0][0])[i] = 0;
    __syncthreads();
    const int64_t g = (int64_t)blockIdx.x * kPrepThreads + threadIdx.x;
    const bool valid = g < n;
    Factor f;
    float mu[3] = {0.f, 0.f, 0.f};
    if (valid) {
        f = make_factor(l_raw, g, beta);
        mu[0] = __ldg(means + 3 * g);
        mu[1] = __ldg(means + 3 * g + 1);
        mu[2] = __ldg(means + 3 * g + 2);
    }
    // 1) the cheap plane-straddle test for every slice
    uint64_t zmask = 0;
    if (valid)
        for (int s = 0; s < S; ++s)
            if (straddles(mu, f, sl[s])) zmask |= 1ull << s;
    // 2) the in-plane test and window for the straddled (slice, Gaussian)
    //    pairs, COMPACTED across the warp: every lane publishes its Gaussian's
    //    L^-T and mean, the warp lists its candidate pairs and each lane takes
    //    every 32nd -- ~2 rounds of full lanes instead of max-over-lanes
    //    (~5) rounds of mostly idle ones
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t nwarp_all = (int64_t)nblk * (kPrepThreads / 32);
    const int64_t gwarp = (int64_t)blockIdx.x * (kPrepThreads / 32) + warp;
    {
        float *fw = &s_fac[warp][0][0];
        fw[0 * 32 + lane] = f.LT[0][0];
        fw[1 * 32 + lane] = f.LT[0][1];
        fw[2 * 32 + lane] = f.LT[0][2];
        fw[3 * 32 + lane] = f.LT[1][1];
        fw[4 * 32 + lane] = f.LT[1][2];
        fw[5 * 32 + lane] = f.LT[2][2];
        fw[6 * 32 + lane] = mu[0];
        fw[7 * 32 + lane] = mu[1];
        fw[8 * 32 + lane] = mu[2];
    }
    for (int s = lane; s < S; s += 32) s_acc[s][warp] = 0u;
    __syncwarp();
    for (int c0 = 0; c0 < S; c0 += 32) {
        const uint32_t zc = (uint32_t)(zmask >> c0);
        const unsigned cnt = __popc(zc);
        unsigned incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const unsigned total = __shfl_sync(0xffffffffu, incl, 31);
        unsigned j = incl - cnt;
        for (uint32_t m = zc; m; m &= m - 1)
            s_list[warp][j++] = (uint16_t)(((c0 + __ffs(m) - 1) << 5) | lane);
        __syncwarp();
        for (unsigned k = lane; k < total; k += 32) {
            const unsigned e = s_list[warp][k];
            const int src = e & 31, sidx = e >> 5;
            const float *fw = &s_fac[warp][0][0];
            Factor fx;
            fx.L00 = fx.L10 = fx.L11 = fx.L20 = fx.L21 = fx.L22 = 0.f;
            fx.LT[0][0] = fw[0 * 32 + src];
            fx.LT[0][1] = fw[1 * 32 + src];
            fx.LT[0][2] = fw[2 * 32 + src];
            fx.LT[1][0] = 0.f;
            fx.LT[1][1] = fw[3 * 32 + src];
            fx.LT[1][2] = fw[4 * 32 + src];
            fx.LT[2][0] = 0.f;
            fx.LT[2][1] = 0.f;
            fx.LT[2][2] = fw[5 * 32 + src];
            const float mx[3] = {fw[6 * 32 + src], fw[7 * 32 + src], fw[8 * 32 + src]};
            Window w;
            if (cull_window_xy(mx, fx, sl[sidx], w)) {
                atomicOr(&s_acc[sidx][warp], 1u << src);
                // the emit pass reads the window back instead of recomputing
                win_sparse[(size_t)sidx * n + gwarp * 32 + src] =
                    make_uint2(w.iu0 | (w.iu1 << 16), w.iv0 | (w.iv1 << 16));
                // integer sums: shared atomics give exact (order-free) totals
                const unsigned nt = (unsigned)window_tiles(w);
                atomicAdd(&s_tiles[sidx], nt);
                atomicAdd(&s_wt[sidx][warp], nt);
                atomicAdd(&s_pairs[sidx],
                          (unsigned)((w.iu1 - w.iu0 + 1) * (w.iv1 - w.iv0 + 1)));
            }
        }
        __syncwarp();
    }
    for (int s = lane; s < S; s += 32) {
        const unsigned bal = s_acc[s][warp];
        amask[(size_t)s * nwarp_all + gwarp] = bal;
        s_bal[s][warp] = (unsigned)__popc(bal);
    }
    __syncthreads();
    // per warp: (accepted, tiles) of the block's EARLIER warps, so the emit
    // pass gets its offsets with one load and no block-wide scan
    for (int i = threadIdx.x; i < S * kW; i += blockDim.x) {
        const int s = i / kW, wp = i % kW;
        unsigned a = 0, t = 0;
        for (int k = 0; k < wp; ++k) {
            a += s_bal[s][k];
            t += s_wt[s][k];
        }
        wcnt[(size_t)s * nwarp_all + (int64_t)blockIdx.x * kW + wp] = make_uint2(a, t);
    }
    for (int s = threadIdx.x; s < S; s += blockDim.x) {
        unsigned a = 0;
#pragma unroll
        for (int wp = 0; wp < kW; ++wp) a += s_bal[s][wp];
        blk_cnt[(size_t)s * nblk + blockIdx.x] = make_uint2(a, s_tiles[s]);
        blk_pairs[(size_t)s * nblk + blockIdx.x] = s_pairs[s];
    }
}

// One block per slice: exclusive scan of blk_cnt[s][:] in place; totals in
// 64-bit (the host rejects batches whose totals exceed the 31-bit budget).
__global__ void __launch_bounds__(1024)
prepare_scan_kernel(uint2 *__restrict__ blk_cnt,
                    const unsigned *__restrict__ blk_pairs, int nblk,
                    unsigned long long *__restrict__ slice_tot) {
    pdl_entry();
    __shared__ unsigned long long wx[32], wy[32], wp[32];
    __shared__ unsigned long long carry_x, carry_y;
    {   // total (pairs) of this slice: plain reduction, fixed order
        unsigned long long acc = 0;
        for (int i = threadIdx.x; i < nblk; i += blockDim.x)
            acc += blk_pairs[(size_t)blockIdx.x * nblk + i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0) wp[threadIdx.x >> 5] = acc;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < 32; ++w) t += wp[w];
            slice_tot[3 * blockIdx.x + 2] = t;
        }
    }
    const int s = blockIdx.x;
    uint2 *row = blk_cnt + (size_t)s * nblk;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { carry_x = 0; carry_y = 0; }
    __syncthreads();
    // passes of 4 consecutive entries per thread: one block scan per 4096
    // entries (one pass for up to 1M Gaussians) instead of one per 1024
    constexpr int kPer = 4;
    for (int base = 0; base < nblk; base += kPer * 1024) {
        const int i0 = base + kPer * threadIdx.x;
        uint2 v[kPer];
        unsigned long long x = 0, y = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            v[k] = i0 + k < nblk ? row[i0 + k] : make_uint2(0, 0);
            x += v[k].x;
            y += v[k].y;
        }
        // inclusive warp scan of the thread totals
        unsigned long long ix = x, iy = y;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            unsigned long long tx = __shfl_up_sync(0xffffffffu, ix, o);
            unsigned long long ty = __shfl_up_sync(0xffffffffu, iy, o);
            if (lane >= o) { ix += tx; iy += ty; }
        }
        if (lane == 31) { wx[warp] = ix; wy[warp] = iy; }
        __syncthreads();
        if (warp == 0) {
            unsigned long long a = wx[lane], b = wy[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                unsigned long long ta = __shfl_up_sync(0xffffffffu, a, o);
                unsigned long long tb = __shfl_up_sync(0xffffffffu, b, o);
                if (lane >= o) { a += ta; b += tb; }
            }
            wx[lane] = a;   // inclusive warp-sum prefix
            wy[lane] = b;
        }
        __syncthreads();
        unsigned long long px = (warp ? wx[warp - 1] : 0ull) + ix - x + carry_x;
        unsigned long long py = (warp ? wy[warp - 1] : 0ull) + iy - y + carry_y;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            if (i0 + k < nblk) row[i0 + k] = make_uint2((unsigned)px, (unsigned)py);
            px += v[k].x;
            py += v[k].y;
        }
        __syncthreads();
        if (threadIdx.x == 0) { carry_x += wx[31]; carry_y += wy[31]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        slice_tot[3 * s] = carry_x;
        slice_tot[3 * s + 1] = carry_y;
    }
}

// Per (slice, warp of 32 Gaussians): the warp's first record and first
// instance, from the block offsets (scan) and the within-block warp offsets
// (count pass).  Empty warps get the offset of the next record, so the
// flattened [S][nwarp] row is non-decreasing -- build_records searches it.
// Every non-empty warp also records itself as the owner of each multiple of
// kBucket among its records: rec_bucket[b] = the flattened warp that holds
// record b * kBucket, so a build warp searches only between rec_bucket[b]
// and rec_bucket[b + 1].
__global__ void warp_offsets_kernel(int S, int64_t nwarp_all, int nblk,
                                    const uint2 *__restrict__ blk_off,
                                    const uint2 *__restrict__ wcnt,
                                    const uint32_t *__restrict__ amask,
                                    const int64_t *__restrict__ slice_base,
                                    int32_t *__restrict__ warp_rec,
                                    int32_t *__restrict__ warp_inst,
                                    int32_t *__restrict__ rec_bucket,
                                    int32_t *__restrict__ rec_inst,
                                    const PlanHdr *__restrict__ hdr) {
    pdl_entry();
    if (plan_overflow(hdr)) return;
    const int64_t m_total = (int64_t)hdr->m, k_total = (int64_t)hdr->k;
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nw = (int64_t)S * nwarp_all;
    if (idx == 0) {
        rec_inst[m_total] = (int32_t)k_total;
        rec_bucket[(m_total + kBucket - 1) / kBucket] = (int32_t)(nw - 1);
    }
    if (idx >= nw) return;
    const int s = (int)(idx / nwarp_all);
    const int64_t gw = idx - (int64_t)s * nwarp_all;
    const uint2 bo = __ldg(blk_off + (size_t)s * nblk + gw / (kPrepThreads / 32));
    const uint2 c = __ldg(wcnt + idx);
    const int32_t r0 = (int32_t)(slice_base[2 * s] + bo.x + c.x);
    warp_rec[idx] = r0;
    warp_inst[idx] = (int32_t)(slice_base[2 * s + 1] + bo.y + c.y);
    const int32_t r1 = r0 + __popc(__ldg(amask + idx));
    for (int32_t q = (r0 + kBucket - 1) / kBucket * kBucket; q < r1; q += kBucket)
        rec_bucket[q / kBucket] = (int32_t)idx;
}

__device__ __forceinline__ unsigned packed_tiles(uint2 w) {
    return (((w.x >> 16) >> 4) - ((w.x & 0xffff) >> 4) + 1) *
           (((w.y >> 16) >> 4) - ((w.y & 0xffff) >> 4) + 1);
}

// One thread per accepted (slice, Gaussian) record.  It finds its Gaussian
// from the record index alone -- (slice, Gaussian warp) by a register binary
// search of the flattened warp_rec window that holds the build warp's 32
// records, lane as the k-th set bit of the warp's accept ballot -- and its
// first instance as the Gaussian warp's plus the tile counts of the warp's
// earlier accepted lanes, by a segmented warp scan (no separate emit pass,
// no serial dependent loads).  Then the
// plane-conditioned exponent (float64, ugs_geometry.cuh PlaneForm) and the
// record's tile instances in row-major tile order, each with its exact
// re-expansion.
#ifndef UGS_BUILD_MINB
#define UGS_BUILD_MINB 8
#endif
__global__ void __launch_bounds__(kBuildThreads, UGS_BUILD_MINB)
build_records_kernel(const float *__restrict__ means, const float *__restrict__ l_raw,
                     const float *__restrict__ intensity_raw,
                     const float *__restrict__ opacity_raw, int64_t n, float beta,
                     const ugs_slice *__restrict__ slices, int S,
                     const int64_t *__restrict__ slice_base,
                     const PlanHdr *__restrict__ hdr, int64_t nwarp_all, const uint32_t *__restrict__ amask,
                     const int32_t *__restrict__ warp_rec,
                     const int32_t *__restrict__ warp_inst,
                     const int32_t *__restrict__ rec_bucket,
                     const uint2 *__restrict__ win_sparse, Rec *__restrict__ rec,
                     int32_t *__restrict__ rec_gid, int32_t *__restrict__ rec_inst,
                     Frag *__restrict__ frag, uint32_t *__restrict__ keys) {
    pdl_entry();
    if (plan_overflow(hdr)) return;
    const int64_t m_total = (int64_t)hdr->m;
    const int ln = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * kBuildThreads + threadIdx.x;
    const int64_t rw0 = r - ln;                   // this warp's first record
    if (rw0 >= m_total) return;                   // whole warp
    const bool valid = r < m_total;
    const int32_t r32 = (int32_t)min(r, m_total - 1);
    // 1) (slice, Gaussian warp) of every lane's record: the flattened warps
    //    holding this warp's 32 records lie between rec_bucket[b] and
    //    rec_bucket[b + 1]; one coalesced load of that warp_rec window and a
    //    register binary search (shuffles), no dependent global loads
    const int64_t b = rw0 / kBucket;
    const int blo = __ldg(rec_bucket + b), bhi = __ldg(rec_bucket + b + 1);
    int flat;
    int32_t first;                                // warp_rec[flat]
    if (bhi - blo < 32) {
        const int32_t e = ln <= bhi - blo ? __ldg(warp_rec + blo + ln) : INT32_MAX;
        int pos = 0;
#pragma unroll
        for (int step = 16; step > 0; step >>= 1) {
            const int32_t v = __shfl_sync(0xffffffffu, e, pos + step);
            if (v <= r32) pos += step;
        }
        flat = blo + pos;
        first = __shfl_sync(0xffffffffu, e, pos);
    } else {                                      // sparse slices: per-lane search
        int lo = blo, hi = bhi;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(warp_rec + mid) <= r32) lo = mid; else hi = mid - 1;
        }
        flat = lo;
        first = __ldg(warp_rec + lo);
    }
    const int s = (int)((unsigned)flat / (unsigned)nwarp_all);
    const int lo = flat - s * (int)nwarp_all;
    const uint32_t word = __ldg(amask + flat);
    const int32_t winst = __ldg(warp_inst + flat);   // with the word, not after the scan
    const int k = (int)(r32 - first);
    const int lane = (int)__fns(word, 0, k + 1);
    const int64_t g = (int64_t)lo * 32 + lane;
    const uint2 *ws = win_sparse + (size_t)s * n + (int64_t)lo * 32;
    const uint2 pw = __ldg(ws + lane);
    // the Gaussian's parameters are issued with the window load, ahead of
    // the first-instance scan, so their round trips overlap it (g is a valid
    // index on every lane: r32 is clamped)
    const float ir = __ldg(intensity_raw + g), orw = __ldg(opacity_raw + g);
    const float mu[3] = {__ldg(means + 3 * g), __ldg(means + 3 * g + 1),
                         __ldg(means + 3 * g + 2)};
    const Factor f = make_factor(l_raw, g, beta);
    // 2) first instance: the Gaussian warp's plus the tiles of its earlier
    //    accepted lanes -- a segmented warp scan over this warp's records
    //    (consecutive records of one Gaussian warp are consecutive lanes),
    //    plus, for the segment that began before this warp, the tiles of its
    //    records in the previous warp (one parallel load per such record)
    const unsigned nt = valid ? packed_tiles(pw) : 0u;
    unsigned incl = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
        const int kf = __shfl_up_sync(0xffffffffu, flat, o);
        if (ln >= o && kf == flat) incl += t;
    }
    const int flat0 = __shfl_sync(0xffffffffu, flat, 0);
    const int k0 = __shfl_sync(0xffffffffu, k, 0);   // records of segment 0 before rw0
    unsigned pre = 0;
    if (k0 > 0) {
        const uint32_t word0 = __shfl_sync(0xffffffffu, word, 0);
        const int s0 = (int)((unsigned)flat0 / (unsigned)nwarp_all);
        const int lo0 = flat0 - s0 * (int)nwarp_all;
        if (ln < k0)
            pre = packed_tiles(__ldg(win_sparse + (size_t)s0 * n + (int64_t)lo0 * 32 +
                                     __fns(word0, 0, ln + 1)));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pre += __shfl_xor_sync(0xffffffffu, pre, o);
    }
    if (!valid) return;
    int64_t inst = (int64_t)winst + (incl - nt) + (flat == flat0 ? pre : 0u);
    rec_gid[r] = (int32_t)g;
    rec_inst[r] = (int32_t)inst;
    const ugs_slice &L = slices[s];
    const float color = sigmoid_f32(ir);
    const float alpha = sigmoid_f32(orw);
    const Window w{(int)(pw.x & 0xffff), (int)(pw.x >> 16), (int)(pw.y & 0xffff),
                   (int)(pw.y >> 16)};
    const PlaneForm P = plane_form(mu, f, L, w);
    const double kq = -0.72134752044448170368;   // -0.5 * log2(e)
    const double log2a = log2((double)alpha);
    const float4 q0 = make_float4((float)(kq * P.H00), (float)(kq * 2.0 * P.H01),
                                  (float)(kq * P.H11), color);
#if UGS_V8
    st_v8(rec + r, q0,
          make_float4(__uint_as_float(pw.x), __uint_as_float(pw.y), alpha,
                      __int_as_float(P.ui | (P.vi << 16))));
#else
    rec[r].r0 = q0;
    rec[r].r1 = make_float4(__uint_as_float(pw.x), __uint_as_float(pw.y), alpha,
                            __int_as_float(P.ui | (P.vi << 16)));
#endif
    const int tx0 = w.iu0 >> 4, tx1 = w.iu1 >> 4;
    const int ty0 = w.iv0 >> 4, ty1 = w.iv1 >> 4;
    for (int ty = ty0; ty <= ty1; ++ty)
        for (int tx = tx0; tx <= tx1; ++tx) {
            const int tu0 = tx * kTile, tv0 = ty * kTile;
            const TileRect t = tile_rect(w.iu0, w.iu1, w.iv0, w.iv1, tu0, tv0, P.ui, P.vi);
            double D, E, F;
            expansion(P, t.pu, t.pv, kq, log2a, D, E, F);
            const int bits = (t.x0 - tu0) | ((t.x1 - tu0) << 4) | ((t.y0 - tv0) << 8) |
                             ((t.y1 - tv0) << 12) | ((t.pu - tu0) << 16) |
                             ((t.pv - tv0) << 20);
            Frag *fp = frag + inst;
#if UGS_V8
            st_v8(fp, q0, make_float4((float)D, (float)E, (float)F, __int_as_float(bits)));
#else
            fp->q0 = q0;
            fp->q1 = make_float4((float)D, (float)E, (float)F, __int_as_float(bits));
#endif
            keys[inst] = (uint32_t)(L.tile_base + ty * L.tiles_x + tx);
            ++inst;
        }
}

// One thread: per-slice record / instance bases and the bin-sort tables from
// the per-slice totals, on the device -- the host only reads the totals back
// (one pinned D2H copy) to size buffers and grids.  totals = (m, k, pairs,
// sort-table entries, sort blocks).
__global__ void plan_slices_kernel(unsigned long long *__restrict__ tot,
                                   const ugs_slice *__restrict__ slices, int S,
                                   int64_t *__restrict__ slice_base,
                                   SortSlice *__restrict__ ss, PlanCaps caps) {
    pdl_entry();
    // one thread per slice: its bases are prefix sums over the earlier
    // slices (S <= 64: a short loop, all slices in parallel)
    __shared__ unsigned long long sm[64], sk[64], sp[64];
    __shared__ int snb[64], snt[64];
    const int s = threadIdx.x;
    if (s < S) {
        sm[s] = tot[3 * s];
        sk[s] = tot[3 * s + 1];
        sp[s] = tot[3 * s + 2];
        snt[s] = slices[s].tiles_x * slices[s].tiles_y;
        snb[s] = (int)((sk[s] + kSortTile - 1) / kSortTile);
    }
    __syncthreads();
    if (s < S) {
        unsigned long long m = 0, k = 0, hn = 0, nbs = 0;
        for (int q = 0; q < s; ++q) {
            m += sm[q];
            k += sk[q];
            nbs += (unsigned long long)snb[q];
            hn += (unsigned long long)snt[q] * snb[q];
        }
        slice_base[2 * s] = (int64_t)m;
        slice_base[2 * s + 1] = (int64_t)k;
        SortSlice q;
        q.inst_base = (int)k;
        q.k = (int)sk[s];
        q.tile_base = slices[s].tile_base;
        q.ntile = snt[s];
        q.nb = snb[s];
        q.bpre = (int)nbs;
        q.hoff = (int)hn;
        q.pad = 0;
        ss[s] = q;
        if (s == S - 1) {
            unsigned long long pr = 0;
            for (int q2 = 0; q2 < S; ++q2) pr += sp[q2];
            unsigned long long *t = tot + 3 * kMaxSlicesSmem;
            t[0] = m + sm[s];
            t[1] = k + sk[s];
            t[2] = pr;
            t[3] = hn + (unsigned long long)snt[s] * snb[s];
            t[4] = nbs + (unsigned long long)snb[s];
            // the batch must fit the buffers the launches were sized for
            // (and the 31-bit index budget); else the plan's later kernels
            // all return at entry and the host grows the buffers and retries
            t[5] = (t[0] > caps.m || t[1] > caps.k || t[3] > caps.hist ||
                    t[4] > caps.nblk || t[0] >= 0x7fffffffull || t[1] >= 0x7fffffffull)
                       ? 1ull : 0ull;
        }
    }
}

}  // namespace

int launch_prepare_count(const ugs_cloud &c, const ugs_slice *slices, int S,
                         uint2 *blk_cnt, unsigned *blk_pairs, int nblk,
                         uint2 *win_sparse, uint32_t *amask, uint2 *wcnt, cudaStream_t st) {
    UGS_PDL(prepare_count_kernel, nblk, kPrepThreads, 0, st,
        c.means, c.l_raw, c.n, (float)c.beta, slices, S, blk_cnt, blk_pairs, nblk,
        win_sparse, amask, wcnt);
    UGS_LAUNCH_CHECK("prepare_count_kernel");
    return UGS_OK;
}

int launch_plan_slices(unsigned long long *slice_tot, const ugs_slice *slices, int S,
                       int64_t *slice_base, SortSlice *ss, PlanCaps caps, cudaStream_t st) {
    UGS_PDL(plan_slices_kernel, 1, 64, 0, st,
        slice_tot, slices, S, slice_base, ss, caps);
    UGS_LAUNCH_CHECK("plan_slices_kernel");
    return UGS_OK;
}

int launch_prepare_scan(uint2 *blk_cnt, const unsigned *blk_pairs, int S, int nblk,
                        unsigned long long *slice_tot, cudaStream_t st) {
    UGS_PDL(prepare_scan_kernel, S, 1024, 0, st,
        blk_cnt, blk_pairs, nblk, slice_tot);
    UGS_LAUNCH_CHECK("prepare_scan_kernel");
    return UGS_OK;
}

int launch_prepare_emit(const ugs_cloud &c, const ugs_slice *slices, int S,
                        const uint2 *blk_off, int nblk, const int64_t *slice_base,
                        Rec *rec, int32_t *rec_gid, int32_t *rec_inst,
                        Frag *frag, uint32_t *keys, const PlanHdr *hdr, int64_t m_grid,
                        const uint2 *win_sparse, const uint32_t *amask,
                        const uint2 *wcnt, int32_t *warp_rec, int32_t *warp_inst,
                        int32_t *rec_bucket, cudaStream_t st) {
    const int64_t nwarp_all = (int64_t)nblk * (kPrepThreads / 32);
    const int64_t nw = (int64_t)S * nwarp_all;
    UGS_PDL(warp_offsets_kernel, (unsigned)((nw + 255) / 256), 256, 0, st,
        S, nwarp_all, nblk, blk_off, wcnt, amask, slice_base, warp_rec, warp_inst,
        rec_bucket, rec_inst, hdr);
    UGS_LAUNCH_CHECK("warp_offsets_kernel");
    if (m_grid <= 0) return UGS_OK;
    UGS_PDL(build_records_kernel, (unsigned)((m_grid + kBuildThreads - 1) / kBuildThreads), kBuildThreads, 0, st,
        c.means, c.l_raw, c.intensity_raw, c.opacity_raw, c.n, (float)c.beta, slices, S,
        slice_base, hdr, nwarp_all, amask, warp_rec, warp_inst, rec_bucket, win_sparse, rec,
        rec_gid, rec_inst, frag, keys);
    UGS_LAUNCH_CHECK("build_records_kernel");
    return UGS_OK;
}

}  // namespace ugs
