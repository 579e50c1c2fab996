// Tile-resident forward accumulation and backward for a batch of slices.
//
// One CTA per (slice, 16x16 tile), 8 warps.  The tile's sorted instance list
// (ascending Gaussian index, from the stable bin sort) is staged through
// shared memory in batches (forward 256, backward 512 instances): each
// instance's 32-byte Frag arrives by cp.async (LDGSTS) issued one batch
// ahead, so the gathers overlap the previous batch's accumulation.  While staging, one thread per instance
// clips the record's window to the tile and precomputes what the lanes need
// (rectangle, offsets from the instance's expansion pixel, lane layout); the
// batch is then ordered by loop trip count with a stable counting sort, so
// the records processed together by a warp need the same number of sweeps.
//
// Per pair the reference evaluates w = alpha exp(-q/2), q = |L^T(p - mu)|^2
// (28 flops, float64).  Phase 1 has conditioned each Gaussian on the slice
// plane (ugs_geometry.cuh, PlaneForm) and re-expanded it exactly around each
// instance's expansion pixel: log2 w is a 2-D quadratic in exact integer
// offsets bounded by the tile, so with x fixed per lane a pair costs 2 FMA +
// one MUFU ex2.
//
//   Forward: narrow records (< 9 clipped columns) two per warp (16-lane
//   groups, cw = pow2 >= width columns x 16/cw rows per sweep); each group
//   adds into its own PRIVATE (num, den) tile buffer (XOR-swizzled float2).
//   Wide records one per warp, lane = (tile column, row parity), each lane
//   keeping the (num, den) of its 8 pixels in REGISTERS across all of the
//   tile's wide records.  At the end the register tiles join the group
//   buffers and the 16 buffers are summed in fixed order -- the reference's
//   multi-worker scheme (private accumulators summed, rasterizer.py:157-173),
//   deterministic because the record -> group / warp assignment is a fixed
//   function of the batch.  `forward_ordered_kernel` keeps the strict
//   ascending-index order per pixel (ref _kernels.py:23-47), selectable with
//   ugs_plan_set_ordered.
//   Backward: sixteen records per warp (2-lane groups), two pixel streams
//   per lane with fixed columns (stage_record2; records wider than 4 columns
//   in 4-column passes), 32 units of sixteen per 512-instance batch taken
//   from a largest-first warp work queue.  The per-Gaussian gradient needs only 7 weighted moments of
//   the pixel offsets (sum G w, sum t, sum t dx, sum t dy, sum t dx^2,
//   sum t dx dy, sum t dy^2; G = dpix/ssum, t = dw w), accumulated in
//   registers; a 2-lane transpose-reduce leaves lane j with moments 4j ..
//   4j + 3 and the group writes one 32-byte partial per tile instance (one
//   256-bit store by its first lane).
// finalize_records sums a record's instance partials in order (shifting each
// to the record's reference pixel) and applies the closed-form float64 chain
// to d_mu, d_L and the raw parameters; update_gather accumulates every
// Gaussian's records in slice order and runs densify statistics + Adam -- no
// atomics anywhere, so gradients are bitwise reproducible.
#include "ugs_adam.cuh"
#include "ugs_geometry.cuh"

namespace ugs {

namespace {

constexpr int kRasterThreads = 256;
constexpr int kWarps = kRasterThreads / 32;
constexpr int kBatch = 256;              // forward: one staged record per thread
#ifndef UGS_BWD_PER
#define UGS_BWD_PER 2
#endif
constexpr int kBwdPer = UGS_BWD_PER;     // backward: staged records per thread
constexpr int kBwdBatch = kBatch * kBwdPer;
constexpr int kMaxTrips = kTile;   // sort buckets: sweeps of a 16-lane group
constexpr int kKeyWide = kMaxTrips + 1;      // forward: warp-per-record class
constexpr int kKeyInvalid = kMaxTrips + 2;   // unused staging slots
constexpr int kKeys = kMaxTrips + 3;
// backward (4-lane groups): trip counts 1..16 (narrow / medium records) and
// 17..32 (wide records, two column passes of h rows: key 16 + h), invalid 33
constexpr int kBwdKeyInvalid = 4 * kMaxTrips + 1;
constexpr int kBwdKeys = 4 * kMaxTrips + 2;
constexpr int kKeysMax = kBwdKeys;
#ifndef UGS_WIDE_MIN
#define UGS_WIDE_MIN 9
#endif
constexpr int kWideMin = UGS_WIDE_MIN;  // forward: clipped widths >= this take the
                                   // register-tile path (one record per warp)
constexpr int kAccStride = kTile * kTile;    // forward: one private tile
constexpr int kGroups = kRasterThreads / 16; //   buffer per 16-lane group

// Private-buffer slot of tile pixel p = 16*Y + X (float2 slots: a 64-bit
// access is served 16 lanes at a time, bank pair = slot mod 16).  The forward
// sweeps a record's rectangle with cw = pow2 >= width lanes per row, so a
// 16-lane phase covers 16/cw rows; X' = X ^ 8*(Y & 1) puts adjacent rows on
// opposite bank halves (2.06 wavefronts per access on average over all
// clipped rectangles, vs 3.10 unswizzled).
__device__ __forceinline__ int acc_swizzle(int p) { return p ^ ((p >> 1) & 8); }

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float sigmoid_bg(const double *bg_raw, int i) {
    return (float)sigmoid_f64(bg_raw[i]);
}

// Packed f32x2 helpers (sm_100 FFMA2/FADD2/FMUL2: two fp32 lanes per
// register pair, each half rounded exactly like its scalar fma.rn).  A u64
// holds a live register pair, so a loop-invariant operand is not re-packed.
using u64 = unsigned long long;
__device__ __forceinline__ u64 pack2(float lo, float hi) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
    u64 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// exact float of a small non-negative int: 2^23 + x
__device__ __forceinline__ float big_float(int x) {
    return __int_as_float(0x4B000000 | x);
}

// Asynchronous staging of a tile's instances: each thread gathers the
// 32-byte Frag of its slot of the NEXT batch with cp.async (LDGSTS, L2 only)
// straight into shared memory while the CTA accumulates the current batch;
// the sorted ids are prefetched a batch further ahead.  A slot is only ever
// written and read by its own thread, so the copies need no barrier:
// cp.async.wait_all makes them visible to that thread.
__device__ __forceinline__ void stage_async(Frag *dst, const Frag *src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d + 16),
                 "l"(reinterpret_cast<const char *>(src) + 16)
                 : "memory");
}
__device__ __forceinline__ void stage_id_async(uint32_t *dst, const uint32_t *src) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void stage_commit() {
    asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void stage_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Per-thread staging pipeline over a tile's sorted range [lo, hi) (forward):
// `nxt` = the next batch's id, prefetched in a register.
struct StagePipeReg {
    uint32_t nxt;
    __device__ __forceinline__ void start(const uint32_t *__restrict__ vals,
                                          const Frag *__restrict__ frag, Frag *raw, int lo,
                                          int hi) {
        const int i = lo + (int)threadIdx.x;
        if (i < hi) stage_async(raw + threadIdx.x, frag + __ldg(vals + i));
        stage_commit();
        nxt = i + kBatch < hi ? __ldg(vals + i + kBatch) : 0u;
    }
    // after this thread staged batch b0 from raw: fetch batch b0 + kBatch
    __device__ __forceinline__ void advance(const uint32_t *__restrict__ vals,
                                            const Frag *__restrict__ frag, Frag *raw, int b0,
                                            int hi) {
        const int i = b0 + kBatch + (int)threadIdx.x;
        if (i < hi) stage_async(raw + threadIdx.x, frag + nxt);
        stage_commit();
        nxt = i + kBatch < hi ? __ldg(vals + i + kBatch) : 0u;
    }
};

// The same pipeline with its state in shared memory (backward, whose
// register budget is full: ids held across a batch were spilled, and the
// spill store waited on the load): ids[tid] = the id of this thread's slot
// of the batch after the one in flight to raw[tid], fetched by a 4-byte
// cp.async; cur[tid] = the id in raw[tid].
struct StagePipe {
    uint32_t *ids, *cur;
    __device__ __forceinline__ StagePipe(uint32_t *ids_, uint32_t *cur_) : ids(ids_), cur(cur_) {}
    __device__ __forceinline__ void start(const uint32_t *__restrict__ vals,
                                          const Frag *__restrict__ frag, Frag *raw, int lo,
                                          int hi) {
#pragma unroll
        for (int r = 0; r < kBwdPer; ++r) {
            const int sl = (int)threadIdx.x + r * kBatch, i = lo + sl;
            if (i < hi) {
                const uint32_t c = __ldg(vals + i);
                cur[sl] = c;
                stage_async(raw + sl, frag + c);
            }
            if (i + kBwdBatch < hi) stage_id_async(ids + sl, vals + i + kBwdBatch);
        }
        stage_commit();
    }
    // after this thread staged batch b0 from raw (and after stage_wait):
    // fetch batch b0 + kBwdBatch, and the ids of the batch after it
    __device__ __forceinline__ void advance(const uint32_t *__restrict__ vals,
                                            const Frag *__restrict__ frag, Frag *raw, int b0,
                                            int hi) {
#pragma unroll
        for (int r = 0; r < kBwdPer; ++r) {
            const int sl = (int)threadIdx.x + r * kBatch, i = b0 + kBwdBatch + sl;
            if (i < hi) {
                // read before the id copy below overwrites the slot: the Frag
                // copy's address depends on it
                const uint32_t c = ids[sl];
                cur[sl] = c;
                stage_async(raw + sl, frag + c);
            }
            if (i + kBwdBatch < hi) stage_id_async(ids + sl, vals + i + kBwdBatch);
        }
        stage_commit();
    }
};

// Shared-memory state of one staged batch.
//   sA = (C1x, C1y, D, E)   x = big_float(lx) - C1x: exact integer offset of
//                           the lane's pixel from the instance's expansion pixel
//   sB = (A, B2, C, F)      log2 w = A x^2 + B2 x y + C y^2 + D x + E y + F
//   sC = (color, ls, -, instance)   ls = log2 of the stream's row stride
//   sL = (cmaskA, lcwA, wideoff, lyoff), sM = (w, h, x0, y0): the record's
//        two-stream lane layout (stage_layout)
template <int NB, int NROWS>
struct BatchT {
    float4 sA[NB], sB[NB], sC[NB];
    uint16_t order[NB];                // staged slot of the j-th record by trips
    uint32_t wcnt[NROWS][kKeysMax];    // per (slot round, warp) key counts
    uint32_t base[kKeysMax];
    uint32_t next[2];                  // work-queue counters of the batch
};
using Batch = BatchT<kBatch, kWarps>;                      // forward
using BwdBatch = BatchT<kBwdBatch, kWarps * kBwdPer>;      // backward
// two-stream layouts (backward), after the BwdBatch, byte fields:
//   sL = lcwA | B column offset << 8 | B row offset << 16  (cmaskA = lcwA)
//   sM = w | h << 8 | x0 << 16 | y0 << 24
struct Layout {
    int2 sLM[kBwdBatch];
};

constexpr size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }
// forward shared memory: Batch | group accumulators | staged Frags
constexpr size_t kFwdAccOff = align16(sizeof(Batch));
constexpr size_t kFwdRawOff = align16(kFwdAccOff + sizeof(float2) * kGroups * kAccStride);
// backward shared memory: Batch | Layout | pixel terms + bg partials |
// staged Frags
constexpr size_t kBwdLyOff = align16(sizeof(BwdBatch));
constexpr size_t kBwdPixOff = kBwdLyOff + sizeof(Layout);
// the backward's per-pixel planes use a row pitch of kTile + 1 floats: the
// rows a warp's sixteen records read fall on different banks
#ifndef UGS_BWD_PITCH
#define UGS_BWD_PITCH (kTile + 1)
#endif
constexpr int kBP = UGS_BWD_PITCH;
constexpr int kBPlane = kBP * kTile;   // floats per plane
constexpr size_t kBwdRawOff =
    align16(kBwdPixOff + sizeof(float) * 2 * kBPlane + sizeof(float2) * kWarps);
constexpr size_t kBwdIdsOff = kBwdRawOff + sizeof(Frag) * kBwdBatch;   // StagePipe ids, cur

// Backward staging of one instance (one thread per record) for a group of 2
// lanes; returns its sort key.  Two pixel streams per lane, A and B, each
// with a fixed column, so that x (hence P, Q) is per-lane constant:
//   narrow  (w <= 2, cw = pow2 >= w): A = (lx, ly), B = A + (0, R), R = 2/cw,
//                                     both advance 2R rows per iteration
//   columns (w 3..16):                A = (gl, 0), B = A + (2, 0), one row
//                                     per iteration, in ceil(w/4) passes
//                                     over 4-column strips
// with lx = gl & (cw-1), ly = gl >> log2 cw.  Key: the loop trip count
// (1..16; multi-pass records 16 (passes - 1) + rows), so a warp's sixteen
// records share passes and rows.
//   sLM = the byte-packed layout (struct Layout), sC.z = passes
__device__ __forceinline__ int stage_record2(const Frag &f, uint32_t inst, BwdBatch &B, Layout &Ly,
                                             int slot) {
    const FragRect t = frag_rect(f.q1.w);
    const int w = t.x1 - t.x0 + 1, h = t.y1 - t.y0 + 1;
    const int lcw = (w > 1) ? 32 - __clz(w - 1) : 0;
    const bool cols = lcw >= 2;                 // column layouts: column-offset B
    const int lcwA = cols ? 1 : lcw;
    const int ls = cols ? 0 : 2 - lcw;          // log2 of the row stride
    const int npass = cols ? (w + 3) >> 2 : 1;
    B.sA[slot] = make_float4(8388608.0f - (float)(t.x0 - t.pu),
                             8388608.0f - (float)(t.y0 - t.pv), f.q1.x, f.q1.y);
    B.sB[slot] = make_float4(f.q0.x, f.q0.y, f.q0.z, f.q1.z);
    B.sC[slot] = make_float4(f.q0.w, __int_as_float(ls), __int_as_float(npass),
                             __int_as_float((int)inst));
    Ly.sLM[slot] = make_int2(lcwA | ((cols ? 2 : 0) << 8) | ((cols ? 0 : (2 >> lcw)) << 16),
                             w | (h << 8) | (t.x0 << 16) | (t.y0 << 24));
    return npass > 1 ? kMaxTrips * (npass - 1) + h : (h + (1 << ls) - 1) >> ls;
}

// Single-stream staging for the forward's 16-lane groups: cw = pow2 >= w
// columns x R = 16/cw rows per sweep.  The lane layout is precomputed in
// byte fields so a lane decodes each with one byte permute:
//   sC.z = cmask | lcw << 8 | (h + R - 1) << 16 | log2(R) << 24
//   sC.w = x0 | y0 << 8 | w << 16 | R << 24
// and sC.xy = (color, 1) is the FFMA2 operand of (num, den) += w (color, 1).
// Returns the number of sweeps.
__device__ __forceinline__ int stage_record_rows(const Frag &f, const FragRect &t, Batch &B,
                                                 int slot) {
    const int w = t.x1 - t.x0 + 1, h = t.y1 - t.y0 + 1;
    const int lcw = (w > 1) ? 32 - __clz(w - 1) : 0;
    const int rows = 16 >> lcw;
    B.sA[slot] = make_float4(8388608.0f - (float)(t.x0 - t.pu),
                             8388608.0f - (float)(t.y0 - t.pv), f.q1.x, f.q1.y);
    B.sB[slot] = make_float4(f.q0.x, f.q0.y, f.q0.z, f.q1.z);
    B.sC[slot] = make_float4(
        f.q0.w, 1.f,
        __int_as_float(((1 << lcw) - 1) | (lcw << 8) | ((h + rows - 1) << 16) |
                       ((4 - lcw) << 24)),
        __int_as_float(t.x0 | (t.y0 << 8) | (w << 16) | (rows << 24)));
    return (h + rows - 1) >> (4 - lcw);
}

__device__ __forceinline__ int byte_of(int x, int k) {
    return (int)__byte_perm((unsigned)x, 0u, 0x4440u | (unsigned)k);
}

// Forward staging of one tile instance (one thread per record).  Narrow
// rectangles (< kWideMin columns) get stage_record_rows' 16-lane layout and
// key = sweep count; wide ones the warp layout of the register-tile path:
//   sA = (pu, pv, D, E)   the expansion pixel (tile-relative, exact floats)
//   sB = (A, B2, C, F)
//   sC = (color, bits(x0 | w << 8), bits(vm0 | vm1 << 8 | um << 16), -)
// where lane (X, ph) owns rows 2m + ph, vm_ph = the m whose row lies in
// [y0, y1], um = vm0 | vm1 (the warp-uniform row pairs).
__device__ __forceinline__ uint32_t stage_forward(const Frag &f, Batch &B, int slot) {
    const FragRect t = frag_rect(f.q1.w);
    const int w = t.x1 - t.x0 + 1;
    if (w < kWideMin) return (uint32_t)stage_record_rows(f, t, B, slot);
    unsigned vmask[2];
#pragma unroll
    for (int ph = 0; ph < 2; ++ph) {
        const int mlo = (t.y0 - ph + 1) >> 1, mhi = (t.y1 - ph) >> 1;
        vmask[ph] = (mhi >= mlo) ? ((2u << mhi) - (1u << mlo)) : 0u;
    }
    B.sA[slot] = make_float4((float)t.pu, (float)t.pv, f.q1.x, f.q1.y);
    B.sB[slot] = make_float4(f.q0.x, f.q0.y, f.q0.z, f.q1.z);
    B.sC[slot] = make_float4(f.q0.w, __int_as_float(t.x0 | (w << 8)),
                             __int_as_float((int)(vmask[0] | (vmask[1] << 8) |
                                                  ((vmask[0] | vmask[1]) << 16))),
                             0.f);
    return (uint32_t)kKeyWide;
}

// Warp-level work queue over a batch's units, LARGEST first: the sorted
// slots ascend by loop trip count, so unit n-1-k is the k-th largest and
// warps that finish early take the remaining small ones (greedy
// longest-first balance; the batch ends at a CTA barrier).  Returns the unit
// index, or -1 when the queue is empty.  Only for work whose result does not
// depend on which warp runs a unit (the backward's per-instance partials);
// the forward's accumulation order must stay a fixed function of the batch.
__device__ __forceinline__ int next_unit(uint32_t *ctr, int nunits) {
    uint32_t k = 0;
    if ((threadIdx.x & 31) == 0) k = atomicAdd(ctr, 1u);
    k = __shfl_sync(0xffffffffu, k, 0);
    return (int)k < nunits ? nunits - 1 - (int)k : -1;
}

// Stable counting sort of the staged slots by key (trip count, or the
// forward's wide class; unused slots last) -- warp match-any ranks +
// per-warp bucket counters: a deterministic record -> lane-group mapping.
// Returns, in B.base, each key's first sorted position.
template <int NK, int PER, class BT>
__device__ __forceinline__ void sort_batch(BT &B, const uint32_t (&key)[PER]) {
    constexpr int KPL = (NK + 31) / 32;   // keys per lane of warp 0
    constexpr int kInvalid = NK - 1;
    constexpr int kRows = kWarps * PER;   // row r kWarps + w: slots r kBatch + 32 w ..
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // 1) per-row key counts: each warp clears and fills its own rows
#pragma unroll
    for (int r = 0; r < PER; ++r)
        for (int k = lane; k < NK; k += 32) B.wcnt[r * kWarps + warp][k] = 0u;
    if (threadIdx.x < 2) B.next[threadIdx.x] = 0u;
    uint32_t rank[PER];
    unsigned peers[PER];
#pragma unroll
    for (int r = 0; r < PER; ++r) {
        peers[r] = __match_any_sync(0xffffffffu, key[r]);
        rank[r] = __popc(peers[r] & ((1u << lane) - 1u));
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < PER; ++r)
        if (rank[r] == 0) B.wcnt[r * kWarps + warp][key[r]] = __popc(peers[r]);
    __syncthreads();
    // 2) warp 0: bucket bases (exclusive scan over keys, lane l holds keys
    //    KPL l .. KPL l + KPL - 1) and each row's running offset per key
    if (warp == 0) {
        uint32_t col[KPL];
#pragma unroll
        for (int q = 0; q < KPL; ++q) {
            col[q] = 0u;
            const int k = KPL * lane + q;
            if (k < NK) {
#pragma unroll
                for (int w = 0; w < kRows; ++w) col[q] += B.wcnt[w][k];
            }
        }
        uint32_t pair = 0u;
#pragma unroll
        for (int q = 0; q < KPL; ++q) pair += col[q];
        uint32_t incl = pair;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        uint32_t run = incl - pair;
#pragma unroll
        for (int q = 0; q < KPL; ++q) {
            const int k = KPL * lane + q;
            if (k < NK) {
                B.base[k] = run;
#pragma unroll
                for (int w = 0; w < kRows; ++w) {
                    const uint32_t c = B.wcnt[w][k];
                    B.wcnt[w][k] = run;
                    run += c;
                }
            }
        }
    }
    __syncthreads();
    // 3) stable positions
#pragma unroll
    for (int r = 0; r < PER; ++r)
        if (key[r] != (uint32_t)kInvalid)
            B.order[B.wcnt[r * kWarps + warp][key[r]] + rank[r]] =
                (uint16_t)(threadIdx.x + r * kBatch);
    __syncthreads();
}


// Raster CTA -> (slice, tile): through the batch's heaviest-first order
// (tile_order_kernel) when present, else the plain (tile, slice) grid.
__device__ __forceinline__ void raster_cta(const int32_t *__restrict__ tile_order,
                                           int max_tiles, int &s, int &t) {
    if (tile_order) {
        const int i = __ldg(tile_order + blockIdx.x);
        s = i / max_tiles;
        t = i - s * max_tiles;
    } else {
        s = blockIdx.y;
        t = blockIdx.x;
    }
}

// Heaviest-first order of the batch's (slice, tile) CTAs for both raster
// kernels (longest-processing-time-first: the costly tiles start in the
// first waves instead of extending the last one).  One CTA: a histogram
// of the tiles over instance-count buckets (8 per octave), a descending
// scan, then each tile takes a slot of its bucket.  The order within a
// bucket is arbitrary (shared atomics): a CTA's results do not depend on
// when it runs.
__global__ void __launch_bounds__(1024)
tile_order_kernel(const int2 *__restrict__ bin_range, const ugs_slice *__restrict__ slices,
                  int S, int max_tiles, int32_t *__restrict__ order,
                  const PlanHdr *__restrict__ hdr) {
    pdl_entry();
    if (plan_overflow(hdr)) return;
#ifndef UGS_ORDER_SUB
#define UGS_ORDER_SUB 3      // log2 of the buckets per octave of the count
#endif
    constexpr int kSub = UGS_ORDER_SUB;
    constexpr int kNB = (32 << kSub) + 1;
    __shared__ unsigned hist[kNB];
    __shared__ int s_nt[64], s_tb[64];
    for (int b = threadIdx.x; b < kNB; b += blockDim.x) hist[b] = 0u;
    if (threadIdx.x < S) {
        s_nt[threadIdx.x] = slices[threadIdx.x].tiles_x * slices[threadIdx.x].tiles_y;
        s_tb[threadIdx.x] = slices[threadIdx.x].tile_base;
    }
    __syncthreads();
    const int total = S * max_tiles;
    auto bucket = [&](int i) -> unsigned {
        if (i >= total) return 0xffffffffu;
        const int s = i / max_tiles, t = i - s * max_tiles;
        if (t >= s_nt[s]) return 0u;
        const int2 rg = bin_range[s_tb[s] + t];
        const unsigned c = (unsigned)(rg.y - rg.x);
        if (c < (2u << kSub)) return c;
        const int e = 31 - __clz(c);                  // octave (>= kSub + 1)
        return (unsigned)(((e - kSub) << kSub) + ((c >> (e - kSub)) & ((1u << kSub) - 1u)) +
                          (1u << kSub));
    };
    const int lane = threadIdx.x & 31;
    // counts: warp-aggregated (one shared atomic per distinct bucket of a warp)
    for (int i0 = 0; i0 < total; i0 += blockDim.x) {
        const unsigned b = bucket(i0 + threadIdx.x);
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        if (b != 0xffffffffu && lane == __ffs(peers) - 1) atomicAdd(&hist[b], __popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < 32) {   // descending exclusive scan: the heaviest bucket first
        constexpr int kPer = (kNB + 31) / 32;   // lane l: buckets kNB-1-kPer l downwards
        unsigned c[kPer], sum = 0u;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int b = kNB - 1 - (lane * kPer + k);
            c[k] = b >= 0 ? hist[b] : 0u;
            sum += c[k];
        }
        unsigned incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        unsigned run = incl - sum;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const int b = kNB - 1 - (lane * kPer + k);
            if (b >= 0) hist[b] = run;
            run += c[k];
        }
    }
    __syncthreads();
    for (int i0 = 0; i0 < total; i0 += blockDim.x) {
        const int i = i0 + threadIdx.x;
        const unsigned b = bucket(i);
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        const int leader = __ffs(peers) - 1;
        unsigned base = 0u;
        if (b != 0xffffffffu && lane == leader) base = atomicAdd(&hist[b], __popc(peers));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (b != 0xffffffffu) order[base + __popc(peers & ((1u << lane) - 1u))] = i;
    }
}

// Forward.  Records are split by clipped width:
//   narrow (< kWideMin columns): two records per warp, each 16-lane group
//     sweeps its record's rectangle and read-modify-writes its own PRIVATE
//     (num, den) tile buffer in shared memory (XOR-swizzled float2);
//   wide (>= kWideMin columns, ~3/4 of the pixel updates at C3): one record
//     per warp, lane = (tile column X, row parity); every lane keeps the
//     (num, den) of its 8 pixels (X, 2m + parity) in REGISTERS across all of
//     the tile's wide records -- no shared-memory traffic per pair, which is
//     what bounds the narrow path.
// At the end each lane adds its register tile into its group's private
// buffer and the 16 buffers are summed in fixed order -- deterministic,
// because the record -> group / warp assignment is a stable sort.
// four CTAs per SM (the shared-memory count): ptxas takes 60 registers
// (436 vs 441 us at the default 56; (256, 1) lets it take 70: slower)
#ifndef UGS_FWD_MINB
#define UGS_FWD_MINB 4
#endif
__global__ void __launch_bounds__(kRasterThreads, UGS_FWD_MINB)
forward_kernel(const Frag *__restrict__ frag, const uint32_t *__restrict__ vals,
               const int2 *__restrict__ bin_range,
               const ugs_slice *__restrict__ slices,
               const double *__restrict__ bg_raw, float *__restrict__ num_out,
               float *__restrict__ den_out, const PlanHdr *__restrict__ hdr,
               const int32_t *__restrict__ tile_order, int max_tiles) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char smem[];
    if (plan_overflow(hdr)) return;
    Batch &B = *reinterpret_cast<Batch *>(smem);
    // one private (num, den) tile buffer per 16-lane group
    float2 *acc = reinterpret_cast<float2 *>(smem + kFwdAccOff);   // [group][256]
    Frag *raw = reinterpret_cast<Frag *>(smem + kFwdRawOff);      // async-staged batch
    int si, t;
    raster_cta(tile_order, max_tiles, si, t);
    const ugs_slice &sl = slices[si];
    if (t >= sl.tiles_x * sl.tiles_y) return;
    const int tu0 = (t % sl.tiles_x) * kTile, tv0 = (t / sl.tiles_x) * kTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int2 rg = bin_range[sl.tile_base + t];
    StagePipeReg pipe;
    pipe.start(vals, frag, raw, rg.x, rg.y);
    for (int i = threadIdx.x; i < kGroups * kAccStride; i += kRasterThreads)
        acc[i] = make_float2(0.f, 0.f);
    float2 *my = acc + (threadIdx.x >> 4) * kAccStride;
    const int gl16 = lane & 15;
    // wide path: this lane's column and row parity, and its register tile:
    // (num, den) of pixels (X, 2m + ph), m = 2qq + {0, 1} in the two halves
    const int X = lane & 15, ph = lane >> 4;
    const float Xf = (float)X, phf = (float)ph;
    float2 an2[4], ad2[4];
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {
        an2[qq] = make_float2(0.f, 0.f);
        ad2[qq] = make_float2(0.f, 0.f);
    }
    for (int b0 = rg.x; b0 < rg.y; b0 += kBatch) {
        const int nb = min(kBatch, rg.y - b0);
        __syncthreads();
        stage_wait();   // this thread's instance of the batch has landed
        uint32_t key = kKeyInvalid;
        if (threadIdx.x < nb) key = stage_forward(raw[threadIdx.x], B, threadIdx.x);
        // the next batch's gathers overlap this batch's accumulation
        pipe.advance(vals, frag, raw, b0, rg.y);
        // narrow records with equal sweep counts share a warp (two per
        // warp); the wide records follow them
        {
            const uint32_t k1[1] = {key};
            sort_batch<kKeys>(B, k1);
        }
        const int n_narrow = (int)B.base[kKeyWide];
        const int n_valid = (int)B.base[kKeyInvalid];
        for (int s0 = warp * 2; s0 < n_narrow; s0 += kWarps * 2) {
            // the group's next record may touch pixels another lane of the
            // group still updates for this one: every iteration ends with a
            // __syncwarp, so no lane leaves it early (no `continue`)
            const int slot = s0 + (lane >> 4);
            const int j = B.order[slot < n_narrow ? slot : s0];
            const float4 a = B.sA[j], b = B.sB[j];
            const u64 c1 = *reinterpret_cast<const u64 *>(&B.sC[j]);   // (color, 1)
            const int2 kk = *reinterpret_cast<const int2 *>(&B.sC[j].z);
            const int k1 = kk.x, k2 = kk.y;
            const int lx = gl16 & byte_of(k1, 0), ly = gl16 >> byte_of(k1, 1);
            if (slot < n_narrow && lx < byte_of(k2, 2)) {
            const int R = byte_of(k2, 3);   // rows per sweep
            // per lane: x fixed, log2 w = P + y (Q + C y), x and y exact
            const float dx = big_float(lx) - a.x;
            const float P = fmaf(fmaf(b.x, dx, a.z), dx, b.w), Q = fmaf(b.y, dx, a.w);
            float dy = big_float(ly) - a.y;
            const int Y = byte_of(k2, 1) + ly;
            const int sX = (byte_of(k2, 0) + lx) ^ ((Y & 1) << 3);   // swizzled column
            float2 *ptr = my + (Y * kTile + sX);
            // the next row's slot: 16 R for even R; R == 1 flips the swizzle
            // every row, so the step is 16 + 8 or 16 - 8 (bit 3 of sX)
            const int s1 = (R == 1) ? 24 - ((sX & 8) << 1) : R * kTile;
            const int s12 = 2 * R * kTile;   // two rows: the lane's parity again
            // rows ly, ly + R, ... < h, two per iteration (same column: P, Q
            // shared; both loads before both stores, the rows never alias)
            const int nrow = (byte_of(k1, 2) - ly) >> byte_of(k1, 3);
            // the two rows of an iteration in packed f32x2 arithmetic (FFMA2:
            // same fma.rn rounding per half, half the issue slots); scalar
            // operands broadcast, and (num, den) += w * (color, 1) is one
            // FFMA2 per pixel
            float2 dy2 = make_float2(dy, dy + (float)R);
            const float2 C2 = make_float2(b.z, b.z), Q2 = make_float2(Q, Q),
                         P2 = make_float2(P, P);
            const float2 step2 = make_float2((float)(2 * R), (float)(2 * R));
            u64 *pa = reinterpret_cast<u64 *>(ptr), *pb = reinterpret_cast<u64 *>(ptr + s1);
#pragma unroll 1
            for (int pairs = nrow >> 1; pairs > 0; --pairs) {
                const float2 e = __ffma2_rn(dy2, __ffma2_rn(C2, dy2, Q2), P2);
                const float wa = ex2_approx(e.x), wb = ex2_approx(e.y);
                const u64 va = *pa, vb = *pb;
                *pa = ffma2(c1, pack2(wa, wa), va);
                *pb = ffma2(c1, pack2(wb, wb), vb);
                dy2 = __fadd2_rn(dy2, step2);
                pa += s12;
                pb += s12;
            }
            ptr = reinterpret_cast<float2 *>(pa);
            if (nrow & 1) {   // odd row count: the last row
                const float dyl = dy2.x;
                const float wa = ex2_approx(fmaf(dyl, fmaf(b.z, dyl, Q), P));
                u64 *pl = reinterpret_cast<u64 *>(ptr);
                *pl = ffma2(c1, pack2(wa, wa), *pl);
            }
            }
            __syncwarp();
        }
        // wide records: one per warp, all 32 lanes, register accumulation;
        // rows 2m + ph in packed pairs (m = 2q, 2q + 1): FFMA2 / FADD2
        for (int q = n_narrow + warp; q < n_valid; q += kWarps) {
            const int j = B.order[q];
            const float4 a = B.sA[j], b = B.sB[j], c = B.sC[j];
            const int xw = __float_as_int(c.y), masks = __float_as_int(c.z);
            const float dx = Xf - a.x;                    // exact small integers
            float P = fmaf(fmaf(b.x, dx, a.z), dx, b.w);
            const float Q = fmaf(b.y, dx, a.w);
            P = (unsigned)(X - (xw & 0xff)) < (unsigned)(xw >> 8) ? P : -INFINITY;
            const unsigned vm = (unsigned)byte_of(masks, ph);
            // provably warp-uniform (a lane-0 broadcast), so the row-pair
            // skips compile to uniform branches without reconvergence barriers
            const unsigned um = (unsigned)__shfl_sync(0xffffffffu, masks, 0) >> 16;
            const float dyb = phf - a.y;                  // row ph (m = 0)
            float2 dy2 = make_float2(dyb, dyb + 2.0f);
            const float2 P2 = make_float2(P, P), Q2 = make_float2(Q, Q),
                         C2 = make_float2(b.z, b.z), col2 = make_float2(c.x, c.x);
            const float2 four = make_float2(4.0f, 4.0f);
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
                if (um & (3u << (2 * qq))) {                 // warp-uniform
                    const float2 e = __ffma2_rn(dy2, __ffma2_rn(C2, dy2, Q2), P2);
                    float2 wv = make_float2(ex2_approx(e.x), ex2_approx(e.y));
                    wv.x = (vm & (1u << (2 * qq))) ? wv.x : 0.f;
                    wv.y = (vm & (2u << (2 * qq))) ? wv.y : 0.f;
                    an2[qq] = __ffma2_rn(wv, col2, an2[qq]);
                    ad2[qq] = __fadd2_rn(ad2[qq], wv);
                }
                dy2 = __fadd2_rn(dy2, four);
            }
        }
    }
    __syncthreads();
    // the register tiles join the group buffers (each lane owns distinct
    // pixels of its group's buffer), then the fixed-order sum
#pragma unroll
    for (int m = 0; m < 8; ++m) {
        const int p = acc_swizzle((2 * m + ph) * kTile + X);
        float2 v = my[p];
        v.x += (m & 1) ? an2[m >> 1].y : an2[m >> 1].x;
        v.y += (m & 1) ? ad2[m >> 1].y : ad2[m >> 1].x;
        my[p] = v;
    }
    __syncthreads();
    const int u = tu0 + (threadIdx.x & 15), v = tv0 + (threadIdx.x >> 4);
    if (u < sl.width && v < sl.height) {
        float n = 0.f, d = 0.f;
        const int sp = acc_swizzle(threadIdx.x);
#pragma unroll
        for (int g = 0; g < kGroups; ++g) {
            const float2 q = acc[g * kAccStride + sp];
            n += q.x;
            d += q.y;
        }
        const float abg = sigmoid_bg(bg_raw, 1), cbg = sigmoid_bg(bg_raw, 0);
        const int64_t p = sl.pix_base + (int64_t)v * sl.width + u;
        const float nn = n + abg * cbg, dd = d + abg;
        if (den_out) {
            num_out[p] = nn;
            den_out[p] = dd;
        } else {   // render mode (ugs_render): clip(num / den, 0, 1), NaN kept
            const float q = __fdiv_rn(nn, dd);
            num_out[p] = q < 0.f ? 0.f : (q > 1.f ? 1.f : q);
        }
    }
}

// Strict-order variant: every pixel walks the tile's list in ascending
// Gaussian order, one f32 add per pair (the reference's sequential loop).
__global__ void __launch_bounds__(kRasterThreads)
forward_ordered_kernel(const Frag *__restrict__ frag, const uint32_t *__restrict__ vals,
                       const int2 *__restrict__ bin_range,
                       const ugs_slice *__restrict__ slices,
                       const double *__restrict__ bg_raw, float *__restrict__ num_out,
                       float *__restrict__ den_out, const PlanHdr *__restrict__ hdr) {
    pdl_entry();
    __shared__ float4 s0[kBatch], s1[kBatch];
    __shared__ float2 s2[kBatch];   // (rectangle bits, colour)
    if (plan_overflow(hdr)) return;
    const ugs_slice &sl = slices[blockIdx.y];
    const int t = blockIdx.x;
    if (t >= sl.tiles_x * sl.tiles_y) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // warp owns an 8 x 4 block so whole warps skip records that miss it
    const int wx0 = (warp & 1) * 8, wy0 = (warp >> 1) * 4;   // tile-relative
    const int x = wx0 + (lane & 7), y = wy0 + (lane >> 3);
    const int u = (t % sl.tiles_x) * kTile + x, v = (t / sl.tiles_x) * kTile + y;
    const int2 rg = bin_range[sl.tile_base + t];
    const float fx = (float)x, fy = (float)y;
    float num = 0.f, den = 0.f;
    for (int b0 = rg.x; b0 < rg.y; b0 += kBatch) {
        const int nb = min(kBatch, rg.y - b0);
        __syncthreads();
        if (threadIdx.x < nb) {
            const Frag f = frag[__ldg(vals + b0 + threadIdx.x)];
            const FragRect r = frag_rect(f.q1.w);
            s0[threadIdx.x] = make_float4((float)r.pu, (float)r.pv, f.q1.x, f.q1.y);
            s1[threadIdx.x] = make_float4(f.q0.x, f.q0.y, f.q0.z, f.q1.z);
            s2[threadIdx.x] = make_float2(f.q1.w, f.q0.w);
        }
        __syncthreads();
        for (int j = 0; j < nb; ++j) {
            const float2 r2 = s2[j];
            const FragRect r = frag_rect(r2.x);
            if (r.x0 > wx0 + 7 || r.x1 < wx0 || r.y0 > wy0 + 3 || r.y1 < wy0) continue;
            const float4 r0 = s0[j], r1 = s1[j];
            const float dx = fx - r0.x, dy = fy - r0.y;   // exact integers
            const float e = fmaf(fmaf(r1.x, dx, fmaf(r1.y, dy, r0.z)), dx,
                                 fmaf(fmaf(r1.z, dy, r0.w), dy, r1.w));
            float w = ex2_approx(e);
            const bool in = (unsigned)(x - r.x0) <= (unsigned)(r.x1 - r.x0) &&
                            (unsigned)(y - r.y0) <= (unsigned)(r.y1 - r.y0);
            w = in ? w : 0.f;
            num = fmaf(w, r2.y, num);
            den += w;
        }
    }
    if (u < sl.width && v < sl.height) {
        const float abg = sigmoid_bg(bg_raw, 1), cbg = sigmoid_bg(bg_raw, 0);
        const int64_t p = sl.pix_base + (int64_t)v * sl.width + u;
        num_out[p] = num + abg * cbg;
        den_out[p] = den + abg;
    }
}


// Transpose-reduce of 8 values across a 2-lane group (one level, 4
// shuffles): on return group lane g holds the group totals of values 4g ..
// 4g + 3.
__device__ __forceinline__ float4 group_reduce8x2(const float a[8]) {
    const bool h1 = threadIdx.x & 1;
    float b[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float send = h1 ? a[k] : a[k + 4];
        const float keep = h1 ? a[k + 4] : a[k];
        b[k] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
    return make_float4(b[0], b[1], b[2], b[3]);
}

__global__ void __launch_bounds__(kRasterThreads, 4)
backward_kernel(const Frag *__restrict__ frag, const uint32_t *__restrict__ vals,
                const int2 *__restrict__ bin_range,
                const ugs_slice *__restrict__ slices,
                const float *__restrict__ num_in, const float *__restrict__ den_in,
                const float *__restrict__ dpix, const double *__restrict__ bg_raw,
                float *__restrict__ partial, float2 *__restrict__ bin_bg,
                const PlanHdr *__restrict__ hdr,
                const int32_t *__restrict__ tile_order, int max_tiles) {
    // the binning outputs (ranges, ids, Frags) are an earlier stage's: the
    // first batch's gathers start before the wait for the loss
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem[];
    if (plan_overflow(hdr)) return;
    BwdBatch &B = *reinterpret_cast<BwdBatch *>(smem);
    Layout &Ly = *reinterpret_cast<Layout *>(smem + kBwdLyOff);
    // per-pixel upstream terms as two planes (a lane's two streams load
    // straight into a register pair): G, then G chat
    float *pixG = reinterpret_cast<float *>(smem + kBwdPixOff);
    float *pixGc = pixG + kBPlane;
    float2 *s_bg = reinterpret_cast<float2 *>(pixGc + kBPlane);
    Frag *raw = reinterpret_cast<Frag *>(smem + kBwdRawOff);      // async-staged batch
    int si, t;
    raster_cta(tile_order, max_tiles, si, t);
    const ugs_slice &sl = slices[si];
    if (t >= sl.tiles_x * sl.tiles_y) return;
    const int tu0 = (t % sl.tiles_x) * kTile, tv0 = (t / sl.tiles_x) * kTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int2 rg = bin_range[sl.tile_base + t];
    // the first batch lands while the pixel terms load
    uint32_t *pipe_ids = reinterpret_cast<uint32_t *>(smem + kBwdIdsOff);
    StagePipe pipe(pipe_ids, pipe_ids + kBwdBatch);
    pipe.start(vals, frag, raw, rg.x, rg.y);
    pdl_wait();   // the loss's upstream terms
    {   // per-pixel upstream terms: G = dpix/ssum, Gc = G * chat, chat = num/ssum
        const int u = tu0 + (threadIdx.x & 15), v = tv0 + (threadIdx.x >> 4);
        float G = 0.f, Gc = 0.f, Gb = 0.f;
        if (u < sl.width && v < sl.height) {
            const int64_t p = sl.pix_base + (int64_t)v * sl.width + u;
            const float ssum = den_in[p];
            const float chat = __fdiv_rn(num_in[p], ssum);
            G = __fdiv_rn(dpix[p], ssum);
            Gc = G * chat;
            // background opacity term dpix*(c_bg - chat)/ssum, per pixel as the
            // reference forms it (gradients.py:110), no cancellation
            Gb = G * (sigmoid_bg(bg_raw, 0) - chat);
        }
        pixG[(threadIdx.x >> 4) * kBP + (threadIdx.x & 15)] = G;
        pixGc[(threadIdx.x >> 4) * kBP + (threadIdx.x & 15)] = Gc;
        float a = G, c = Gb;   // background partials of this tile, fixed order
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (lane == 0) s_bg[warp] = make_float2(a, c);
    }
    for (int b0 = rg.x; b0 < rg.y; b0 += kBwdBatch) {
        const int nb = min(kBwdBatch, rg.y - b0);
        __syncthreads();
        stage_wait();   // this thread's instances of the batch have landed
        uint32_t key[kBwdPer];
#pragma unroll
        for (int r = 0; r < kBwdPer; ++r) {
            const int sl = (int)threadIdx.x + r * kBatch;
            key[r] = sl < nb ? (uint32_t)stage_record2(raw[sl], pipe.cur[sl], B, Ly, sl)
                             : (uint32_t)kBwdKeyInvalid;
        }
        pipe.advance(vals, frag, raw, b0, rg.y);   // next batch, during this one
        sort_batch<kBwdKeys>(B, key);
        // sixteen records per warp (2-lane groups); every lane takes part in
        // the shuffles, empty lanes carry zeros
        const int nunits = (nb + 15) >> 4;
        for (int u = next_unit(&B.next[0], nunits); u >= 0; u = next_unit(&B.next[0], nunits)) {
            const int s0 = u * 16;
            const int slot = s0 + (lane >> 1);
            const bool live = slot < nb;
            const int j = live ? B.order[slot] : B.order[s0];
            const float4 a = B.sA[j], b = B.sB[j], c = B.sC[j];
            const int2 lm = Ly.sLM[j];
            const int Lx = byte_of(lm.x, 0), Lz = byte_of(lm.x, 1), Lw = byte_of(lm.x, 2);
            const int Mx = byte_of(lm.y, 0), Mz = byte_of(lm.y, 2), Mw = byte_of(lm.y, 3);
            const int gl = lane & 1;
            const int h = live ? byte_of(lm.y, 1) : 0;
            const int ls = __float_as_int(c.y), stride = 1 << ls;
            const int npass = __float_as_int(c.z);   // 4-column strips
            const float2 C2 = make_float2(b.z, b.z), c2 = make_float2(c.x, c.x);
            const float2 fs2 = make_float2((float)stride, (float)stride);
            float m[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
            for (int pass = 0; pass < npass; ++pass) {
                // the two pixel streams of stage_record2
                const int lxA = (gl & Lx) + 4 * pass, lyA = gl >> Lx;
                const int lxB = lxA + Lz, lyB = lyA + Lw;
                const bool okA = lxA < Mx && lyA < h, okB = lxB < Mx && lyB < h;
                const int nA = okA ? (h - lyA + stride - 1) >> ls : 0;
                // column layouts always pair A with B (B masked when out of
                // the rectangle)
                const int nB = okB ? (h - lyB + stride - 1) >> ls : (Lz ? nA : 0);
                // per lane dx is fixed per stream: log2 w = P + dy (Q + C dy);
                // the x moments follow from the per-stream sums (sum t dx =
                // dx S0, ...)
                const float dxA = big_float(lxA) - a.x, dxB = dxA + (float)Lz;
                const float PA = fmaf(fmaf(b.x, dxA, a.z), dxA, b.w), QA = fmaf(b.y, dxA, a.w);
                const float PB = okB ? fmaf(fmaf(b.x, dxB, a.z), dxB, b.w) : -INFINITY;
                const float QB = fmaf(b.y, dxB, a.w);
                const float dyA0 = big_float(lyA) - a.y;
                const float *gA = pixG + (Mw + lyA) * kBP + Mz + lxA;
                const float *gB = okB ? gA + (Lw * kBP + Lz) : gA;
                const int gstep = okB ? stride * kBP : 0;
                // the G chat plane sits kBPlane floats after the G plane
                // streams A and B in packed f32x2 arithmetic (FFMA2 / FADD2 /
                // FMUL2, per-half fma.rn rounding): lo = A, hi = B
                float2 dy2 = make_float2(dyA0, dyA0 + (float)Lw);
                const float2 P2 = make_float2(PA, PB), Q2 = make_float2(QA, QB);
                float2 m02 = make_float2(0.f, 0.f), S02 = m02, Sy2 = m02, Syy2 = m02;
                int i = 0;
#pragma unroll 1
                for (; i < nB; ++i) {
                    const float2 e = __ffma2_rn(dy2, __ffma2_rn(C2, dy2, Q2), P2);
                    const float2 w2 = make_float2(ex2_approx(e.x), ex2_approx(e.y));
                    const float2 gx = make_float2(gA[0], gB[0]);
                    const float2 gy = make_float2(-gA[kBPlane], -gB[kBPlane]);
                    const float2 t2 = __fmul2_rn(__ffma2_rn(gx, c2, gy), w2);   // dw * w
                    m02 = __ffma2_rn(gx, w2, m02);
                    S02 = __fadd2_rn(S02, t2);
                    const float2 ty2 = __fmul2_rn(t2, dy2);
                    Sy2 = __fadd2_rn(Sy2, ty2);
                    Syy2 = __ffma2_rn(ty2, dy2, Syy2);
                    dy2 = __fadd2_rn(dy2, fs2);
                    gA += stride * kBP;
                    gB += gstep;
                }
                float m0 = m02.x + m02.y;
                float S0a = S02.x, Sya = Sy2.x, Syya = Syy2.x;
                const float S0b = S02.y, Syb = Sy2.y, Syyb = Syy2.y;
                if (i < nA) {   // narrow tail: one more row of stream A
                    const float dyA = dy2.x;
                    const float wa = ex2_approx(fmaf(dyA, fmaf(b.z, dyA, QA), PA));
                    const float ga = gA[0];
                    const float ta = fmaf(ga, c.x, -gA[kBPlane]) * wa;
                    m0 = fmaf(ga, wa, m0);
                    S0a += ta;
                    const float tya = ta * dyA;
                    Sya += tya;
                    Syya = fmaf(tya, dyA, Syya);
                }
                m[0] += m0;
                m[1] += S0a + S0b;
                m[2] += fmaf(dxA, S0a, dxB * S0b);
                m[3] += Sya + Syb;
                m[4] += fmaf(dxA * dxA, S0a, dxB * dxB * S0b);
                m[5] += fmaf(dxA, Sya, dxB * Syb);
                m[6] += Syya + Syyb;
            }
            const float4 red = group_reduce8x2(m);
#if UGS_V8_BWD
            // the pair's second half to its first lane: one 32-byte store
            const float4 hi = make_float4(__shfl_down_sync(0xffffffffu, red.x, 1),
                                          __shfl_down_sync(0xffffffffu, red.y, 1),
                                          __shfl_down_sync(0xffffffffu, red.z, 1),
                                          __shfl_down_sync(0xffffffffu, red.w, 1));
            if (live && gl == 0)
                st_v8(partial + (size_t)(uint32_t)__float_as_int(c.w) * 8, red, hi);
#else
            if (live)
                *reinterpret_cast<float4 *>(
                    partial + (size_t)(uint32_t)__float_as_int(c.w) * 8 + 4 * gl) = red;
#endif
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            acc.x += s_bg[w].x;
            acc.y += s_bg[w].y;
        }
        bin_bg[sl.tile_base + t] = acc;
    }
}

// The closed-form float64 chain of one record from its summed moments Sm
// (about the record's reference pixel): raw-parameter gradients o[11].
__device__ __forceinline__ void record_chain(const Rec &R, const float lr[6],
                                             const float muf[3], const ugs_slice &sl,
                                             const double Sm[7], float beta, float o[11]) {
    const int uv = __float_as_int(R.r1.w), ui = uv & 0xffff, vi = uv >> 16;
    // build_L (model.py:101-118): diagonal f32(l^2) + f32(beta)
    const double L00 = __fadd_rn(__fmul_rn(lr[0], lr[0]), beta);
    const double L11 = __fadd_rn(__fmul_rn(lr[1], lr[1]), beta);
    const double L22 = __fadd_rn(__fmul_rn(lr[2], lr[2]), beta);
    const double mu[3] = {muf[0], muf[1], muf[2]};
    const double du[3] = {sl.du[0], sl.du[1], sl.du[2]};
    const double dv[3] = {sl.dv[0], sl.dv[1], sl.dv[2]};
    const double cu = (double)ui, cv = (double)vi;
    double es[3];
    for (int k = 0; k < 3; ++k)
        es[k] = ((double)sl.origin[k] - mu[k]) + cu * du[k] + cv * dv[k];
    const double Tc = Sm[0], S0 = Sm[1], Sx = Sm[2], Sy = Sm[3], Sxx = Sm[4],
                 Sxy = Sm[5], Syy = Sm[6];
    double V[3], wv[3];
    for (int k = 0; k < 3; ++k) {
        wv[k] = Sx * du[k] + Sy * dv[k];
        V[k] = S0 * es[k] + wv[k];
    }
    double Mm[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            Mm[i][j] = S0 * es[i] * es[j] + es[i] * wv[j] + wv[i] * es[j] +
                       Sxx * du[i] * du[j] + Sxy * (du[i] * dv[j] + dv[i] * du[j]) +
                       Syy * dv[i] * dv[j];
    const double L[3][3] = {{L00, 0.0, 0.0},
                            {(double)lr[3], L11, 0.0},
                            {(double)lr[4], (double)lr[5], L22}};
    double LtV[3];
    for (int k = 0; k < 3; ++k) LtV[k] = L[0][k] * V[0] + L[1][k] * V[1] + L[2][k] * V[2];
    for (int i = 0; i < 3; ++i)
        o[i] = (float)(L[i][0] * LtV[0] + L[i][1] * LtV[1] + L[i][2] * LtV[2]);
    auto dL = [&](int i, int j) {
        return -(Mm[i][0] * L[0][j] + Mm[i][1] * L[1][j] + Mm[i][2] * L[2][j]);
    };
    o[3] = (float)(dL(0, 0) * 2.0 * (double)lr[0]);   // L_jj = l_jj^2 + beta
    o[4] = (float)(dL(1, 1) * 2.0 * (double)lr[1]);
    o[5] = (float)(dL(2, 2) * 2.0 * (double)lr[2]);
    o[6] = (float)dL(1, 0);
    o[7] = (float)dL(2, 0);
    o[8] = (float)dL(2, 1);
    const double c = R.r0.w, a = R.r1.z;
    o[9] = (float)(Tc * c * (1.0 - c));
    o[10] = (float)(S0 * (1.0 - a));   // (S0 / a) * a (1 - a)
}

// Raw-parameter gradients of one record (ref gradients.py:84-103): sum its
// instance partials in order (moments in the integer offsets from the
// record's reference pixel), then with e* = e(reference pixel),
// V = S0 e* + Sx du + Sy dv and
// M = S0 e*e*^T + e* w^T + w e*^T + Sxx du du^T + Sxy (du dv^T + dv du^T)
//     + Syy dv dv^T  (w = Sx du + Sy dv, dq = -t/2):
//   d_mu = Lambda V,  d_L = -(M L) lower,  d_c = Tc,  d_a = S0 / alpha.
// o = [d_mu 3 | d_l_raw 6 | d_c_raw | d_a_raw].
__device__ __forceinline__ void record_grad(int64_t r, const ugs_slice &sl,
                                            const Rec *__restrict__ rec,
                                            const int32_t *__restrict__ rec_gid,
                                            const int32_t *__restrict__ rec_inst,
                                            const float *__restrict__ partial,
                                            const float *__restrict__ means,
                                            const float *__restrict__ l_raw, float beta,
                                            float o[11]) {
    // instance moments are about each instance's expansion pixel; shift them
    // (float64, exact integer offsets) to the record's reference pixel
#if UGS_V8
    Rec R;
    ld_v8(rec + r, R.r0, R.r1);
#else
    const Rec R = rec[r];
#endif
    // the Gaussian's parameters are loaded before the instance loop, so
    // their round trip overlaps the partials' instead of following it
    const int64_t g = rec_gid[r];
    const float lr[6] = {__ldg(l_raw + 6 * g), __ldg(l_raw + 6 * g + 1),
                         __ldg(l_raw + 6 * g + 2), __ldg(l_raw + 6 * g + 3),
                         __ldg(l_raw + 6 * g + 4), __ldg(l_raw + 6 * g + 5)};
    const float muf[3] = {__ldg(means + 3 * g), __ldg(means + 3 * g + 1),
                          __ldg(means + 3 * g + 2)};
    const int wub = __float_as_int(R.r1.x), wvb = __float_as_int(R.r1.y);
    const int iu0 = wub & 0xffff, iu1 = wub >> 16, iv0 = wvb & 0xffff, iv1 = wvb >> 16;
    const int uv = __float_as_int(R.r1.w), ui = uv & 0xffff, vi = uv >> 16;
    const int tx0 = iu0 >> 4, tx1 = iu1 >> 4;
    double Sm[7] = {0, 0, 0, 0, 0, 0, 0};
    const int i0 = rec_inst[r], i1 = rec_inst[r + 1];
    int tx = tx0, ty = iv0 >> 4;
#ifndef UGS_FIN_UNROLL
#define UGS_FIN_UNROLL 2
#endif
#if UGS_FIN_UNROLL > 1
#define UGS_STR_(x) #x
#define UGS_UNROLL_(n) _Pragma(UGS_STR_(unroll n))
    UGS_UNROLL_(UGS_FIN_UNROLL)
#endif
    for (int i = i0; i < i1; ++i) {
        const TileRect t = tile_rect(iu0, iu1, iv0, iv1, tx * kTile, ty * kTile, ui, vi);
        const double ox = (double)(t.pu - ui), oy = (double)(t.pv - vi);
        if (++tx > tx1) { tx = tx0; ++ty; }
#if UGS_V8
        float4 pa, pb;
        ld_v8(partial + (size_t)i * 8, pa, pb);
#else
        const float4 pa = *reinterpret_cast<const float4 *>(partial + (size_t)i * 8);
        const float4 pb = *reinterpret_cast<const float4 *>(partial + (size_t)i * 8 + 4);
#endif
        const double s0 = pa.y, sx = pa.z, sy = pa.w;
        Sm[0] += pa.x;
        Sm[1] += s0;
        Sm[2] += sx + ox * s0;
        Sm[3] += sy + oy * s0;
        Sm[4] += (double)pb.x + ox * (2.0 * sx + ox * s0);
        Sm[5] += (double)pb.y + ox * sy + oy * sx + ox * oy * s0;
        Sm[6] += (double)pb.z + oy * (2.0 * sy + oy * s0);
    }
    record_chain(R, lr, muf, sl, Sm, beta, o);
}

// One thread per record: its raw-parameter gradient (float64 chain) into
// rgrad[r][0..10] (AoS-12 row), for the staged update below.
#ifndef UGS_FIN_MINB
#define UGS_FIN_MINB 6   // with the two-instance unroll below (variant sweep: 95 -> 92 us)
#endif
__global__ void __launch_bounds__(128, UGS_FIN_MINB)
finalize_records_kernel(const Rec *__restrict__ rec, const int32_t *__restrict__ rec_gid,
                        const int32_t *__restrict__ rec_inst,
                        const float *__restrict__ partial, const PlanHdr *__restrict__ hdr,
                        const int64_t *__restrict__ slice_base, int S,
                        const ugs_slice *__restrict__ slices,
                        const float *__restrict__ means, const float *__restrict__ l_raw,
                        float beta, float *__restrict__ rgrad) {
    pdl_entry();
    // the slices' record bases in shared memory: the per-thread slice search
    // runs on it instead of on dependent global loads
    __shared__ int64_t s_rb[64];
    if (plan_overflow(hdr)) return;
    const int64_t m_total = (int64_t)hdr->m;
    if ((int64_t)blockIdx.x * blockDim.x >= m_total) return;   // whole block
    for (int q = threadIdx.x; q < S; q += blockDim.x) s_rb[q] = slice_base[2 * q];
    __syncthreads();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m_total) return;
    int s = 0;
    for (int step = 32; step > 0; step >>= 1)   // last slice whose base <= r
        if (s + step < S && s_rb[s + step] <= r) s += step;
    float o[11];
    record_grad(r, slices[s], rec, rec_gid, rec_inst, partial, means, l_raw, beta, o);
    float4 *dst = reinterpret_cast<float4 *>(rgrad + (size_t)r * kG);
    dst[0] = make_float4(o[0], o[1], o[2], o[3]);
    dst[1] = make_float4(o[4], o[5], o[6], o[7]);
    dst[2] = make_float4(o[8], o[9], o[10], 0.f);
}

constexpr int kUpdThreads = 256;
constexpr int kUpdWarps = kUpdThreads / 32;
constexpr int kUpdRows = 64;    // staged record-gradient rows per warp and pass

// Every WARP works alone on its 32 Gaussians (the count pass's warp ->
// Gaussian mapping), synchronising only with __syncwarp, so one warp's
// memory round trips overlap the others' instead of meeting at block
// barriers.  For every slice of the batch the accept ballot says which of
// the warp's Gaussians have a record; those records are consecutive from
// warp_rec.  The warp stages its record-gradient rows (finalize_records) in
// shared memory with parallel loads -- one round trip per pass of up to 64
// rows -- then each lane adds its Gaussian's rows in SLICE ORDER,
// acc = fma(scale, row, acc): deterministic, no atomics.  Then (adam != 0,
// single GPU) densify statistics and Adam run for EVERY Gaussian --
// zero-gradient rows still move (trainer.py:182-199) -- and the dense
// gradient never touches HBM; or (adam == 0) the rows are added into the
// dense AoS-12 buffer; or (adam == 2, the multi-GPU step) every row of the
// dense buffer is WRITTEN -- the scaled sum, zeros for Gaussians no slice
// accepted, the pad slot = accepted -- so the caller neither zeroes nor
// reads it first.
#ifndef UGS_UPD_MINB
#define UGS_UPD_MINB 4
#endif
__global__ void __launch_bounds__(kUpdThreads, UGS_UPD_MINB)
update_gather_kernel(const uint32_t *__restrict__ amask, const int32_t *__restrict__ warp_rec,
                     const float *__restrict__ rgrad, int S, int64_t nwarp_all, int64_t n,
                     float scale, int adam, float *__restrict__ grad,
                     uint8_t *__restrict__ touched, CloudMut p, float *__restrict__ m,
                     float *__restrict__ v, AdamConst k, float *__restrict__ grad_sum,
                     int32_t *__restrict__ grad_cnt, int aligned,
                     const PlanHdr *__restrict__ hdr) {
    // the accept words and record bases are the binning's: read before the
    // wait for finalize's record gradients
    pdl_trigger();
    __shared__ float4 rows_all[kUpdWarps][kUpdRows][3];
    if (plan_overflow(hdr)) return;
    __shared__ float4 prm_all[kUpdWarps][24 + 48];   // means | l_raw rows of the warp
    __shared__ uint32_t word_all[kUpdWarps][64];
    __shared__ int off_all[kUpdWarps][65], base_all[kUpdWarps][64];
    __shared__ uint8_t rs_all[kUpdWarps][kUpdRows];   // row -> slice of a pass
    const int64_t g = (int64_t)blockIdx.x * kUpdThreads + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * kUpdWarps + warp;
    if (gw >= nwarp_all) return;   // whole warp
    float4(*rows)[3] = rows_all[warp];
    uint32_t *s_word = word_all[warp];
    int *s_off = off_all[warp], *s_base = base_all[warp];
    uint8_t *s_rs = rs_all[warp];
    const uint32_t lt = (1u << lane) - 1u;
    const int mode = adam;
    adam = mode == 1;
    if (adam && g < n) {
        // the update's streams (moments, parameters) start towards L2 while
        // the gather runs: no registers held, the latency overlaps
        asm volatile("prefetch.global.L2 [%0];" ::"l"(m + kG * g));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(v + kG * g));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p.l_raw + 6 * g));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(p.means + 3 * g));
    }
    // slice words, record bases and the exclusive prefix of the warp's rows
    // over the slices (lane s handles slice s; S <= 64: two rounds)
    int total = 0;
    for (int sw = 0; sw < S; sw += 32) {
        const int sl = sw + lane;
        uint32_t w = 0;
        if (sl < S) {
            // both loads in flight together (the record base is only used
            // when the word has bits; the entry exists either way)
            const int32_t wr = __ldg(warp_rec + (size_t)sl * nwarp_all + gw);
            w = __ldg(amask + (size_t)sl * nwarp_all + gw);
            s_word[sl] = w;
            s_base[sl] = w ? wr : 0;
        }
        const int c = __popc(w);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (sl < S) s_off[sl] = total + incl - c;
        total += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_off[S] = total;
    __syncwarp();
    pdl_wait();
    float acc[11];
#pragma unroll
    for (int j = 0; j < 11; ++j) acc[j] = 0.f;
    bool hit = false;
    int sfirst = 0;   // first slice with rows at or after `base`
    // passes of up to kUpdRows rows in slice order (a lane's rows ascend
    // with the slice, so every lane still accumulates in slice order)
    for (int base = 0; base < total; base += kUpdRows) {
        const int nr = min(kUpdRows, total - base);
        while (s_off[sfirst + 1] <= base) ++sfirst;
        int slast = sfirst;   // last slice with rows before base + nr
        while (slast + 1 < S && s_off[slast + 1] < base + nr) ++slast;
        // row -> slice table of this pass (each slice's rows are one run)
        for (int sl = sfirst + lane; sl <= slast; sl += 32) {
            const int r0 = max(s_off[sl], base), r1 = min(s_off[sl + 1], base + nr);
            for (int i = r0; i < r1; ++i) s_rs[i - base] = (uint8_t)sl;
        }
        __syncwarp();
        {   // the rows as a flat float4 stream (each slice's rows are
            // consecutive records): coalesced, all loads before the stores
            constexpr int kPer = kUpdRows * 3 / 32;
            const float4 *src4 = reinterpret_cast<const float4 *>(rgrad);
            float4 *dst4 = &rows[0][0];
            float4 t[kPer];
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const int f = lane + 32 * j;
                if (f < 3 * nr) {
                    const int i = f / 3;
                    const int sl = s_rs[i];
                    const int64_t r = (int64_t)s_base[sl] + (base + i - s_off[sl]);
                    t[j] = __ldg(src4 + 3 * (size_t)r + (f - 3 * i));
                }
            }
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const int f = lane + 32 * j;
                if (f < 3 * nr) dst4[f] = t[j];
            }
        }
        __syncwarp();
        for (int sl = sfirst; sl <= slast; ++sl) {
            const uint32_t word = s_word[sl];
            if (!((word >> lane) & 1u)) continue;
            const int slot = s_off[sl] + __popc(word & lt) - base;
            if (slot < 0 || slot >= nr) continue;
            const float4 t0 = rows[slot][0], t1 = rows[slot][1], t2 = rows[slot][2];
            const float o[11] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w,
                                 t2.x, t2.y, t2.z};
#pragma unroll
            for (int j = 0; j < 11; ++j) acc[j] = fmaf(scale, o[j], acc[j]);
            hit = true;
        }
        __syncwarp();   // rows / s_rs reused by the next pass
    }
    const int64_t g0 = gw * 32;
    if (adam && aligned && g0 + 32 <= n) {
        // full warp: the warp's moment rows (2 x 1536 B) and parameter rows
        // (means 384 B, l_raw 768 B) move as coalesced float4 streams through
        // shared memory instead of 48 / 12 / 24-byte strided per-lane rows
        float4 *mv = &rows[0][0];   // [0, 96) m, [96, 192) v
        float4 *pm = prm_all[warp];  // [0, 24) means, [24, 72) l_raw
        const float4 *gm = reinterpret_cast<const float4 *>(m + kG * g0);
        const float4 *gv = reinterpret_cast<const float4 *>(v + kG * g0);
        const float4 *gmu = reinterpret_cast<const float4 *>(p.means + 3 * g0);
        const float4 *gl = reinterpret_cast<const float4 *>(p.l_raw + 6 * g0);
        float4 a[3], b[3], c0, c1, c2 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            a[j] = gm[lane + 32 * j];
            b[j] = gv[lane + 32 * j];
        }
        c0 = lane < 24 ? gmu[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
        c1 = gl[lane];
        if (lane < 16) c2 = gl[32 + lane];
        float pr[11];
        pr[9] = p.intensity_raw[g];
        pr[10] = p.opacity_raw[g];
        const bool stats = hit && grad_sum;
        float gs = 0.f;
        int32_t gc = 0;
        if (stats) {
            gs = grad_sum[g];
            gc = grad_cnt[g];
        }
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            mv[lane + 32 * j] = a[j];
            mv[96 + lane + 32 * j] = b[j];
        }
        if (lane < 24) pm[lane] = c0;
        pm[24 + lane] = c1;
        if (lane < 16) pm[56 + lane] = c2;
        __syncwarp();
        float mm[kG], vv[kG];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const float4 x = mv[3 * lane + q], y = mv[96 + 3 * lane + q];
            mm[4 * q] = x.x; mm[4 * q + 1] = x.y; mm[4 * q + 2] = x.z; mm[4 * q + 3] = x.w;
            vv[4 * q] = y.x; vv[4 * q + 1] = y.y; vv[4 * q + 2] = y.z; vv[4 * q + 3] = y.w;
        }
        float *pf = reinterpret_cast<float *>(pm);
#pragma unroll
        for (int q = 0; q < 3; ++q) pr[q] = pf[3 * lane + q];
#pragma unroll
        for (int q = 0; q < 6; ++q) pr[3 + q] = pf[96 + 6 * lane + q];
        float gr[kG];
#pragma unroll
        for (int j = 0; j < 11; ++j) gr[j] = acc[j];
        gr[11] = 0.f;
        adam_row(gr, pr, mm, vv, k);
        __syncwarp();   // every lane has read its rows
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            mv[3 * lane + q] = make_float4(mm[4 * q], mm[4 * q + 1], mm[4 * q + 2], mm[4 * q + 3]);
            mv[96 + 3 * lane + q] =
                make_float4(vv[4 * q], vv[4 * q + 1], vv[4 * q + 2], vv[4 * q + 3]);
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) pf[3 * lane + q] = pr[q];
#pragma unroll
        for (int q = 0; q < 6; ++q) pf[96 + 6 * lane + q] = pr[3 + q];
        p.intensity_raw[g] = pr[9];
        p.opacity_raw[g] = pr[10];
        if (stats) {
            grad_sum[g] = __fadd_rn(gs, norm3_f32(gr[0], gr[1], gr[2]));
            grad_cnt[g] = gc + 1;
        }
        __syncwarp();
        float4 *wm = reinterpret_cast<float4 *>(m + kG * g0);
        float4 *wv = reinterpret_cast<float4 *>(v + kG * g0);
        float4 *wmu = reinterpret_cast<float4 *>(p.means + 3 * g0);
        float4 *wl = reinterpret_cast<float4 *>(p.l_raw + 6 * g0);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            wm[lane + 32 * j] = mv[lane + 32 * j];
            wv[lane + 32 * j] = mv[96 + lane + 32 * j];
        }
        if (lane < 24) wmu[lane] = pm[lane];
        wl[lane] = pm[24 + lane];
        if (lane < 16) wl[32 + lane] = pm[56 + lane];
        return;
    }
    if (g >= n) return;
    if (adam) {
        float gr[kG];
#pragma unroll
        for (int j = 0; j < 11; ++j) gr[j] = acc[j];
        gr[11] = 0.f;
        adam_gaussian(g, gr, m + kG * g, v + kG * g, p, k, hit, grad_sum, grad_cnt);
    } else if (mode == 2) {
        float4 *row = reinterpret_cast<float4 *>(grad + kG * g);
        row[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        row[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        row[2] = make_float4(acc[8], acc[9], acc[10], hit ? 1.f : 0.f);
        if (touched) touched[g] = hit ? 1 : 0;
    } else if (hit) {
        float *row = grad + kG * g;
#pragma unroll
        for (int j = 0; j < 11; ++j) row[j] += acc[j];
        row[11] = 1.f;   // accepted by a slice of this batch (peer update)
        if (touched) touched[g] = 1;
    }
}

// Background gradients (gradients.py:106-112): block s tree-reduces slice
// s's tile partials in fixed order; the last step adds the slices in order.
__global__ void bg_slice_kernel(const float2 *__restrict__ bin_bg,
                                const ugs_slice *__restrict__ slices,
                                double2 *__restrict__ out, const PlanHdr *__restrict__ hdr) {
    pdl_entry();
    __shared__ double sa[256], sc_[256];
    if (plan_overflow(hdr)) return;
    const int s = blockIdx.x;
    const int tile_base = slices[s].tile_base;
    const int ntile = slices[s].tiles_x * slices[s].tiles_y;
    double a = 0.0, c = 0.0;
    for (int i = threadIdx.x; i < ntile; i += blockDim.x) {
        a += bin_bg[tile_base + i].x;
        c += bin_bg[tile_base + i].y;
    }
    sa[threadIdx.x] = a;
    sc_[threadIdx.x] = c;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sa[threadIdx.x] += sa[threadIdx.x + o];
            sc_[threadIdx.x] += sc_[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[s] = make_double2(sa[0], sc_[0]);
}

// Adds the background gradients into grad_bg, or (adam != 0) applies the
// background Adam step with them.
__global__ void bg_finalize_kernel(const double2 *__restrict__ sums, int S,
                                   double *__restrict__ bg_raw,
                                   float *__restrict__ grad_bg, float scale, int adam,
                                   float *__restrict__ m_bg, float *__restrict__ v_bg,
                                   AdamConst k, const PlanHdr *__restrict__ hdr) {
    pdl_entry();
    if (threadIdx.x != 0 || plan_overflow(hdr)) return;
    const double cbg = sigmoid_f64(bg_raw[0]), abg = sigmoid_f64(bg_raw[1]);
    // adam: 0 accumulate into grad_bg, 1 Adam step, 2 overwrite grad_bg
    float g[2] = {adam ? 0.f : grad_bg[0], adam ? 0.f : grad_bg[1]};
    for (int s = 0; s < S; ++s) {
        const double d_cbg = (double)(float)abg * sums[s].x;   // sum dpix*f32(a_bg)/ssum
        const double d_abg = sums[s].y;                        // sum dpix*(c_bg-chat)/ssum
        g[0] += (float)((double)scale * d_cbg * cbg * (1.0 - cbg));
        g[1] += (float)((double)scale * d_abg * abg * (1.0 - abg));
    }
    if (adam == 1) {
        adam_bg(bg_raw, g, m_bg, v_bg, k);
    } else {
        grad_bg[0] = g[0];
        grad_bg[1] = g[1];
    }
}

constexpr size_t kFwdSmem = kFwdRawOff + sizeof(Frag) * kBatch;
constexpr size_t kBwdSmem = kBwdIdsOff + 2 * sizeof(uint32_t) * kBwdBatch;
// four backward CTAs per SM (the register budget's count): 228 KB of shared
// memory per SM, 1 KB of it reserved per CTA
static_assert(4 * (kBwdSmem + 1024) <= 228 * 1024, "backward shared memory per CTA");
static_assert(4 * (kFwdSmem + 1024) <= 228 * 1024, "forward shared memory per CTA");

int set_smem_attrs() {
    static std::atomic<unsigned long long> done{0};
    if (device_setup_done(done)) return UGS_OK;
    UGS_CUDA(cudaFuncSetAttribute(forward_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kFwdSmem));
    UGS_CUDA(cudaFuncSetAttribute(backward_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kBwdSmem));
    mark_device_setup(done);
    return UGS_OK;
}

}  // namespace

#ifndef UGS_TILE_ORDER
#define UGS_TILE_ORDER 1
#endif
const int32_t *raster_order(const ugs_plan &p) {
    return UGS_TILE_ORDER ? p.b.tile_order : nullptr;
}
dim3 raster_grid(const ugs_plan &p) {
    return raster_order(p) ? dim3((unsigned)(p.S * p.max_tiles)) : dim3(p.max_tiles, p.S);
}

int launch_tile_order(const ugs_plan &p, cudaStream_t st) {
    if (!raster_order(p) || p.S == 0) return UGS_OK;
    UGS_PDL(tile_order_kernel, 1, 1024, 0, st, p.b.bin_range, p.b.slices, p.S, p.max_tiles,
        p.b.tile_order, plan_hdr(p.b));
    UGS_LAUNCH_CHECK("tile_order_kernel");
    return UGS_OK;
}

int launch_forward(const ugs_plan &p, const ugs_cloud &c, const uint32_t *vals,
                   float *num, float *den, cudaStream_t st) {
    if (p.S == 0) return UGS_OK;
    int rc = set_smem_attrs();
    if (rc) return rc;
    dim3 grid(p.max_tiles, p.S);
    ugs_plan *pm = const_cast<ugs_plan *>(&p);
    stage_begin(pm, kStageForward, st);
    if (p.ordered) {
        UGS_PDL(forward_ordered_kernel, grid, kRasterThreads, 0, st,
        p.b.frag, vals, p.b.bin_range, p.b.slices, c.bg_raw, num, den, plan_hdr(p.b));
        UGS_LAUNCH_CHECK("forward_ordered_kernel");
    } else {
        UGS_PDL(forward_kernel, raster_grid(p), kRasterThreads, kFwdSmem, st,
        p.b.frag, vals, p.b.bin_range, p.b.slices, c.bg_raw, num, den, plan_hdr(p.b),
            (const int32_t *)raster_order(p), p.max_tiles);
        UGS_LAUNCH_CHECK("forward_kernel");
    }
    stage_end(pm, kStageForward, st);
    return UGS_OK;
}

int launch_backward(const ugs_plan &p, const ugs_cloud &c, const uint32_t *vals,
                    const float *num, const float *den, const float *dpix,
                    float *grad, uint8_t *touched, float scale, const AdamArgs *adam,
                    cudaStream_t st, bool dense) {
    if (p.S == 0) return UGS_OK;
    int rc = set_smem_attrs();
    if (rc) return rc;
    ugs_plan *pm = const_cast<ugs_plan *>(&p);
    stage_begin(pm, kStageBackward, st);
#ifndef UGS_PDL_BWD
#define UGS_PDL_BWD 1
#endif
#ifndef UGS_PDL_FIN
#define UGS_PDL_FIN 0   // finalize CTAs parked during the backward's tail: 1.53 -> 1.49 ms/step
#endif
    UGS_LAUNCH_EX(UGS_PDL_BWD, backward_kernel, raster_grid(p), kRasterThreads, kBwdSmem, st,
        p.b.frag, vals, p.b.bin_range, p.b.slices, num, den, dpix,
        c.bg_raw, p.b.partial, p.b.bin_bg, plan_hdr(p.b), (const int32_t *)raster_order(p),
        p.max_tiles);
    UGS_LAUNCH_CHECK("backward_kernel");
    stage_end(pm, kStageBackward, st);
    // the two background parameters (bg_slice -> bg_finalize) only need the
    // backward's per-tile partials: they run on a side stream, overlapping
    // the per-record finalize + update, and are joined before returning
    if (!pm->side) UGS_CUDA(cudaStreamCreateWithFlags(&pm->side, cudaStreamNonBlocking));
    if (!pm->ev_fork) {   // (the side stream may come from the bin's order fork)
        UGS_CUDA(cudaEventCreateWithFlags(&pm->ev_fork, cudaEventDisableTiming));
        UGS_CUDA(cudaEventCreateWithFlags(&pm->ev_join, cudaEventDisableTiming));
    }
    cudaStream_t side = pm->side;
    UGS_CUDA(cudaEventRecord(pm->ev_fork, st));
    UGS_CUDA(cudaStreamWaitEvent(side, pm->ev_fork, 0));
    UGS_PDL(bg_slice_kernel, p.S, 256, 0, side,
        p.b.bin_bg, p.b.slices, p.b.bg_sums, plan_hdr(p.b));
    UGS_LAUNCH_CHECK("bg_slice_kernel");
    if (adam) {
        UGS_PDL(bg_finalize_kernel, 1, 32, 0, side,
        p.b.bg_sums, p.S, const_cast<double *>(c.bg_raw),
                                               nullptr, scale, 1, adam->m + kG * c.n,
                                               adam->v + kG * c.n, adam->k, plan_hdr(p.b));
    } else {
        UGS_PDL(bg_finalize_kernel, 1, 32, 0, side,
        p.b.bg_sums, p.S, const_cast<double *>(c.bg_raw),
                                               grad + kG * c.n, scale, dense ? 2 : 0,
                                               nullptr, nullptr,
                                               AdamConst{}, plan_hdr(p.b));
    }
    UGS_LAUNCH_CHECK("bg_finalize_kernel");
    UGS_CUDA(cudaEventRecord(pm->ev_join, side));
    stage_begin(pm, kStageFinalize, st);
    const CloudMut cm{const_cast<float *>(c.means), const_cast<float *>(c.l_raw),
                      const_cast<float *>(c.intensity_raw),
                      const_cast<float *>(c.opacity_raw)};
    if (p.m_grid > 0) {
        const int th = 128;
        UGS_LAUNCH_EX(UGS_PDL_FIN, finalize_records_kernel, (unsigned)((p.m_grid + th - 1) / th), th, 0, st,
        p.b.rec, p.b.rec_gid, p.b.rec_inst, p.b.partial, plan_hdr(p.b), p.b.slice_base, p.S,
            p.b.slices, c.means, c.l_raw, (float)c.beta, p.b.rgrad);
        UGS_LAUNCH_CHECK("finalize_records_kernel");
    }
    stage_end(pm, kStageFinalize, st);
    stage_begin(pm, kStageUpdate, st);
    if (c.n > 0 && (adam || dense || p.m_grid > 0)) {
        const int64_t nblk = (c.n + kPrepThreads - 1) / kPrepThreads;
        const int64_t nwarp_all = nblk * (kPrepThreads / 32);
        static_assert(kUpdThreads == kPrepThreads, "update blocks mirror count blocks");
        // the warp-coalesced Adam path moves rows as float4: 16-byte bases
        const int aligned =
            adam && ((((uintptr_t)c.means | (uintptr_t)c.l_raw | (uintptr_t)adam->m |
                       (uintptr_t)adam->v) & 15) == 0);
        UGS_PDL(update_gather_kernel, (unsigned)nblk, kUpdThreads, 0, st,
        p.b.amask, p.b.warp_rec, p.b.rgrad, p.S, nwarp_all, c.n, scale,
            adam ? 1 : (dense ? 2 : 0),
            grad, touched, cm, adam ? adam->m : nullptr, adam ? adam->v : nullptr,
            adam ? adam->k : AdamConst{}, adam ? adam->grad_sum : nullptr,
            adam ? adam->grad_cnt : nullptr, aligned, plan_hdr(p.b));
        UGS_LAUNCH_CHECK("update_gather_kernel");
    }
    stage_end(pm, kStageUpdate, st);
    UGS_CUDA(cudaStreamWaitEvent(st, pm->ev_join, 0));   // background joined
    return UGS_OK;
}

}  // namespace ugs
