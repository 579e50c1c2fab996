/*
 * ugs.h -- C ABI of the B200-native (sm_100a) UltraGauss probe-plane
 * rasterizer and training step ("libugs.so").
 *
 * Drop-in boundary for the reference's native path (echosplat,
 * pkg/src/echosplat/):
 *   ugs_bin            replaces _prepare (rasterizer.py:109-137) -- build_L,
 *                      invert_lower_triangular, chi^2 boxes, cull, compact,
 *                      clamped windows -- plus the tile binning / radix sort
 *                      that the GPU forward needs (no counterpart in the ref)
 *   ugs_forward        replaces forward_kernel (_kernels.py:19-47) and the
 *                      background blend of rasterize (rasterizer.py:175-177)
 *   ugs_backward       replaces backward_kernel (_kernels.py:50-101) and the
 *                      raw-parameter chain + background grads of backward
 *                      (gradients.py:84-113)
 *   ugs_grad_stats     replaces the densify statistics (trainer.py:399-401)
 *   ugs_adam_step      replaces adam_step (trainer.py:170-200)
 *   ugs_densify_apply  replaces the row surgery of densify_prune_resample
 *                      (trainer.py:208-279; selection/RNG stay on the host)
 *
 * Conventions (the reference kernels: caller owns and zeroes the outputs,
 * no error path; here every entry point returns 0 on success or a negative
 * ugs_status and ugs_last_error() describes the failure):
 *   - every pointer marked (dev) is CUDA device memory, (host) host memory;
 *   - work is enqueued on the given cudaStream_t (passed as void*), nothing
 *     synchronizes except ugs_bin (one device->host read of the per-slice
 *     counts, needed to size the tile lists; ugs_bin_async avoids it) and
 *     ugs_plan_poll (waits for one event); ugs_backward /
 *     ugs_backward_adam also run the two background-parameter kernels on the
 *     plan's own side stream, forked from and joined back into the caller's
 *     stream with events, so the call stays stream-ordered;
 *   - a ugs_plan owns the binning buffers of one batch; distinct plans may
 *     be used concurrently from different threads/streams;
 *   - no torch types: plain pointers and sizes, so ctypes / cffi / JNI /
 *     cgo bindings are mechanical.
 */
#ifndef UGS_H
#define UGS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define UGS_API __attribute__((visibility("default")))
#else
#define UGS_API
#endif

#define UGS_ABI_VERSION 2
#define UGS_TILE 16 /* pixels per tile side */

typedef enum ugs_status {
    UGS_OK = 0,
    UGS_ERR_INVALID = -1, /* bad argument (InvalidParameterError in the ref) */
    UGS_ERR_CUDA = -2,    /* CUDA runtime / launch failure */
    UGS_ERR_OOM = -3,     /* device allocation failed */
    UGS_ERR_RANGE = -4    /* sizes beyond the 32-bit index budget */
} ugs_status;

/* Per-slice constants, formed on the host exactly as the reference forms
 * them (geometry.py:61-64 inverse, :107-120 plane_axes, rasterizer.py:115-135
 * casts): everything float32. */
typedef struct ugs_slice {
    float rw[9];      /* f32(R^T), row-major: world -> probe rotation */
    float tw[3];      /* f32(-R^T t) */
    float origin[3];  /* f32(t - cx*du - cy*dv): world position of pixel (0,0) */
    float du[3];      /* f32(R[:,0]*spacing) */
    float dv[3];      /* f32(R[:,1]*spacing) */
    float sqrt_cut;   /* sqrtf(f32(chi2.ppf(p, 3))) */
    float s;          /* f32(spacing) */
    float cx, cy;     /* f32((W-1)/2), f32((H-1)/2) */
    float x1h, x2h;   /* f32((W-1)/2*spacing), f32((H-1)/2*spacing) */
    int32_t width, height;
    int32_t tiles_x, tiles_y; /* ceil(W/16), ceil(H/16): filled by ugs_bin */
    int32_t tile_base;        /* first bin id of this slice: filled by ugs_bin */
    int32_t reserved;
    int64_t pix_base;         /* offset of this slice in the (S,H,W) outputs */
} ugs_slice;

/* The Gaussian cloud (GaussianCloud, model.py:31-89), structure of arrays. */
typedef struct ugs_cloud {
    const float *means;         /* (dev) (n,3) mm, world frame */
    const float *l_raw;         /* (dev) (n,6): L11,L22,L33,L21,L31,L32 raw */
    const float *intensity_raw; /* (dev) (n,) */
    const float *opacity_raw;   /* (dev) (n,) */
    const double *bg_raw;       /* (dev) [2]: bg_intensity_raw, bg_opacity_raw */
    int64_t n;
    double beta;                /* L_jj = l_jj^2 + beta, beta > 0 (f32(beta)
                                   on the float32 render path, as the ref) */
} ugs_cloud;

typedef struct ugs_plan ugs_plan;

UGS_API const char *ugs_last_error(void);
UGS_API int ugs_abi_version(void);

UGS_API int ugs_plan_create(ugs_plan **out);
UGS_API int ugs_plan_destroy(ugs_plan *plan);

/* Phase 1 + binning for a batch of S slices (host array `slices`; the
 * library fills tiles_x/tiles_y/tile_base and keeps a device copy).
 * Writes per-slice accepted counts m_out[S], tile-instance counts k_out[S]
 * and (Gaussian, pixel) pair counts p_out[S] (host; any may be NULL).
 * Synchronizes `stream` once. */
UGS_API int ugs_bin(ugs_plan *plan, const ugs_cloud *cloud, ugs_slice *slices, int S,
            void *stream, int64_t *m_out, int64_t *k_out, int64_t *p_out);

/* ugs_bin without the host synchronisation (no reference counterpart: the
 * reference sizes everything on the host).  The record / instance / sort
 * buffers are used at the capacities the plan already has (an earlier
 * ugs_bin sized them, with headroom; on a plan never binned synchronously,
 * or with more than 1024 tiles per slice, this call IS ugs_bin).  The device
 * compares the batch's totals with those capacities: if the batch does not
 * fit, every later kernel of this plan (forward, backward, the fused update)
 * returns at entry, leaving parameters and moments untouched.  The counts
 * arrive with ugs_plan_poll. */
UGS_API int ugs_bin_async(ugs_plan *plan, const ugs_cloud *cloud, ugs_slice *slices,
                          int S, void *stream);

/* Counts of the plan's last ugs_bin / ugs_bin_async (waits for that call's
 * count stage only -- an event, not the stream).  *overflowed = 1 if that
 * sync-free batch did not fit: its forward / backward / update did nothing,
 * the plan has now grown to fit it, and the caller re-issues the step.
 * Any output pointer may be NULL. */
UGS_API int ugs_plan_poll(ugs_plan *plan, int *overflowed, int64_t *m_out, int64_t *k_out,
                          int64_t *p_out);

/* Accepted Gaussian indices (ascending per slice, slices concatenated) and
 * their inclusive pixel windows (iu0,iu1,iv0,iv1) -- the reference's
 * RenderBuffers.accepted and _prepare windows.  Either pointer may be NULL. */
UGS_API int ugs_export_accepted(const ugs_plan *plan, int32_t *accepted /* (dev) M */,
                        int32_t *windows /* (dev) M x 4 */, void *stream);

/* Sorted tile lists: bin_range (dev, n_bins x 2 = [start,end)) and, per
 * sorted entry, the Gaussian index it refers to (dev, K).  n_bins_out and
 * k_total_out (host) may be queried with NULL device pointers. */
UGS_API int ugs_export_bins(const ugs_plan *plan, int32_t *bin_range,
                    int32_t *sorted_gauss, int32_t *n_bins_out,
                    int64_t *k_total_out, void *stream);

/* Forward accumulation + background for every slice of the last ugs_bin:
 * num/den (dev) float32, slice s at slices[s].pix_base, row-major H x W.
 * Fully overwrites the covered pixels (no caller zeroing needed). */
UGS_API int ugs_forward(ugs_plan *plan, const ugs_cloud *cloud, float *num, float *den,
                void *stream);

/* Render-only forward (the serving path: rasterizer.py:182-186 render_slice,
 * server.py:103-126): pixels (dev) float32 = clip(num / den, 0, 1) written
 * directly, same layout as ugs_forward's outputs, bitwise equal to
 * clip(num / den) of ugs_forward's num and den. */
UGS_API int ugs_render(ugs_plan *plan, const ugs_cloud *cloud, float *pixels, void *stream);

/* ugs_bin_async + ugs_render in one call (the batched serving path,
 * rasterizer.py:182-186 render_slice per slice of a batch): on a sized plan
 * the binning chain (count -> scan -> plan -> emit -> bin sort) is one CUDA
 * graph, captured on first use and replayed while the plan's buffers, the
 * cloud and the batch shape repeat; the render follows it on the stream.
 * Same contract as the two calls: ugs_plan_poll reports an overflowed
 * batch, which the caller re-issues (ugs_bin + ugs_render).  An unsized
 * plan takes the synchronous bin. */
UGS_API int ugs_render_batch(ugs_plan *plan, const ugs_cloud *cloud, ugs_slice *slices, int S,
                     float *pixels, void *stream);

/* Gradient / Adam-moment layout ("AoS-12", float32, 12 n + 2 entries):
 * Gaussian g owns [12 g, 12 g + 12) = [d_means 0..2 | d_l_raw 3..8 |
 * d_intensity_raw 9 | d_opacity_raw 10 | pad 11]; [12 n, 12 n + 2) holds
 * the background (intensity, opacity).  16-byte aligned. */

/* Backward for every slice of the last ugs_bin.  d_pixels (dev, same layout
 * as num).  Accumulates `scale` x (raw-parameter gradients) into grad (dev,
 * AoS-12), sets the pad slot of every accepted Gaussian's row to 1 and
 * touched[g] = 1 (touched may be NULL).  Slices are reduced in order, without atomics: deterministic. */
UGS_API int ugs_backward(ugs_plan *plan, const ugs_cloud *cloud, const float *num,
                 const float *den, const float *d_pixels, float *grad,
                 uint8_t *touched, float scale, void *stream);

/* ugs_backward that OVERWRITES grad instead of accumulating: every row of
 * the AoS-12 buffer (all n Gaussians, zeros where no slice accepted g, pad
 * slot = 1 where one did) and the two background entries -- the caller
 * neither zeroes it nor has it read back (the multi-GPU step's per-rank
 * gradient).  grad 16-byte aligned. */
UGS_API int ugs_backward_dense(ugs_plan *plan, const ugs_cloud *cloud, const float *num,
                               const float *den, const float *d_pixels, float *grad,
                               float scale, void *stream);

/* The single-GPU training step's backward half in one call: backward +
 * ordered accumulation + densify statistics (grad_sum/grad_cnt, may be NULL)
 * + Adam on every parameter (trainer.py:170-200, bit-compatible arithmetic),
 * without materialising the dense gradient.  The cloud's parameter arrays
 * and bg_raw are updated IN PLACE (the const in ugs_cloud notwithstanding).
 * m, v: AoS-12 moments; t: step count after increment; lr as ugs_adam_step. */
UGS_API int ugs_backward_adam(ugs_plan *plan, const ugs_cloud *cloud,
                              const float *num, const float *den,
                              const float *d_pixels, float scale, float *m,
                              float *v, int64_t t, const double *lr,
                              double beta1, double beta2, double eps,
                              float *grad_sum, int32_t *grad_cnt, void *stream);

/* grad_sum[g] += ||d_means[g]||, grad_cnt[g] += 1 for touched Gaussians,
 * then clears touched (trainer.py:399-401).  grad: AoS-12. */
UGS_API int ugs_grad_stats(const float *grad, int64_t n, uint8_t *touched,
                   float *grad_sum, int32_t *grad_cnt, void *stream);

/* One Adam step over all groups, bit-compatible with trainer.py:170-200.
 * lr[0] means, lr[1] l_raw, lr[2] intensity, lr[3] opacity, lr[4] bg.
 * grad, m, v (dev) AoS-12.  t is the step count after increment.  If
 * zero_grad != 0 the gradient buffer is cleared after use.  touched /
 * grad_sum / grad_cnt (all or none) fold in ugs_grad_stats. */
UGS_API int ugs_adam_step(float *means, float *l_raw, float *intensity_raw,
                  float *opacity_raw, double *bg_raw, float *grad, float *m,
                  float *v, int64_t n, int64_t t, const double *lr,
                  double beta1, double beta2, double eps, int zero_grad,
                  uint8_t *touched, float *grad_sum, int32_t *grad_cnt,
                  void *stream);

/* Densify/prune row surgery (trainer.py:208-279, model.py:147-152):
 * dst row j < n_keep copies src row keep[j]; then for each of the n_new
 * candidates c (cand = index into the KEPT rows): split[c] != 0 ->
 * parent row cand[c] gets child mean mu + Linv^T z[c][0:3] and the shrunk
 * l_raw, and new row n_keep+c gets mu + Linv^T z[c][3:6] with the same
 * l_raw; split[c] == 0 -> new row is a copy.  New rows' Adam moments are
 * zero.  src/dst param and moment buffers must not alias. */
UGS_API int ugs_densify_apply(const ugs_cloud *src, const float *m_src,
                      const float *v_src, const int32_t *keep, int64_t n_keep,
                      const int32_t *cand, const uint8_t *split,
                      const double *z, int64_t n_new, double split_factor,
                      float *means, float *l_raw, float *intensity_raw,
                      float *opacity_raw, float *m_dst, float *v_dst,
                      void *stream);

/* Training loss for S slices of H x W (ref trainer.py:130-151,
 * metrics.py:23-98), float64 arithmetic: pred = f32(num/den);
 * loss[s] = (1-lam)*mean|pred-target| + lam*(1 - SSIM)  (or mean squared
 * error if l2 != 0) and d_pixels = d loss / d pred (float32, (S,H,W)).
 * loss_out / ssim_out (dev, S doubles) may be NULL; den may be NULL
 * (pred = num: the public ssim / loss API on images).  `workspace` (dev) must
 * hold ugs_loss_workspace_bytes(S, H, W).  Deterministic. */
UGS_API size_t ugs_loss_workspace_bytes(int S, int H, int W);
UGS_API int ugs_loss(const float *num, const float *den, const float *target,
                     int S, int H, int W, double lam, int l2, float *d_pixels,
                     double *loss_out, double *ssim_out, void *workspace,
                     void *stream);

/* ugs_loss with the targets gathered from a dataset -- slice s compares
 * against target + target_index[s] * H * W (target_index: dev int64, NULL =
 * slice s itself) -- and the batch-mean loss written to loss_mean_out (dev
 * double, may be NULL).  S <= 64. */
UGS_API int ugs_loss_ex(const float *num, const float *den, const float *target,
                        const int64_t *target_index, int S, int H, int W, double lam,
                        int l2, float *d_pixels, double *loss_out, double *ssim_out,
                        double *loss_mean_out, void *workspace, void *stream);

/* Forward accumulation order.  0 (default): each of the 8 warps of a tile
 * accumulates its share of the tile's records into a private buffer and the
 * buffers are summed in fixed order -- the reference's multi-worker scheme
 * (rasterizer.py:157-173).  1: every pixel adds its Gaussians strictly in
 * ascending index, the reference's sequential workers=1 order
 * (_kernels.py:23-47).  Both are deterministic. */
UGS_API int ugs_plan_set_ordered(ugs_plan *plan, int ordered);

/* ---- multi-GPU update over peer memory (the reference
 * is single-process) -------------------------------------------------------
 * Each rank owns an "arena" (ugs_ipc_alloc: device memory + a 64-byte CUDA
 * IPC handle) holding its parameters, AoS-12 gradient and moments and the
 * densify statistics; every process maps each peer's arena (ugs_ipc_open)
 * and describes all of them, as mapped locally, with ugs_peer_view. */
typedef struct ugs_peer_view {
    float *means, *l_raw, *intensity_raw, *opacity_raw; /* SoA, n rows */
    float *grad, *m, *v;   /* AoS-12 (12 n + 2), 16-byte aligned */
    float *grad_sum;       /* densify statistics, n */
    int32_t *grad_cnt;
    double *bg_raw;        /* the rank's background pair */
    uint32_t *sync;        /* 64 words: ready[8], done[8], block counter --
                              the device-side step barrier (ugs_peer_signal /
                              ugs_peer_update / ugs_peer_wait), zeroed at
                              allocation */
} ugs_peer_view;

UGS_API int ugs_ipc_alloc(size_t bytes, void **ptr, void *handle64);
UGS_API int ugs_ipc_open(const void *handle64, void **ptr);
UGS_API int ugs_ipc_close(void *ptr);
UGS_API int ugs_ipc_free(void *ptr);

/* Fused reduce-scatter + Adam + all-gather (replaces the all-reduce of the
 * gradient and the replicated adam_step, trainer.py:170-200): for g in the
 * rank's shard [lo, hi) sums the W ranks' gradient rows in rank order (pad
 * slot > 0 marks a Gaussian some rank's slice accepted: densify statistics,
 * trainer.py:399-401, when stats != 0), applies the bit-compatible Adam to
 * the owned rows of this rank's arena and writes the new parameter rows into
 * every peer's arena (coalesced 16-byte stores over NVLink for full warps of
 * 32 rows: shard bounds are multiples of 32, ugs_peer_shard); every rank
 * updates the background pair identically.
 * epoch > 0: the step barriers run on the device -- every block first waits
 * until each rank's ready[] flag in this arena reaches `epoch` (set by the
 * ranks' ugs_peer_signal after their gradients were written), and the last
 * block to finish sets done[rank] = epoch in every peer's arena, which
 * ugs_peer_wait awaits.  epoch = 0: the caller brackets the call with its
 * own barriers (all gradients written before; all parameter rows stored
 * after). */
UGS_API int ugs_peer_update(const ugs_peer_view *views, int world, int rank, int64_t n,
                            int64_t lo, int64_t hi, int64_t t, const double *lr,
                            double beta1, double beta2, double eps, int stats,
                            uint32_t epoch, void *stream);

/* [lo, hi) of rank q's shard: multiples of 32 Gaussians (hi = n for the last
 * rank), so a warp's rows move as whole 16-byte vectors. */
UGS_API int ugs_peer_shard(int64_t n, int world, int q, int64_t *lo, int64_t *hi);

/* Device-side step barrier halves (stream-ordered, no host involvement):
 * signal stores ready[rank] = epoch into every peer's arena after a
 * system-scope fence (this rank's gradient, written by earlier kernels on the
 * stream, is then visible to the peers); wait spins until done[q] >= epoch
 * for every rank q (all parameter rows of the step stored here).  Spins are
 * bounded (~20 s): a missing peer traps the kernel instead of hanging. */
UGS_API int ugs_peer_signal(const ugs_peer_view *views, int world, int rank, uint32_t epoch,
                            void *stream);
UGS_API int ugs_peer_wait(const ugs_peer_view *views, int world, int rank, uint32_t epoch,
                          void *stream);

/* Before densify: copies the m, v, grad_sum, grad_cnt rows owned by other
 * ranks (the ugs_peer_shard shards) into this rank's arena. */
UGS_API int ugs_peer_gather(const ugs_peer_view *views, int world, int rank, int64_t n,
                            void *stream);

/* ---- diagnostics (no counterpart in the reference, which has no tracing:
 * SURVEY section 5) --------------------------------------------------- */

/* Kernels launched by this library since it was loaded. */
UGS_API long long ugs_launch_count(void);

/* Enable CUDA-event timing of the plan's stages (phase-1 count, emit, sort,
 * ranges, forward, backward, finalize).  Adds no synchronization of its own:
 * finished events are harvested at the next ugs_bin (which synchronizes
 * anyway) or by ugs_plan_timings. */
UGS_API int ugs_plan_set_timing(ugs_plan *plan, int enabled);

/* Host helper: fill S ugs_slice structs (pix_base = running pixel offset)
 * from float64 poses -- rot (S,3,3) row-major, trans (S,3) -- spacing, width,
 * height and the chi-square cut chi2.ppf(p, 3); the reference's float64
 * operation order then float32, byte-identical to the package's numpy
 * fill_slice (ProbePose.inverse geometry.py:61-64, plane_axes :107-120). */
UGS_API int ugs_fill_slices(const double *rot, const double *trans, const double *spacing,
                            const int32_t *width, const int32_t *height, int S, double cut,
                            ugs_slice *out);

/* Accumulated milliseconds and call counts per stage (host arrays of n);
 * returns the number of stages.  reset != 0 clears the accumulators. */
/* FP32 FMA throughput probe: `blocks` x 256 threads each run `iters`
 * iterations of 8 independent FMA chains; writes a checksum to out (dev).
 * Flops = blocks*256*iters*16.  Used to measure the FP32 roofline peak. */
UGS_API int ugs_fp32_peak_probe(float *out, int blocks, int iters, void *stream);

UGS_API int ugs_plan_timings(ugs_plan *plan, double *ms_total, int64_t *calls,
                             int n, int reset);

#ifdef __cplusplus
}
#endif
#endif /* UGS_H */
