// Fused training loss: (1-lam)*L1 + lam*(1-SSIM) and its pixel gradient for
// a batch of slices (ref trainer.py:130-151, metrics.py:23-98), float64 like
// the reference, in two launches.
//
// SSIM: 11x11 Gaussian window (sigma 1.5), C1 = 1e-4, C2 = 9e-4, valid
// windows only.  Its gradient is adj(A) + 2x adj(B) + y adj(C) with
// A = dS/dmu - 2 mu_x dS/dsxx - mu_y dS/dsxy, B = dS/dsxx, C = dS/dsxy on the
// valid grid and adj() the zero-padded full correlation (the adjoint of the
// valid filter).  One CTA owns a 32x32 output tile: it loads the 52x52 input
// neighbourhood, filters the five moments (x, y, x^2, y^2, xy) separably onto
// the 42x42 valid points it needs, forms A, B, C there, applies the adjoint
// separably back onto its 32x32 pixels (register-blocked runs of outputs per
// thread) and writes d_pixels (float32, what
// the backward consumes -- gradients.py:62 casts the same way).  Per-tile
// sums (sum|diff| over owned pixels, sum SSIM over owned valid points) are
// reduced per slice in fixed order by a second tiny kernel: deterministic.
#include "ugs_internal.cuh"

namespace ugs {
namespace {

constexpr int kLT = 32;              // output tile
constexpr int kPad = 5;              // window radius
constexpr int kF = kLT + 2 * kPad;   // 42: valid points needed
constexpr int kI = kF + 2 * kPad;    // 52: input points needed
constexpr int kLossThreads = 384;    // 12 warps, two 109 KB CTAs per SM

__constant__ double c_win[11];

// Register blocking: every pass gives a thread a run of consecutive outputs
// (6 or 8) of one row/column, so each shared-memory value it loads feeds up
// to 11 outputs from registers (the earlier one-output-per-thread passes were
// shared-memory bound).  Per output the taps are still added in increasing
// order with the same expressions, so the sums are unchanged.
constexpr int kHB = 6;               // horizontal / vertical moment run
constexpr int kAB = 4;               // adjoint run

struct LossSmem {
    float X[kI][kI];                  // prediction (f32 num/den, exact in float)
    float Y[kI][kI];                  // target
    union {
        double h[5][kI][kF];          // horizontal moment pass
        struct {                      // after the vertical pass (h dead):
            double F[3][kF][kF];      //   A, B, C on the valid grid
            double ha[3][kF][kLT];    //   horizontal adjoint pass
        } a;
    } u;
    double red[2][kLossThreads / 32];
};
// the vertical pass has at most one work item per thread, so its A, B, C
// are held in registers across the barrier that retires h, and F reuses h's
// storage: 109 KB per CTA, two CTAs per SM
static_assert(kF * (kF / kHB) <= kLossThreads, "one vertical item per thread");

__global__ void __launch_bounds__(kLossThreads, 2)
loss_tile_kernel(const float *__restrict__ num, const float *__restrict__ den,
                 const float *__restrict__ target, const int64_t *__restrict__ target_index,
                 int H, int W, double lam,
                 int l2, float *__restrict__ dpix, double *__restrict__ tile_sums,
                 int tiles_x, int tiles_per_slice) {
    pdl_entry();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    LossSmem &sm = *reinterpret_cast<LossSmem *>(smem_raw);
    const int s = blockIdx.y;
    const int tile = blockIdx.x;
    const int p0 = (tile / tiles_x) * kLT, q0 = (tile % tiles_x) * kLT;
    const size_t base = (size_t)s * H * W;
    // the targets may be gathered from a dataset: slice s reads target_index[s]
    const size_t tbase = (target_index ? (size_t)target_index[s] : (size_t)s) * H * W;
    const int tid = threadIdx.x;
    const int HV = H - 2 * kPad, WV = W - 2 * kPad;   // valid grid
    const double npx = (double)H * W, nv = (double)HV * WV;
    // load the 52x52 neighbourhood (rows p0-10 .., cols q0-10 ..): all of a
    // thread's global loads are issued before any is consumed
    constexpr int kLd = (kI * kI + kLossThreads - 1) / kLossThreads;
    float ln[kLd], ld[kLd], lt[kLd];
#pragma unroll
    for (int j = 0; j < kLd; ++j) {
        const int i = tid + j * kLossThreads;
        const int r = i / kI, c = i % kI;
        const int P = p0 - 2 * kPad + r, Q = q0 - 2 * kPad + c;
        ln[j] = 0.f;
        ld[j] = 1.f;
        lt[j] = 0.f;
        if (i < kI * kI && P >= 0 && P < H && Q >= 0 && Q < W) {
            const size_t o = base + (size_t)P * W + Q;
            ln[j] = __ldg(num + o);
            ld[j] = den ? __ldg(den + o) : 1.f;   // den NULL: pred = num
            lt[j] = __ldg(target + (tbase + (size_t)P * W + Q));
        }
    }
#pragma unroll
    for (int j = 0; j < kLd; ++j) {
        const int i = tid + j * kLossThreads;
        if (i >= kI * kI) continue;
        const int r = i / kI, c = i % kI;
        sm.X[r][c] = __fdiv_rn(ln[j], ld[j]);   // pred = num / den (float32); 0 outside
        sm.Y[r][c] = lt[j];
    }
    __syncthreads();
    double ssim_sum = 0.0;
    const bool ssim = !l2 && lam > 0.0;
    if (ssim) {
        // horizontal pass: h[f][r][c] = sum_b w[b] f(r, c+b), c in [0,42)
        constexpr int kCh = kF / kHB;   // 7 runs per row
        for (int it = tid; it < kI * kCh; it += kLossThreads) {
            const int r = it / kCh, c0 = (it % kCh) * kHB;
            double a[5][kHB];
#pragma unroll
            for (int f = 0; f < 5; ++f)
#pragma unroll
                for (int o = 0; o < kHB; ++o) a[f][o] = 0.0;
#pragma unroll
            for (int kk = 0; kk < kHB + 10; ++kk) {
                // the product images first (as the reference filters x*x,
                // y*y, x*y), once per input point for all the run's outputs
                const double x = sm.X[r][c0 + kk], y = sm.Y[r][c0 + kk];
                const double xx = x * x, yy = y * y, xy = x * y;
#pragma unroll
                for (int o = 0; o < kHB; ++o) {
                    const int b = kk - o;
                    if (b < 0 || b > 10) continue;
                    const double w = c_win[b];
                    a[0][o] += w * x;
                    a[1][o] += w * y;
                    a[2][o] += w * xx;
                    a[3][o] += w * yy;
                    a[4][o] += w * xy;
                }
            }
#pragma unroll
            for (int f = 0; f < 5; ++f)
#pragma unroll
                for (int o = 0; o < kHB; ++o) sm.u.h[f][r][c0 + o] = a[f][o];
        }
        __syncthreads();
        // vertical pass -> moments at valid point (i, j) = (p0-10+r, q0-10+c)
        double FA[kHB], FB[kHB], FC[kHB];
        const int vit = tid;
        if (vit < kF * kCh) {
            const int c = vit % kF, r0 = (vit / kF) * kHB;
            double m[5][kHB];
#pragma unroll
            for (int f = 0; f < 5; ++f)
#pragma unroll
                for (int o = 0; o < kHB; ++o) m[f][o] = 0.0;
#pragma unroll
            for (int kk = 0; kk < kHB + 10; ++kk) {
                double v[5];
#pragma unroll
                for (int f = 0; f < 5; ++f) v[f] = sm.u.h[f][r0 + kk][c];
#pragma unroll
                for (int o = 0; o < kHB; ++o) {
                    const int a = kk - o;
                    if (a < 0 || a > 10) continue;
                    const double w = c_win[a];
#pragma unroll
                    for (int f = 0; f < 5; ++f) m[f][o] += w * v[f];
                }
            }
#pragma unroll
            for (int o = 0; o < kHB; ++o) {
                const int r = r0 + o;
                const int i = p0 - 2 * kPad + r, j = q0 - 2 * kPad + c;
                double A = 0, B = 0, C = 0;
                if (i >= 0 && i < HV && j >= 0 && j < WV) {
                    const double mx = m[0][o], my = m[1][o];
                    const double sxx = m[2][o] - mx * mx, syy = m[3][o] - my * my;
                    const double sxy = m[4][o] - mx * my;
                    const double C1 = 1e-4, C2 = 9e-4;
                    const double a1 = 2.0 * mx * my + C1, a2 = 2.0 * sxy + C2;
                    const double b1 = mx * mx + my * my + C1, b2 = sxx + syy + C2;
                    const double sv = (a1 * a2) / (b1 * b2);
                    const double d_mu = (2.0 * my * a2) / (b1 * b2) -
                                        (2.0 * mx * a1 * a2) / (b1 * b1 * b2);
                    const double d_sxx = -sv / b2, d_sxy = 2.0 * a1 / (b1 * b2);
                    A = d_mu - 2.0 * mx * d_sxx - my * d_sxy;
                    B = d_sxx;
                    C = d_sxy;
                    if (r >= 2 * kPad && c >= 2 * kPad) ssim_sum += sv;   // owned point
                }
                FA[o] = A;
                FB[o] = B;
                FC[o] = C;
            }
        }
        __syncthreads();   // every read of h is done: F may overwrite it
        if (vit < kF * kCh) {
            const int c = vit % kF, r0 = (vit / kF) * kHB;
#pragma unroll
            for (int o = 0; o < kHB; ++o) {
                sm.u.a.F[0][r0 + o][c] = FA[o];
                sm.u.a.F[1][r0 + o][c] = FB[o];
                sm.u.a.F[2][r0 + o][c] = FC[o];
            }
        }
        __syncthreads();
        // adjoint horizontal: ha[f][r][q] = sum_b w[b] F[f][r][q+b], q in [0,32)
        constexpr int kAq = kLT / kAB;   // 4 runs per row
        for (int it = tid; it < kF * kAq; it += kLossThreads) {
            const int r = it / kAq, q0r = (it % kAq) * kAB;
            double a[3][kAB];
#pragma unroll
            for (int f = 0; f < 3; ++f)
#pragma unroll
                for (int o = 0; o < kAB; ++o) a[f][o] = 0.0;
#pragma unroll
            for (int kk = 0; kk < kAB + 10; ++kk) {
                double v[3];
#pragma unroll
                for (int f = 0; f < 3; ++f) v[f] = sm.u.a.F[f][r][q0r + kk];
#pragma unroll
                for (int o = 0; o < kAB; ++o) {
                    const int b = kk - o;
                    if (b < 0 || b > 10) continue;
#pragma unroll
                    for (int f = 0; f < 3; ++f) a[f][o] += c_win[b] * v[f];
                }
            }
#pragma unroll
            for (int f = 0; f < 3; ++f)
#pragma unroll
                for (int o = 0; o < kAB; ++o) sm.u.a.ha[f][r][q0r + o] = a[f][o];
        }
        __syncthreads();
    }
    // pixels of this tile: gradient and L1 term (column q, a run of rows)
    double l1_sum = 0.0;
    constexpr int kAp = kLT / kAB;
    for (int it = tid; it < kLT * kAp; it += kLossThreads) {
        const int q = it % kLT, pr0 = (it / kLT) * kAB;
        double aA[kAB], aB[kAB], aC[kAB];
#pragma unroll
        for (int o = 0; o < kAB; ++o) aA[o] = aB[o] = aC[o] = 0.0;
        if (ssim) {
#pragma unroll
            for (int kk = 0; kk < kAB + 10; ++kk) {
                const double vA = sm.u.a.ha[0][pr0 + kk][q], vB = sm.u.a.ha[1][pr0 + kk][q],
                             vC = sm.u.a.ha[2][pr0 + kk][q];
#pragma unroll
                for (int o = 0; o < kAB; ++o) {
                    const int a = kk - o;
                    if (a < 0 || a > 10) continue;
                    const double w = c_win[a];
                    aA[o] += w * vA;
                    aB[o] += w * vB;
                    aC[o] += w * vC;
                }
            }
        }
#pragma unroll
        for (int o = 0; o < kAB; ++o) {
            const int p = pr0 + o;
            const int P = p0 + p, Q = q0 + q;
            if (P >= H || Q >= W) continue;
            const double x = sm.X[p + 2 * kPad][q + 2 * kPad];
            const double y = sm.Y[p + 2 * kPad][q + 2 * kPad];
            const double diff = x - y;
            double g;
            if (l2) {
                l1_sum += diff * diff;
                g = 2.0 * diff / npx;
            } else {
                l1_sum += fabs(diff);
                const double sg = (diff > 0.0) ? 1.0 : ((diff < 0.0) ? -1.0 : 0.0);
                g = (1.0 - lam) * sg / npx;
                if (ssim) g -= lam * (aA[o] + 2.0 * x * aB[o] + y * aC[o]) / nv;
            }
            dpix[base + (size_t)P * W + Q] = (float)g;
        }
    }
    // block sums in fixed order
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        l1_sum += __shfl_xor_sync(0xffffffffu, l1_sum, o);
        ssim_sum += __shfl_xor_sync(0xffffffffu, ssim_sum, o);
    }
    if (lane == 0) {
        sm.red[0][warp] = l1_sum;
        sm.red[1][warp] = ssim_sum;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0, b = 0;
        for (int w = 0; w < kLossThreads / 32; ++w) {
            a += sm.red[0][w];
            b += sm.red[1][w];
        }
        tile_sums[2 * ((size_t)s * tiles_per_slice + tile)] = a;
        tile_sums[2 * ((size_t)s * tiles_per_slice + tile) + 1] = b;
    }
}

// One block for the whole batch, one warp per slice (all slices in
// parallel): lane-strided sums of the slice's tile partials, then a fixed
// xor tree -- the same order on every call (deterministic) -- loss / SSIM
// per slice, and the batch-mean loss in slice order.
constexpr int kReduceWarps = 32;

__global__ void __launch_bounds__(32 * kReduceWarps)
loss_reduce_kernel(const double *__restrict__ tile_sums, int tiles_per_slice, int S, int H,
                   int W, double lam, int l2, double *__restrict__ loss_out,
                   double *__restrict__ ssim_out, double *__restrict__ mean_out) {
    pdl_entry();
    __shared__ double lv[64];
    const double npx = (double)H * W;
    const double nv = (double)(H - 2 * kPad) * (W - 2 * kPad);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = warp; s < S; s += kReduceWarps) {
        const double *ts = tile_sums + 2 * (size_t)s * tiles_per_slice;
        double a = 0, b = 0;
        for (int t = lane; t < tiles_per_slice; t += 32) {
            a += ts[2 * t];
            b += ts[2 * t + 1];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
        }
        if (lane == 0) {
            double v;
            const double mean_s = b / nv;
            if (l2) {
                v = a / npx;
            } else {
                v = (1.0 - lam) * (a / npx);
                if (lam > 0.0) v += lam * (1.0 - mean_s);
            }
            if (loss_out) loss_out[s] = v;
            if (ssim_out) ssim_out[s] = mean_s;
            lv[s] = v;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && mean_out) {
        double m = 0.0;
        for (int s = 0; s < S; ++s) m += lv[s];
        *mean_out = m / (double)S;
    }
}

std::atomic<unsigned long long> g_win_ready{0};

int upload_window() {
    if (device_setup_done(g_win_ready)) return UGS_OK;
    double w[11], sum = 0.0;
    for (int i = 0; i < 11; ++i) {
        const double x = (double)(i - kPad) / 1.5;
        w[i] = exp(-0.5 * x * x);
        sum += w[i];
    }
    for (int i = 0; i < 11; ++i) w[i] /= sum;
    UGS_CUDA(cudaMemcpyToSymbol(c_win, w, sizeof(w)));
    mark_device_setup(g_win_ready);
    return UGS_OK;
}

}  // namespace
}  // namespace ugs

using namespace ugs;

extern "C" size_t ugs_loss_workspace_bytes(int S, int H, int W) {
    const int tx = (W + kLT - 1) / kLT, ty = (H + kLT - 1) / kLT;
    return sizeof(double) * 2 * (size_t)S * tx * ty;
}

extern "C" int ugs_loss_ex(const float *num, const float *den, const float *target,
                           const int64_t *target_index, int S, int H, int W, double lam,
                           int l2, float *d_pixels, double *loss_out, double *ssim_out,
                           double *loss_mean_out, void *workspace, void *stream) {
    if (!num || !target || !d_pixels || !workspace || S < 1 || S > 64 || H < 1 ||
        W < 1) {
        set_error("ugs_loss: invalid arguments (1 <= S <= 64)");
        return UGS_ERR_INVALID;
    }
    if (!l2 && lam > 0.0 && (H < 11 || W < 11)) {
        set_error("ugs_loss: images must be at least 11x11 for SSIM");
        return UGS_ERR_INVALID;
    }
    int rc = upload_window();
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const int tx = (W + kLT - 1) / kLT, ty = (H + kLT - 1) / kLT;
    const size_t smem = sizeof(LossSmem);
    static std::atomic<unsigned long long> attr{0};
    if (!device_setup_done(attr)) {
        UGS_CUDA(cudaFuncSetAttribute(loss_tile_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
        mark_device_setup(attr);
    }
    dim3 grid(tx * ty, S);
    double *sums = static_cast<double *>(workspace);
    UGS_PDL(loss_tile_kernel, grid, kLossThreads, smem, st,
        num, den, target, target_index, H, W,
                                                       lam, l2, d_pixels, sums, tx, tx * ty);
    UGS_LAUNCH_CHECK("loss_tile_kernel");
    UGS_PDL(loss_reduce_kernel, 1, 32 * kReduceWarps, 0, st,
        sums, tx * ty, S, H, W, lam, l2, loss_out,
                                          ssim_out, loss_mean_out);
    UGS_LAUNCH_CHECK("loss_reduce_kernel");
    return UGS_OK;
}

extern "C" int ugs_loss(const float *num, const float *den, const float *target,
                        int S, int H, int W, double lam, int l2, float *d_pixels,
                        double *loss_out, double *ssim_out, void *workspace,
                        void *stream) {
    return ugs_loss_ex(num, den, target, nullptr, S, H, W, lam, l2, d_pixels, loss_out,
                       ssim_out, nullptr, workspace, stream);
}
