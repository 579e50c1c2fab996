// Per-Gaussian Adam update shared by the standalone Adam kernel and the fused
// backward -> accumulate -> stats -> Adam kernel.
//
// Gradient / moment layout ("AoS-12"): Gaussian g owns 12 consecutive floats
//   [d_means 0..2 | d_l_raw 3..8 | d_intensity_raw 9 | d_opacity_raw 10 | pad]
// and the two background entries follow at [12 n, 12 n + 1].  One record of
// the backward is then three float4 read-modify-writes.
//
// The arithmetic reproduces the reference's numpy rounding sequence exactly
// (ref trainer.py:182-199; the oracle's ugo_adam_group):
//   m = f32(m*f32(b1)) + f32(f32(1-b1)*g)          (f32)
//   v = f32(f64(f32(v*f32(b2))) + (1-b2)*f64(g)^2) (f64 add, one rounding)
//   upd = f32(f32(lr)*f32(m/f32(bc1))) / f32(sqrt(f32(v/f32(bc2))) + f32(eps))
// with explicitly rounded intrinsics only, so no build flag can contract it.
#pragma once
#include "ugs_internal.cuh"

namespace ugs {

constexpr int kG = 12;   // floats per Gaussian in the AoS gradient / moments

struct AdamConst {
    float b1, one_m_b1, b2, bc1, bc2, eps;
    double one_m_b2;
    float lr[5];   // means, l_raw, intensity, opacity, bg
};

inline AdamConst make_adam_const(int64_t t, const double *lr, double beta1,
                                 double beta2, double eps) {
    AdamConst k;
    k.b1 = (float)beta1;
    k.one_m_b1 = (float)(1.0 - beta1);
    k.b2 = (float)beta2;
    k.one_m_b2 = 1.0 - beta2;
    k.bc1 = (float)(1.0 - pow(beta1, (double)t));
    k.bc2 = (float)(1.0 - pow(beta2, (double)t));
    k.eps = (float)eps;
    for (int i = 0; i < 5; ++i) k.lr[i] = (float)lr[i];
    return k;
}

__device__ __forceinline__ float adam_update(float g, float &m, float &v,
                                             const AdamConst &k, float lr) {
    const float mi = __fadd_rn(__fmul_rn(m, k.b1), __fmul_rn(k.one_m_b1, g));
    float vi = __fmul_rn(v, k.b2);
    const double gd = (double)g;
    vi = (float)__dadd_rn((double)vi, __dmul_rn(k.one_m_b2, __dmul_rn(gd, gd)));
    m = mi;
    v = vi;
    // a zero numerator short-cuts the IEEE division exactly (0/x = 0 with
    // the numerator's sign for x > 0); rows that have never seen a gradient
    // (m = v = 0) would otherwise take the division's slow path (x = eps)
    const float mh = mi == 0.f ? mi : __fdiv_rn(mi, k.bc1);
    const float vh = vi == 0.f ? vi : __fdiv_rn(vi, k.bc2);
    const float num = __fmul_rn(lr, mh);
    return num == 0.f ? num : __fdiv_rn(num, __fadd_rn(__fsqrt_rn(vh), k.eps));
}

// ||d_means|| as numpy computes it for float32 rows: sqrt((x^2 + y^2) + z^2)
__device__ __forceinline__ float norm3_f32(float x, float y, float z) {
    return __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y)),
                                __fmul_rn(z, z)));
}

struct CloudMut {
    float *means, *l_raw, *intensity_raw, *opacity_raw;
};

// Optimizer state handed to the fused backward (ugs_backward_adam).
struct AdamArgs {
    float *m, *v;            // AoS-12 moments (+ 2 background entries)
    AdamConst k;
    float *grad_sum;         // densify statistics (both may be null)
    int32_t *grad_cnt;
};

// Adam on one Gaussian's row held in registers: parameters pr[11] in the
// AoS-12 order, moments mm / vv.
__device__ __forceinline__ void adam_row(const float gr[kG], float pr[11], float mm[kG],
                                         float vv[kG], const AdamConst &k) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
        pr[c] = __fsub_rn(pr[c], adam_update(gr[c], mm[c], vv[c], k, k.lr[0]));
#pragma unroll
    for (int c = 0; c < 6; ++c)
        pr[3 + c] = __fsub_rn(pr[3 + c], adam_update(gr[3 + c], mm[3 + c], vv[3 + c], k,
                                                     k.lr[1]));
    pr[9] = __fsub_rn(pr[9], adam_update(gr[9], mm[9], vv[9], k, k.lr[2]));
    pr[10] = __fsub_rn(pr[10], adam_update(gr[10], mm[10], vv[10], k, k.lr[3]));
}

// Adam on Gaussian g given its 11 gradient entries; m, v point at the
// Gaussian's AoS-12 rows.  Optional densify statistics (trainer.py:399-401).
// Every load first (parameters, moments, statistics), then the math, then
// every store: the parameter arrays are distinct but not __restrict__, so an
// interleaved load-update-store sequence would serialise the round trips.
__device__ __forceinline__ void adam_gaussian(int64_t g, const float gr[kG],
                                              float *__restrict__ m,
                                              float *__restrict__ v,
                                              const CloudMut &p,
                                              const AdamConst &k, bool touched,
                                              float *grad_sum, int32_t *grad_cnt) {
    float pr[11];
#pragma unroll
    for (int c = 0; c < 3; ++c) pr[c] = p.means[3 * g + c];
#pragma unroll
    for (int c = 0; c < 6; ++c) pr[3 + c] = p.l_raw[6 * g + c];
    pr[9] = p.intensity_raw[g];
    pr[10] = p.opacity_raw[g];
    float4 *m4 = reinterpret_cast<float4 *>(m), *v4 = reinterpret_cast<float4 *>(v);
    float mm[kG], vv[kG];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const float4 a = m4[q], b = v4[q];
        mm[4 * q] = a.x; mm[4 * q + 1] = a.y; mm[4 * q + 2] = a.z; mm[4 * q + 3] = a.w;
        vv[4 * q] = b.x; vv[4 * q + 1] = b.y; vv[4 * q + 2] = b.z; vv[4 * q + 3] = b.w;
    }
    const bool stats = touched && grad_sum;
    float gs = 0.f;
    int32_t gc = 0;
    if (stats) {
        gs = grad_sum[g];
        gc = grad_cnt[g];
    }
    adam_row(gr, pr, mm, vv, k);
    if (stats) {
        grad_sum[g] = __fadd_rn(gs, norm3_f32(gr[0], gr[1], gr[2]));
        grad_cnt[g] = gc + 1;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) p.means[3 * g + c] = pr[c];
#pragma unroll
    for (int c = 0; c < 6; ++c) p.l_raw[6 * g + c] = pr[3 + c];
    p.intensity_raw[g] = pr[9];
    p.opacity_raw[g] = pr[10];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        m4[q] = make_float4(mm[4 * q], mm[4 * q + 1], mm[4 * q + 2], mm[4 * q + 3]);
        v4[q] = make_float4(vv[4 * q], vv[4 * q + 1], vv[4 * q + 2], vv[4 * q + 3]);
    }
}

// Background group: python-float parameters updated as
// float(f32(f32(raw) - upd)) (NEP 50: python float - np.float32 -> float32).
__device__ __forceinline__ void adam_bg(double *bg_raw, const float *g, float *m,
                                        float *v, const AdamConst &k) {
    for (int i = 0; i < 2; ++i) {
        float mm = m[i], vv = v[i];
        const float upd = adam_update(g[i], mm, vv, k, k.lr[4]);
        m[i] = mm;
        v[i] = vv;
        bg_raw[i] = (double)__fsub_rn((float)bg_raw[i], upd);
    }
}

}  // namespace ugs
