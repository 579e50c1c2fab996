// Per-Gaussian phase-1 geometry, bit-exact with the reference's float32
// numpy sequence (ref pkg/src/echosplat/rasterizer.py:109-137; SURVEY
// section 8 a4').  Every operation is an explicitly rounded intrinsic so nvcc
// can never contract or reassociate it.
#pragma once
#include "ugs_internal.cuh"

namespace ugs {

struct Factor {
    float L00, L10, L11, L20, L21, L22;   // build_L (model.py:101-118)
    float LT[3][3];                       // (L^-1)^T (model.py:121-138)
};

__device__ __forceinline__ Factor make_factor(const float *__restrict__ l_raw,
                                              int64_t g, float beta) {
    Factor f;
    const float *l = l_raw + 6 * g;
    float l0, l1, l2;
    if ((reinterpret_cast<uintptr_t>(l_raw) & 7) == 0) {   // rows of 24 B: float2 loads
        const float2 *l2p = reinterpret_cast<const float2 *>(l);
        const float2 a = __ldg(l2p), b = __ldg(l2p + 1), c = __ldg(l2p + 2);
        l0 = a.x; l1 = a.y; l2 = b.x;
        f.L10 = b.y; f.L20 = c.x; f.L21 = c.y;
    } else {
        l0 = __ldg(l + 0); l1 = __ldg(l + 1); l2 = __ldg(l + 2);
        f.L10 = __ldg(l + 3); f.L20 = __ldg(l + 4); f.L21 = __ldg(l + 5);
    }
    f.L00 = __fadd_rn(__fmul_rn(l0, l0), beta);
    f.L11 = __fadd_rn(__fmul_rn(l1, l1), beta);
    f.L22 = __fadd_rn(__fmul_rn(l2, l2), beta);
    float i00 = __fdiv_rn(1.0f, f.L00);
    float i11 = __fdiv_rn(1.0f, f.L11);
    float i22 = __fdiv_rn(1.0f, f.L22);
    float i10 = __fmul_rn(__fmul_rn(-f.L10, i00), i11);
    float i21 = __fmul_rn(__fmul_rn(-f.L21, i11), i22);
    float i20 = __fmul_rn(-__fadd_rn(__fmul_rn(f.L20, i00), __fmul_rn(f.L21, i10)), i22);
    f.LT[0][0] = i00; f.LT[0][1] = i10; f.LT[0][2] = i20;
    f.LT[1][0] = 0.f; f.LT[1][1] = i11; f.LT[1][2] = i21;
    f.LT[2][0] = 0.f; f.LT[2][1] = 0.f; f.LT[2][2] = i22;
    return f;
}

struct Window {
    int iu0, iu1, iv0, iv1;
};

// Returns true iff the Gaussian is accepted for this slice (straddles the
// plane, footprint meets the image rectangle, non-empty clamped window).
// Probe-frame box along axis i: mean_probe_i -/+ sqrt(cut) * ||(Rw L^-T)_i||.
__device__ __forceinline__ void box_axis(int i, const float mu[3], const Factor &f,
                                         const ugs_slice &sl, float &bmin, float &bmax) {
    // einsum order (a0 + a1) + a2 with LT = (L^-1)^T upper-triangular: the
    // terms with LT[j][k] == 0 are +-0 and adding +-0 leaves a sum unchanged
    // up to the sign of zero, which the squares below discard -- so dropping
    // them is bit-exact.
    const float r[3] = {
        __fmul_rn(sl.rw[3 * i + 0], f.LT[0][0]),
        __fadd_rn(__fmul_rn(sl.rw[3 * i + 0], f.LT[0][1]),
                  __fmul_rn(sl.rw[3 * i + 1], f.LT[1][1])),
        __fadd_rn(__fadd_rn(__fmul_rn(sl.rw[3 * i + 0], f.LT[0][2]),
                            __fmul_rn(sl.rw[3 * i + 1], f.LT[1][2])),
                  __fmul_rn(sl.rw[3 * i + 2], f.LT[2][2]))};
    float nrm = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(r[0], r[0]),
                                               __fmul_rn(r[1], r[1])),
                                     __fmul_rn(r[2], r[2])));
    float half = __fmul_rn(sl.sqrt_cut, nrm);
    // OpenBLAS sgemm (N,3)@(3,3): FMA chain, then + tw
    float mp = __fmaf_rn(mu[2], sl.rw[3 * i + 2],
                         __fmaf_rn(mu[1], sl.rw[3 * i + 1],
                                   __fmul_rn(mu[0], sl.rw[3 * i + 0])));
    mp = __fadd_rn(mp, sl.tw[i]);
    bmin = __fsub_rn(mp, half);
    bmax = __fadd_rn(mp, half);
}

// The plane-straddle test (axis z) rejects most Gaussians; it is evaluated
// on its own first.  Every axis is computed exactly as the reference does,
// so splitting the AND-ed test cannot change the outcome.
__device__ __forceinline__ bool straddles(const float mu[3], const Factor &f,
                                          const ugs_slice &sl) {
    float bmin, bmax;
    box_axis(2, mu, f, sl, bmin, bmax);
    return (bmin <= 0.0f) && (bmax >= 0.0f);
}

// In-plane overlap + clamped window of a Gaussian that straddles the plane.
__device__ __forceinline__ bool cull_window_xy(const float mu[3], const Factor &f,
                                               const ugs_slice &sl, Window &w) {
    float bmin[2], bmax[2];
    box_axis(0, mu, f, sl, bmin[0], bmax[0]);
    box_axis(1, mu, f, sl, bmin[1], bmax[1]);
    bool keep = (bmax[0] >= -sl.x1h) && (bmin[0] <= sl.x1h) &&
                (bmax[1] >= -sl.x2h) && (bmin[1] <= sl.x2h);
    if (!keep) return false;
    float fu0 = ceilf(__fadd_rn(__fdiv_rn(bmin[0], sl.s), sl.cx));
    float fu1 = floorf(__fadd_rn(__fdiv_rn(bmax[0], sl.s), sl.cx));
    float fv0 = ceilf(__fadd_rn(__fdiv_rn(bmin[1], sl.s), sl.cy));
    float fv1 = floorf(__fadd_rn(__fdiv_rn(bmax[1], sl.s), sl.cy));
    fu0 = fmaxf(fu0, 0.0f);
    fv0 = fmaxf(fv0, 0.0f);
    fu1 = fminf(fu1, (float)(sl.width - 1));
    fv1 = fminf(fv1, (float)(sl.height - 1));
    // accepted boxes overlap the image, so the clamped values are in range
    w.iu0 = (int)fu0;
    w.iu1 = (int)fu1;
    w.iv0 = (int)fv0;
    w.iv1 = (int)fv1;
    return (w.iu0 <= w.iu1) && (w.iv0 <= w.iv1);
}

__device__ __forceinline__ int window_tiles(const Window &w) {
    return ((w.iu1 >> 4) - (w.iu0 >> 4) + 1) * ((w.iv1 >> 4) - (w.iv0 >> 4) + 1);
}

__device__ __forceinline__ float sigmoid_f32(float x) {
    // numpy float32: 1.0 / (1.0 + exp(-x))   (model.py:27-28)
    return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-x)));
}

__device__ __forceinline__ double sigmoid_f64(double x) {
    return 1.0 / (1.0 + exp(-x));
}

// Plane-conditioned form of one accepted Gaussian on one slice (float64).
// With e(u,v) = origin + u du + v dv - mu and y = L^T e = c + u a + v b
// (a = L^T du, b = L^T dv, c = L^T (origin - mu)), the reference's q = |y|^2
// is a 2-D quadratic in the pixel coordinates.  Around any integer pixel
// (pu, pv), with y_p = y(pu, pv) and exact integer offsets x = u - pu,
// y = v - pv:
//   q = H00 x^2 + 2 H01 x y + H11 y^2 + 2 (a.y_p) x + 2 (b.y_p) y + |y_p|^2.
// plane_form computes H and the record's reference pixel (ui, vi): the
// in-plane conditional mean rounded and clamped to the window (the window
// centre when the in-plane precision is singular or ill-conditioned);
// expansion() gives the linear/constant terms at a pixel.  Expanding each
// tile instance around the point of its rectangle nearest (ui, vi) keeps the
// float32 terms bounded by H times the tile size: no cancellation however
// large or anisotropic the Gaussian (the reference evaluates every pair in
// float64, _kernels.py:34-45).
struct PlaneForm {
    double H00, H01, H11;
    double a[3], b[3], c[3];
    int ui, vi;            // reference pixel
};

__device__ __forceinline__ void lt_mul(const Factor &f, const double x[3],
                                       double y[3]) {
    // y = L^T x, L lower-triangular
    y[0] = (double)f.L00 * x[0] + (double)f.L10 * x[1] + (double)f.L20 * x[2];
    y[1] = (double)f.L11 * x[1] + (double)f.L21 * x[2];
    y[2] = (double)f.L22 * x[2];
}

__device__ __forceinline__ PlaneForm plane_form(const float mu[3],
                                                const Factor &f,
                                                const ugs_slice &sl,
                                                const Window &w) {
    PlaneForm P;
    double du[3] = {sl.du[0], sl.du[1], sl.du[2]};
    double dv[3] = {sl.dv[0], sl.dv[1], sl.dv[2]};
    double d[3] = {(double)sl.origin[0] - mu[0], (double)sl.origin[1] - mu[1],
                   (double)sl.origin[2] - mu[2]};
    lt_mul(f, du, P.a);
    lt_mul(f, dv, P.b);
    lt_mul(f, d, P.c);
    P.H00 = P.a[0] * P.a[0] + P.a[1] * P.a[1] + P.a[2] * P.a[2];
    P.H01 = P.a[0] * P.b[0] + P.a[1] * P.b[1] + P.a[2] * P.b[2];
    P.H11 = P.b[0] * P.b[0] + P.b[1] * P.b[1] + P.b[2] * P.b[2];
    const double h0 = P.a[0] * P.c[0] + P.a[1] * P.c[1] + P.a[2] * P.c[2];
    const double h1 = P.b[0] * P.c[0] + P.b[1] * P.c[1] + P.b[2] * P.c[2];
    const double det = P.H00 * P.H11 - P.H01 * P.H01;
    double us = 0.5 * (double)(w.iu0 + w.iu1), vs = 0.5 * (double)(w.iv0 + w.iv1);
    if (det > 1e-12 * P.H00 * P.H11) {
        const double u1 = (P.H01 * h1 - P.H11 * h0) / det;
        const double v1 = (P.H01 * h0 - P.H00 * h1) / det;
        if (isfinite(u1) && isfinite(v1)) { us = u1; vs = v1; }
    }
    P.ui = (int)fmin(fmax(rint(us), (double)w.iu0), (double)w.iu1);
    P.vi = (int)fmin(fmax(rint(vs), (double)w.iv0), (double)w.iv1);
    return P;
}

// Linear and constant exponent terms (log2 domain, kq = -log2(e)/2, log2
// alpha folded into F) around pixel (pu, pv).
__device__ __forceinline__ void expansion(const PlaneForm &P, int pu, int pv, double kq,
                                          double log2a, double &D, double &E, double &F) {
    double y[3];
    for (int k = 0; k < 3; ++k) y[k] = P.c[k] + (double)pu * P.a[k] + (double)pv * P.b[k];
    D = 2.0 * kq * (P.a[0] * y[0] + P.a[1] * y[1] + P.a[2] * y[2]);
    E = 2.0 * kq * (P.b[0] * y[0] + P.b[1] * y[1] + P.b[2] * y[2]);
    F = kq * (y[0] * y[0] + y[1] * y[1] + y[2] * y[2]) + log2a;
}

// Clipped rectangle of window w in the tile whose pixel origin is (tu0, tv0),
// and that rectangle's expansion pixel (ui, vi) clamped into it.
struct TileRect {
    int x0, x1, y0, y1;    // absolute pixel coordinates, inclusive
    int pu, pv;
};

__device__ __forceinline__ TileRect tile_rect(int iu0, int iu1, int iv0, int iv1,
                                              int tu0, int tv0, int ui, int vi) {
    TileRect t;
    t.x0 = max(iu0, tu0);
    t.x1 = min(iu1, tu0 + kTile - 1);
    t.y0 = max(iv0, tv0);
    t.y1 = min(iv1, tv0 + kTile - 1);
    t.pu = min(max(ui, t.x0), t.x1);
    t.pv = min(max(vi, t.y0), t.y1);
    return t;
}

// Decoded Frag rectangle (tile-relative, inclusive).
struct FragRect {
    int x0, x1, y0, y1, pu, pv;
};
__device__ __forceinline__ FragRect frag_rect(float bits_f) {
    const unsigned b = (unsigned)__float_as_int(bits_f);
    FragRect r;
    r.x0 = b & 15;
    r.x1 = (b >> 4) & 15;
    r.y0 = (b >> 8) & 15;
    r.y1 = (b >> 12) & 15;
    r.pu = (b >> 16) & 15;
    r.pv = (b >> 20) & 15;
    return r;
}

}  // namespace ugs
