/*
 * ORACLE -- test infrastructure only.  CPU restatement of the reference
 * (echosplat, arXiv 2505.05643) hot path, used as the parity checker by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg.  Nothing in the product path links or calls this file.
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py -> the tests/golden npz files, checked by
 * tests/test_oracle_golden.py).
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC (see
 * oracle/Makefile).  -ffp-contract=off matters: the reference computes every
 * elementwise expression without FMA contraction (numpy ufuncs, numba with
 * fastmath=False), except the (N,3)@(3,3) matmul which OpenBLAS runs as an
 * FMA chain (written with explicit fmaf below).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

/*
 * Phase 1 of rendering: build_L + invert_lower_triangular + probe-frame
 * chi^2 boxes + cull + compact + clamped pixel windows.
 *   ref: pkg/src/echosplat/rasterizer.py:109-137 (_prepare),
 *        rasterizer.py:77-80 (_boxes_vectorized), :83-101 (cull),
 *        :104-106 (compact), model.py:101-118 (build_L),
 *        model.py:121-138 (invert_lower_triangular).
 * All arithmetic is float32 with the reference's operation order:
 *   build_L:  Ljj = f32(l*l) + f32(beta)
 *   inverse:  i_jj = 1/L_jj; i10 = ((-L10)*i00)*i11; i21 = ((-L21)*i11)*i22;
 *             i20 = (-((L20*i00) + (L21*i10)))*i22
 *   rows = einsum('ij,njk->nik', Rw, Linv^T): (a0 + a1) + a2, unfused
 *   norm = sqrt((r0^2 + r1^2) + r2^2), unfused
 *   mean_probe = means @ Rw^T + tw: fma(m2,R[j2],fma(m1,R[j1],m0*R[j0])) + tw
 *   window: ceil(f32(b/s) + cx) etc. with f32 s, cx, cy.
 * Outputs: accepted (ascending int64), windows[m][4] = iu0,iu1,iv0,iv1,
 * Ls (n,3,3) row-major lower-triangular factors (may be NULL).
 * Returns the accepted count m.
 */
int64_t ugo_prepare(int64_t n, const float *means, const float *l_raw,
                    float beta, const float *rw, const float *tw,
                    float sqrt_cut, float s, float cx, float cy, float x1h,
                    float x2h, int32_t width, int32_t height,
                    int64_t *accepted, int64_t *windows, float *Ls)
{
    int64_t m = 0;
    for (int64_t g = 0; g < n; ++g) {
        const float *l = l_raw + 6 * g;
        float L00 = l[0] * l[0] + beta;
        float L11 = l[1] * l[1] + beta;
        float L22 = l[2] * l[2] + beta;
        float L10 = l[3], L20 = l[4], L21 = l[5];
        if (Ls) {
            float *o = Ls + 9 * g;
            o[0] = L00; o[1] = 0.f; o[2] = 0.f;
            o[3] = L10; o[4] = L11; o[5] = 0.f;
            o[6] = L20; o[7] = L21; o[8] = L22;
        }
        float i00 = 1.0f / L00, i11 = 1.0f / L11, i22 = 1.0f / L22;
        float i10 = ((-L10) * i00) * i11;
        float i21 = ((-L21) * i11) * i22;
        float i20 = (-((L20 * i00) + (L21 * i10))) * i22;
        /* LT[j][k] = Linv[k][j] */
        float LT[3][3] = {{i00, i10, i20}, {0.f, i11, i21}, {0.f, 0.f, i22}};
        const float *mu = means + 3 * g;
        float bmin[3], bmax[3];
        for (int i = 0; i < 3; ++i) {
            float r[3];
            for (int k = 0; k < 3; ++k) {
                float a0 = rw[3 * i + 0] * LT[0][k];
                float a1 = rw[3 * i + 1] * LT[1][k];
                float a2 = rw[3 * i + 2] * LT[2][k];
                r[k] = (a0 + a1) + a2;
            }
            float sq0 = r[0] * r[0], sq1 = r[1] * r[1], sq2 = r[2] * r[2];
            float nrm = sqrtf((sq0 + sq1) + sq2);
            float half = sqrt_cut * nrm;
            float mp = fmaf(mu[2], rw[3 * i + 2],
                            fmaf(mu[1], rw[3 * i + 1], mu[0] * rw[3 * i + 0]));
            mp = mp + tw[i];
            bmin[i] = mp - half;
            bmax[i] = mp + half;
        }
        int keep = (bmin[2] <= 0.0f) && (bmax[2] >= 0.0f) &&
                   (bmax[0] >= -x1h) && (bmin[0] <= x1h) &&
                   (bmax[1] >= -x2h) && (bmin[1] <= x2h);
        if (!keep) continue;
        float fu0 = ceilf(bmin[0] / s + cx);
        float fu1 = floorf(bmax[0] / s + cx);
        float fv0 = ceilf(bmin[1] / s + cy);
        float fv1 = floorf(bmax[1] / s + cy);
        if (fu0 < 0.f) fu0 = 0.f;
        if (fv0 < 0.f) fv0 = 0.f;
        if (fu1 > (float)(width - 1)) fu1 = (float)(width - 1);
        if (fv1 > (float)(height - 1)) fv1 = (float)(height - 1);
        int64_t iu0 = (int64_t)fu0, iu1 = (int64_t)fu1;
        int64_t iv0 = (int64_t)fv0, iv1 = (int64_t)fv1;
        if (iu0 > iu1 || iv0 > iv1) continue;
        accepted[m] = g;
        windows[4 * m + 0] = iu0;
        windows[4 * m + 1] = iu1;
        windows[4 * m + 2] = iv0;
        windows[4 * m + 3] = iv1;
        ++m;
    }
    return m;
}

/*
 * forward_kernel restated (ref: pkg/src/echosplat/_kernels.py:19-47).
 * numba types px/e/y/q/w as float64 (int64 pixel index * float32 step
 * promotes to float64); the f32 accumulators are rounded after every add.
 * Inputs are the compacted (gathered) per-Gaussian arrays; windows[m][4].
 */
void ugo_forward(int64_t m, const float *means, const float *Ls,
                 const float *colors, const float *alphas,
                 const int64_t *windows, const float *origin, const float *du,
                 const float *dv, int32_t width, float *num, float *den)
{
    for (int64_t g = 0; g < m; ++g) {
        double mx = means[3 * g], my = means[3 * g + 1], mz = means[3 * g + 2];
        const float *L = Ls + 9 * g;
        double l00 = L[0], l10 = L[3], l11 = L[4], l20 = L[6], l21 = L[7],
               l22 = L[8];
        double c = colors[g], a = alphas[g];
        int64_t iu0 = windows[4 * g], iu1 = windows[4 * g + 1];
        int64_t iv0 = windows[4 * g + 2], iv1 = windows[4 * g + 3];
        for (int64_t v = iv0; v <= iv1; ++v) {
            double px = (double)origin[0] + (double)v * (double)dv[0];
            double py = (double)origin[1] + (double)v * (double)dv[1];
            double pz = (double)origin[2] + (double)v * (double)dv[2];
            for (int64_t u = iu0; u <= iu1; ++u) {
                double e0 = (px + (double)u * (double)du[0]) - mx;
                double e1 = (py + (double)u * (double)du[1]) - my;
                double e2 = (pz + (double)u * (double)du[2]) - mz;
                double y0 = (l00 * e0 + l10 * e1) + l20 * e2;
                double y1 = l11 * e1 + l21 * e2;
                double y2 = l22 * e2;
                double q = (y0 * y0 + y1 * y1) + y2 * y2;
                double w = a * exp(-0.5 * q);
                int64_t p = v * width + u;
                num[p] = (float)((double)num[p] + w * c);
                den[p] = (float)((double)den[p] + w);
            }
        }
    }
}

/*
 * backward_kernel restated (ref: pkg/src/echosplat/_kernels.py:50-101).
 * Same typing as numba: (c - chat) and gpix*(c - chat) are float32, the
 * rest float64; accumulators f32.  d_L is (m,3,3) row-major.
 */
void ugo_backward(int64_t m, const float *means, const float *Ls,
                  const float *colors, const float *alphas,
                  const int64_t *windows, const float *origin, const float *du,
                  const float *dv, int32_t width, const float *chat,
                  const float *ssum, const float *dpix, float *d_mu,
                  float *d_L, float *d_c, float *d_a)
{
    for (int64_t g = 0; g < m; ++g) {
        double mx = means[3 * g], my = means[3 * g + 1], mz = means[3 * g + 2];
        const float *L = Ls + 9 * g;
        double l00 = L[0], l10 = L[3], l11 = L[4], l20 = L[6], l21 = L[7],
               l22 = L[8];
        float cf = colors[g];
        double a = alphas[g];
        int64_t iu0 = windows[4 * g], iu1 = windows[4 * g + 1];
        int64_t iv0 = windows[4 * g + 2], iv1 = windows[4 * g + 3];
        float *dm = d_mu + 3 * g, *dL = d_L + 9 * g;
        for (int64_t v = iv0; v <= iv1; ++v) {
            double px = (double)origin[0] + (double)v * (double)dv[0];
            double py = (double)origin[1] + (double)v * (double)dv[1];
            double pz = (double)origin[2] + (double)v * (double)dv[2];
            for (int64_t u = iu0; u <= iu1; ++u) {
                int64_t p = v * width + u;
                float gpix = dpix[p];
                if (gpix == 0.0f) continue;
                double e0 = (px + (double)u * (double)du[0]) - mx;
                double e1 = (py + (double)u * (double)du[1]) - my;
                double e2 = (pz + (double)u * (double)du[2]) - mz;
                double y0 = (l00 * e0 + l10 * e1) + l20 * e2;
                double y1 = l11 * e1 + l21 * e2;
                double y2 = l22 * e2;
                double q = (y0 * y0 + y1 * y1) + y2 * y2;
                double expq = exp(-0.5 * q);
                double w = a * expq;
                double inv_s = 1.0 / (double)ssum[p];
                d_c[g] = (float)((double)d_c[g] + ((double)gpix * w) * inv_s);
                float gdiff = gpix * (cf - chat[p]);
                double dw = (double)gdiff * inv_s;
                d_a[g] = (float)((double)d_a[g] + dw * expq);
                double dq = (-0.5 * w) * dw;
                double r0 = l00 * y0;
                double r1 = l10 * y0 + l11 * y1;
                double r2 = (l20 * y0 + l21 * y1) + l22 * y2;
                dm[0] = (float)((double)dm[0] + (-2.0 * dq) * r0);
                dm[1] = (float)((double)dm[1] + (-2.0 * dq) * r1);
                dm[2] = (float)((double)dm[2] + (-2.0 * dq) * r2);
                double t = 2.0 * dq;
                dL[0] = (float)((double)dL[0] + (t * e0) * y0);
                dL[3] = (float)((double)dL[3] + (t * e1) * y0);
                dL[4] = (float)((double)dL[4] + (t * e1) * y1);
                dL[6] = (float)((double)dL[6] + (t * e2) * y0);
                dL[7] = (float)((double)dL[7] + (t * e2) * y1);
                dL[8] = (float)((double)dL[8] + (t * e2) * y2);
            }
        }
    }
}

/*
 * One Adam update of a float32 group, bit-for-bit the reference's numpy
 * sequence (ref: pkg/src/echosplat/trainer.py:170-200):
 *   m = f32(m*f32(b1)); m = f32(m + f32(f32(1-b1)*g))
 *   v = f32(v*f32(b2)); v = f32(f64(v) + (1-b2)*f64(g)^2)
 *   upd = f32(f32(lr)*f32(m/f32(1-b1^t))) / f32(sqrt(f32(v/f32(1-b2^t))) + f32(eps))
 *   p -= upd
 * p may be NULL (the background group, applied by the caller).
 */
void ugo_adam_group(int64_t n, float *p, const float *g, float *m, float *v,
                    double lr, int64_t t, double beta1, double beta2,
                    double eps, float *upd_out)
{
    float b1 = (float)beta1, b2 = (float)beta2;
    float one_m_b1 = (float)(1.0 - beta1);
    double one_m_b2 = 1.0 - beta2;
    float bc1 = (float)(1.0 - pow(beta1, (double)t));
    float bc2 = (float)(1.0 - pow(beta2, (double)t));
    float lrf = (float)lr, epsf = (float)eps;
    for (int64_t i = 0; i < n; ++i) {
        float mi = m[i] * b1;
        mi = mi + one_m_b1 * g[i];
        float vi = v[i] * b2;
        double gd = (double)g[i];
        vi = (float)((double)vi + one_m_b2 * (gd * gd));
        m[i] = mi;
        v[i] = vi;
        float mh = mi / bc1;
        float vh = vi / bc2;
        float upd = (lrf * mh) / (sqrtf(vh) + epsf);
        if (p) p[i] = p[i] - upd;
        if (upd_out) upd_out[i] = upd;
    }
}
