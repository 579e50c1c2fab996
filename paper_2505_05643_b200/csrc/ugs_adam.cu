// Fused Adam over the parameter SoA, densify statistics and densify/prune
// row surgery.
//
// Adam is an HBM stream: per element it reads p, g, m, v and writes p, m, v
// (and optionally zeroes g): 28-32 B/element, 308-352 B/Gaussian.  The
// arithmetic reproduces the reference's numpy rounding sequence exactly
// (ref trainer.py:182-199, see ugo_adam_group in the oracle):
//   m = f32(m*f32(b1)) + f32(f32(1-b1)*g)          (f32)
//   v = f32(f64(f32(v*f32(b2))) + (1-b2)*f64(g)^2) (f64 add, one rounding)
//   upd = f32(f32(lr)*f32(m/f32(bc1))) / f32(sqrt(f32(v/f32(bc2))) + f32(eps))
// so every multiply/add is an explicitly rounded intrinsic (no contraction).
#include "ugs_geometry.cuh"

namespace ugs {

namespace {

struct AdamConst {
    float b1, one_m_b1, b2, bc1, bc2, eps;
    double one_m_b2;
    float lr[5];
};

__device__ __forceinline__ float adam_update(float g, float &m, float &v,
                                             const AdamConst &k, float lr) {
    float mi = __fadd_rn(__fmul_rn(m, k.b1), __fmul_rn(k.one_m_b1, g));
    float vi = __fmul_rn(v, k.b2);
    const double gd = (double)g;
    vi = (float)__dadd_rn((double)vi, __dmul_rn(k.one_m_b2, __dmul_rn(gd, gd)));
    m = mi;
    v = vi;
    const float mh = __fdiv_rn(mi, k.bc1);
    const float vh = __fdiv_rn(vi, k.bc2);
    return __fdiv_rn(__fmul_rn(lr, mh), __fadd_rn(__fsqrt_rn(vh), k.eps));
}

// One thread per float4 of a group (vectorised stream); scalar tail.
__global__ void adam_group_kernel(float *__restrict__ p, float *__restrict__ g,
                                  float *__restrict__ m, float *__restrict__ v,
                                  int64_t count, AdamConst k, float lr,
                                  int zero_grad, int use_vec) {
    const int64_t n4 = use_vec ? (count >> 2) : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += stride) {
        float4 pp = reinterpret_cast<float4 *>(p)[i];
        float4 gg = reinterpret_cast<float4 *>(g)[i];
        float4 mm = reinterpret_cast<float4 *>(m)[i];
        float4 vv = reinterpret_cast<float4 *>(v)[i];
        pp.x = __fsub_rn(pp.x, adam_update(gg.x, mm.x, vv.x, k, lr));
        pp.y = __fsub_rn(pp.y, adam_update(gg.y, mm.y, vv.y, k, lr));
        pp.z = __fsub_rn(pp.z, adam_update(gg.z, mm.z, vv.z, k, lr));
        pp.w = __fsub_rn(pp.w, adam_update(gg.w, mm.w, vv.w, k, lr));
        reinterpret_cast<float4 *>(p)[i] = pp;
        reinterpret_cast<float4 *>(m)[i] = mm;
        reinterpret_cast<float4 *>(v)[i] = vv;
        if (zero_grad) reinterpret_cast<float4 *>(g)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
         i < count; i += stride) {
        float mm = m[i], vv = v[i];
        p[i] = __fsub_rn(p[i], adam_update(g[i], mm, vv, k, lr));
        m[i] = mm;
        v[i] = vv;
        if (zero_grad) g[i] = 0.f;
    }
}

// Background group: python-float parameters updated as
// float(f32(f32(raw) - upd)) (NEP 50: python float - np.float32 -> float32).
__global__ void adam_bg_kernel(double *bg_raw, float *g, float *m, float *v,
                               AdamConst k, int zero_grad) {
    const int i = threadIdx.x;
    if (i >= 2) return;
    float mm = m[i], vv = v[i];
    const float upd = adam_update(g[i], mm, vv, k, k.lr[4]);
    m[i] = mm;
    v[i] = vv;
    bg_raw[i] = (double)__fsub_rn((float)bg_raw[i], upd);
    if (zero_grad) g[i] = 0.f;
}

// trainer.py:399-401: norms = ||d_means|| (f32, ((x^2+y^2)+z^2)),
// grad_sum[acc] += norms[acc]; grad_cnt[acc] += 1.
__global__ void grad_stats_kernel(const float *__restrict__ grad, int64_t n,
                                  uint8_t *__restrict__ touched,
                                  float *__restrict__ grad_sum,
                                  int32_t *__restrict__ grad_cnt) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n || !touched[g]) return;
    const float x = grad[3 * g], y = grad[3 * g + 1], z = grad[3 * g + 2];
    const float nrm = __fsqrt_rn(__fadd_rn(__fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y)),
                                           __fmul_rn(z, z)));
    grad_sum[g] = __fadd_rn(grad_sum[g], nrm);
    grad_cnt[g] += 1;
    touched[g] = 0;
}

// ---- densify / prune --------------------------------------------------
// flat moment layout: [means 3n | l_raw 6n | intensity n | opacity n | bg 2]
__global__ void densify_keep_kernel(const ugs_cloud src, const float *__restrict__ m_src,
                                    const float *__restrict__ v_src,
                                    const int32_t *__restrict__ keep, int64_t n_keep,
                                    int64_t n_dst, float *__restrict__ means,
                                    float *__restrict__ l_raw,
                                    float *__restrict__ c_raw, float *__restrict__ a_raw,
                                    float *__restrict__ m_dst, float *__restrict__ v_dst) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n_keep) return;
    const int64_t i = keep[j];
    const int64_t ns = src.n;
    for (int k = 0; k < 3; ++k) {
        means[3 * j + k] = src.means[3 * i + k];
        m_dst[3 * j + k] = m_src[3 * i + k];
        v_dst[3 * j + k] = v_src[3 * i + k];
    }
    for (int k = 0; k < 6; ++k) {
        l_raw[6 * j + k] = src.l_raw[6 * i + k];
        m_dst[3 * n_dst + 6 * j + k] = m_src[3 * ns + 6 * i + k];
        v_dst[3 * n_dst + 6 * j + k] = v_src[3 * ns + 6 * i + k];
    }
    c_raw[j] = src.intensity_raw[i];
    a_raw[j] = src.opacity_raw[i];
    m_dst[9 * n_dst + j] = m_src[9 * ns + i];
    v_dst[9 * n_dst + j] = v_src[9 * ns + i];
    m_dst[10 * n_dst + j] = m_src[10 * ns + i];
    v_dst[10 * n_dst + j] = v_src[10 * ns + i];
    if (j < 2) {
        m_dst[11 * n_dst + j] = m_src[11 * ns + j];
        v_dst[11 * n_dst + j] = v_src[11 * ns + j];
    }
}

// Sequential over candidates is unnecessary: each candidate touches its own
// parent row and its own appended row (model.py:147-152, trainer.py:255-272).
__global__ void densify_new_kernel(const int32_t *__restrict__ cand,
                                   const uint8_t *__restrict__ split,
                                   const double *__restrict__ z, int64_t n_new,
                                   int64_t n_keep, int64_t n_dst, double beta,
                                   double f, float *__restrict__ means,
                                   float *__restrict__ l_raw,
                                   float *__restrict__ c_raw, float *__restrict__ a_raw,
                                   float *__restrict__ m_dst, float *__restrict__ v_dst) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_new) return;
    const int64_t gi = cand[c];
    const int64_t dst = n_keep + c;
    float nm[3], nl[6];
    if (split[c]) {
        double l[6];
        for (int k = 0; k < 6; ++k) l[k] = (double)l_raw[6 * gi + k];
        double ln[6];
        for (int k = 0; k < 3; ++k) ln[k] = sqrt(f * (l[k] * l[k] + beta) - beta);
        const double sf = sqrt(f);
        for (int k = 3; k < 6; ++k) ln[k] = sf * l[k];
        // parent L (float64, build_L) and its inverse by forward substitution
        const double L00 = l[0] * l[0] + beta, L11 = l[1] * l[1] + beta,
                     L22 = l[2] * l[2] + beta;
        const double L10 = l[3], L20 = l[4], L21 = l[5];
        const double i00 = 1.0 / L00, i11 = 1.0 / L11, i22 = 1.0 / L22;
        const double i10 = -L10 * i00 * i11;
        const double i21 = -L21 * i11 * i22;
        const double i20 = -(L20 * i00 + L21 * i10) * i22;
        const double mu[3] = {means[3 * gi], means[3 * gi + 1], means[3 * gi + 2]};
        double ch[2][3];
        for (int q = 0; q < 2; ++q) {
            const double *zz = z + 6 * c + 3 * q;
            // y = mu + Linv^T z, Linv lower: (Linv^T z)_k = sum_{j>=k} Linv[j][k] z_j
            ch[q][0] = mu[0] + (i00 * zz[0] + i10 * zz[1] + i20 * zz[2]);
            ch[q][1] = mu[1] + (i11 * zz[1] + i21 * zz[2]);
            ch[q][2] = mu[2] + (i22 * zz[2]);
        }
        for (int k = 0; k < 3; ++k) {
            means[3 * gi + k] = (float)ch[0][k];
            nm[k] = (float)ch[1][k];
        }
        for (int k = 0; k < 6; ++k) {
            nl[k] = (float)ln[k];
        }
        // parent row update happens after its own values were read above;
        // no other candidate reads row gi.
        for (int k = 0; k < 6; ++k) l_raw[6 * gi + k] = nl[k];
    } else {
        for (int k = 0; k < 3; ++k) nm[k] = means[3 * gi + k];
        for (int k = 0; k < 6; ++k) nl[k] = l_raw[6 * gi + k];
    }
    for (int k = 0; k < 3; ++k) means[3 * dst + k] = nm[k];
    for (int k = 0; k < 6; ++k) l_raw[6 * dst + k] = nl[k];
    c_raw[dst] = c_raw[gi];
    a_raw[dst] = a_raw[gi];
    for (int k = 0; k < 3; ++k) { m_dst[3 * dst + k] = 0.f; v_dst[3 * dst + k] = 0.f; }
    for (int k = 0; k < 6; ++k) {
        m_dst[3 * n_dst + 6 * dst + k] = 0.f;
        v_dst[3 * n_dst + 6 * dst + k] = 0.f;
    }
    m_dst[9 * n_dst + dst] = 0.f; v_dst[9 * n_dst + dst] = 0.f;
    m_dst[10 * n_dst + dst] = 0.f; v_dst[10 * n_dst + dst] = 0.f;
}

int grid_for(int64_t n, int th) {
    int64_t b = (n + th - 1) / th;
    if (b > 148 * 16) b = 148 * 16;
    return b < 1 ? 1 : (int)b;
}

}  // namespace

}  // namespace ugs

using namespace ugs;

extern "C" int ugs_adam_step(float *means, float *l_raw, float *intensity_raw,
                             float *opacity_raw, double *bg_raw, float *grad,
                             float *m, float *v, int64_t n, int64_t t,
                             const double *lr, double beta1, double beta2,
                             double eps, int zero_grad, void *stream) {
    if (n < 0 || t < 1 || !lr) {
        set_error("ugs_adam_step: invalid arguments");
        return UGS_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    AdamConst k;
    k.b1 = (float)beta1;
    k.one_m_b1 = (float)(1.0 - beta1);
    k.b2 = (float)beta2;
    k.one_m_b2 = 1.0 - beta2;
    k.bc1 = (float)(1.0 - pow(beta1, (double)t));
    k.bc2 = (float)(1.0 - pow(beta2, (double)t));
    k.eps = (float)eps;
    for (int i = 0; i < 5; ++i) k.lr[i] = (float)lr[i];
    const int th = 256;
    struct G { float *p; int64_t off, cnt; int lri; } groups[4] = {
        {means, 0, 3 * n, 0}, {l_raw, 3 * n, 6 * n, 1},
        {intensity_raw, 9 * n, n, 2}, {opacity_raw, 10 * n, n, 3}};
    for (auto &gr : groups) {
        if (gr.cnt == 0) continue;
        // float4 path needs 16-byte aligned group starts
        const bool aligned = ((gr.off & 3) == 0) &&
                             (((uintptr_t)gr.p & 15) == 0) &&
                             (((uintptr_t)grad & 15) == 0) &&
                             (((uintptr_t)m & 15) == 0) &&
                             (((uintptr_t)v & 15) == 0);
        adam_group_kernel<<<grid_for(aligned ? gr.cnt / 4 + 1 : gr.cnt, th), th,
                            0, st>>>(gr.p, grad + gr.off, m + gr.off, v + gr.off,
                                     gr.cnt, k, k.lr[gr.lri], zero_grad, aligned ? 1 : 0);
        UGS_LAUNCH_CHECK("adam_group_kernel");
    }
    adam_bg_kernel<<<1, 32, 0, st>>>(bg_raw, grad + 11 * n, m + 11 * n,
                                     v + 11 * n, k, zero_grad);
    UGS_LAUNCH_CHECK("adam_bg_kernel");
    return UGS_OK;
}

extern "C" int ugs_grad_stats(const float *grad, int64_t n, uint8_t *touched,
                              float *grad_sum, int32_t *grad_cnt, void *stream) {
    if (n <= 0) return UGS_OK;
    const int th = 256;
    grad_stats_kernel<<<(unsigned)((n + th - 1) / th), th, 0, (cudaStream_t)stream>>>(
        grad, n, touched, grad_sum, grad_cnt);
    UGS_LAUNCH_CHECK("grad_stats_kernel");
    return UGS_OK;
}

extern "C" int ugs_densify_apply(const ugs_cloud *src, const float *m_src,
                                 const float *v_src, const int32_t *keep,
                                 int64_t n_keep, const int32_t *cand,
                                 const uint8_t *split, const double *z,
                                 int64_t n_new, double split_factor,
                                 float *means, float *l_raw,
                                 float *intensity_raw, float *opacity_raw,
                                 float *m_dst, float *v_dst, void *stream) {
    if (!src || n_keep < 0 || n_new < 0 || n_keep > src->n) {
        set_error("ugs_densify_apply: invalid arguments");
        return UGS_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n_dst = n_keep + n_new;
    const int th = 256;
    if (n_keep > 0) {
        densify_keep_kernel<<<(unsigned)((n_keep + th - 1) / th), th, 0, st>>>(
            *src, m_src, v_src, keep, n_keep, n_dst, means, l_raw, intensity_raw,
            opacity_raw, m_dst, v_dst);
        UGS_LAUNCH_CHECK("densify_keep_kernel");
    } else {
        UGS_CUDA(cudaMemcpyAsync(m_dst + 11 * n_dst, m_src + 11 * src->n,
                                 2 * sizeof(float), cudaMemcpyDeviceToDevice, st));
        UGS_CUDA(cudaMemcpyAsync(v_dst + 11 * n_dst, v_src + 11 * src->n,
                                 2 * sizeof(float), cudaMemcpyDeviceToDevice, st));
    }
    if (n_new > 0) {
        densify_new_kernel<<<(unsigned)((n_new + th - 1) / th), th, 0, st>>>(
            cand, split, z, n_new, n_keep, n_dst, src->beta, split_factor, means,
            l_raw, intensity_raw, opacity_raw, m_dst, v_dst);
        UGS_LAUNCH_CHECK("densify_new_kernel");
    }
    return UGS_OK;
}
