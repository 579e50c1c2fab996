// Adam over the parameter SoA (gradient/moments in the AoS-12 layout of
// ugs_adam.cuh), densify statistics and densify/prune row surgery.
//
// Adam is an HBM stream: per Gaussian it reads params (44 B), gradient and
// both moments (3 x 48 B) and writes params, moments (and optionally zeroes
// the gradient): ~380 B/Gaussian.  The single-GPU training step does not use
// this kernel -- there the update is fused into the gradient accumulation
// (ugs_raster.cu, update_gather_kernel) and the dense gradient never exists.
#include "ugs_adam.cuh"
#include "ugs_geometry.cuh"

namespace ugs {

namespace {

// One thread per Gaussian.
__global__ void adam_kernel(CloudMut p, float *__restrict__ grad, float *__restrict__ m,
                            float *__restrict__ v, int64_t n, AdamConst k,
                            int zero_grad, uint8_t *__restrict__ touched,
                            float *__restrict__ grad_sum, int32_t *__restrict__ grad_cnt) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    float gr[kG];
    float4 *g4 = reinterpret_cast<float4 *>(grad + kG * g);
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const float4 a = g4[q];
        gr[4 * q] = a.x; gr[4 * q + 1] = a.y; gr[4 * q + 2] = a.z; gr[4 * q + 3] = a.w;
    }
    bool t = false;
    if (touched) {
        t = touched[g] != 0;
        touched[g] = 0;
    }
    adam_gaussian(g, gr, m + kG * g, v + kG * g, p, k, t, grad_sum, grad_cnt);
    if (zero_grad)
#pragma unroll
        for (int q = 0; q < 3; ++q) g4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void adam_bg_kernel(double *bg_raw, float *g, float *m, float *v,
                               AdamConst k, int zero_grad) {
    if (threadIdx.x != 0) return;
    adam_bg(bg_raw, g, m, v, k);
    if (zero_grad) { g[0] = 0.f; g[1] = 0.f; }
}

// trainer.py:399-401: grad_sum[acc] += ||d_means||; grad_cnt[acc] += 1.
__global__ void grad_stats_kernel(const float *__restrict__ grad, int64_t n,
                                  uint8_t *__restrict__ touched,
                                  float *__restrict__ grad_sum,
                                  int32_t *__restrict__ grad_cnt) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n || !touched[g]) return;
    const float *r = grad + kG * g;
    grad_sum[g] = __fadd_rn(grad_sum[g], norm3_f32(r[0], r[1], r[2]));
    grad_cnt[g] += 1;
    touched[g] = 0;
}

// ---- densify / prune --------------------------------------------------
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
    for (int k = 0; k < 3; ++k) means[3 * j + k] = src.means[3 * i + k];
    for (int k = 0; k < 6; ++k) l_raw[6 * j + k] = src.l_raw[6 * i + k];
    c_raw[j] = src.intensity_raw[i];
    a_raw[j] = src.opacity_raw[i];
    const float4 *ms = reinterpret_cast<const float4 *>(m_src + kG * i);
    const float4 *vs = reinterpret_cast<const float4 *>(v_src + kG * i);
    float4 *md = reinterpret_cast<float4 *>(m_dst + kG * j);
    float4 *vd = reinterpret_cast<float4 *>(v_dst + kG * j);
    for (int q = 0; q < 3; ++q) {
        md[q] = ms[q];
        vd[q] = vs[q];
    }
    if (j < 2) {   // background moments follow the rows
        m_dst[kG * n_dst + j] = m_src[kG * src.n + j];
        v_dst[kG * n_dst + j] = v_src[kG * src.n + j];
    }
}

// Each candidate touches only its own parent row and its own appended row
// (model.py:147-152, trainer.py:255-272), so candidates run in parallel.
__global__ void densify_new_kernel(const int32_t *__restrict__ cand,
                                   const uint8_t *__restrict__ split,
                                   const double *__restrict__ z, int64_t n_new,
                                   int64_t n_keep, double beta, double f,
                                   float *__restrict__ means, float *__restrict__ l_raw,
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
        for (int k = 0; k < 6; ++k) nl[k] = (float)ln[k];
        for (int k = 0; k < 6; ++k) l_raw[6 * gi + k] = nl[k];
    } else {
        for (int k = 0; k < 3; ++k) nm[k] = means[3 * gi + k];
        for (int k = 0; k < 6; ++k) nl[k] = l_raw[6 * gi + k];
    }
    for (int k = 0; k < 3; ++k) means[3 * dst + k] = nm[k];
    for (int k = 0; k < 6; ++k) l_raw[6 * dst + k] = nl[k];
    c_raw[dst] = c_raw[gi];
    a_raw[dst] = a_raw[gi];
    for (int k = 0; k < kG; ++k) {
        m_dst[kG * dst + k] = 0.f;
        v_dst[kG * dst + k] = 0.f;
    }
}

}  // namespace

}  // namespace ugs

using namespace ugs;

extern "C" int ugs_adam_step(float *means, float *l_raw, float *intensity_raw,
                             float *opacity_raw, double *bg_raw, float *grad,
                             float *m, float *v, int64_t n, int64_t t,
                             const double *lr, double beta1, double beta2,
                             double eps, int zero_grad, uint8_t *touched,
                             float *grad_sum, int32_t *grad_cnt, void *stream) {
    if (n < 0 || t < 1 || !lr || !grad || !m || !v || !bg_raw) {
        set_error("ugs_adam_step: invalid arguments");
        return UGS_ERR_INVALID;
    }
    if ((touched || grad_sum || grad_cnt) && !(touched && grad_sum && grad_cnt)) {
        set_error("ugs_adam_step: touched, grad_sum and grad_cnt go together");
        return UGS_ERR_INVALID;
    }
    if ((((uintptr_t)grad | (uintptr_t)m | (uintptr_t)v) & 15) != 0) {
        set_error("ugs_adam_step: grad, m, v must be 16-byte aligned");
        return UGS_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const AdamConst k = make_adam_const(t, lr, beta1, beta2, eps);
    const CloudMut p{means, l_raw, intensity_raw, opacity_raw};
    if (n > 0) {
        const int th = 256;
        adam_kernel<<<(unsigned)((n + th - 1) / th), th, 0, st>>>(
            p, grad, m, v, n, k, zero_grad, touched, grad_sum, grad_cnt);
        UGS_LAUNCH_CHECK("adam_kernel");
    }
    adam_bg_kernel<<<1, 32, 0, st>>>(bg_raw, grad + kG * n, m + kG * n, v + kG * n, k,
                                     zero_grad);
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
    }
    if (n_keep < 2) {   // background moments (copied by the keep kernel otherwise)
        UGS_CUDA(cudaMemcpyAsync(m_dst + kG * n_dst, m_src + kG * src->n,
                                 2 * sizeof(float), cudaMemcpyDeviceToDevice, st));
        UGS_CUDA(cudaMemcpyAsync(v_dst + kG * n_dst, v_src + kG * src->n,
                                 2 * sizeof(float), cudaMemcpyDeviceToDevice, st));
    }
    if (n_new > 0) {
        densify_new_kernel<<<(unsigned)((n_new + th - 1) / th), th, 0, st>>>(
            cand, split, z, n_new, n_keep, src->beta, split_factor, means, l_raw,
            intensity_raw, opacity_raw, m_dst, v_dst);
        UGS_LAUNCH_CHECK("densify_new_kernel");
    }
    return UGS_OK;
}
