// Tile-resident forward accumulation and backward for a batch of slices.
//
// One CTA per (slice, 16x16 tile); 8 warps, each owning an 8x4 pixel block
// so a Gaussian whose window misses the warp's block is skipped with a
// warp-uniform branch.  Gaussian records of the tile's sorted list are staged
// through shared memory in batches; every pixel then walks the list in
// ascending Gaussian order (the reference's sequential order, ref
// _kernels.py:23-47), so each f32 accumulator sees the same sequence of adds.
//
// Per pair the reference evaluates w = alpha exp(-q/2), q = |L^T(p - mu)|^2
// (28 flops, float64).  Here the preprocess has conditioned the Gaussian on
// the slice plane (ugs_geometry.cuh, PlaneForm): log2 w is a 2-D quadratic
// in the pixel offset from the in-plane centre, so a pair costs 4 FADD +
// 5 FMA + one MUFU ex2, with the centre split into integer + fraction to
// avoid cancellation.
//
// Backward: each pixel computes t = dw*w and G*w (G = dpix/ssum); the
// per-Gaussian gradient needs only 7 weighted moments over the window
// (sum G w, sum t, sum t dx, sum t dy, sum t dx^2, sum t dx dy, sum t dy^2),
// reduced per warp with a transpose-reduce (9 shuffles for 8 values), then
// across warps in fixed order, and written per tile instance.  A finalize
// pass per slice sums a record's instance partials in order and applies the
// closed-form chain to d_mu, d_L and the raw parameters (float64) -- no
// atomics anywhere, so gradients are bitwise reproducible.
#include "ugs_geometry.cuh"

namespace ugs {

namespace {

constexpr int kRasterThreads = 256;
constexpr int kFwdBatch = 256;
constexpr int kBwdBatch = 128;

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct PixelCoord {
    int u, v;       // absolute pixel
    int wu0, wv0;   // warp block origin (8 x 4)
};

__device__ __forceinline__ PixelCoord pixel_of_thread(int tx, int ty) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    PixelCoord p;
    p.wu0 = tx * kTile + (warp & 1) * 8;
    p.wv0 = ty * kTile + (warp >> 1) * 4;
    p.u = p.wu0 + (lane & 7);
    p.v = p.wv0 + (lane >> 3);
    return p;
}

__device__ __forceinline__ bool warp_misses(int wu, int wv, const PixelCoord &p) {
    const int iu0 = wu & 0xffff, iu1 = wu >> 16;
    const int iv0 = wv & 0xffff, iv1 = wv >> 16;
    return iu0 > p.wu0 + 7 || iu1 < p.wu0 || iv0 > p.wv0 + 3 || iv1 < p.wv0;
}

__device__ __forceinline__ bool in_window(int wu, int wv, int u, int v) {
    const int iu0 = wu & 0xffff, iu1 = wu >> 16;
    const int iv0 = wv & 0xffff, iv1 = wv >> 16;
    return (unsigned)(u - iu0) <= (unsigned)(iu1 - iu0) &&
           (unsigned)(v - iv0) <= (unsigned)(iv1 - iv0);
}

__device__ __forceinline__ void bg_values(const double *bg_raw, float *abg,
                                          float *cbg) {
    // rasterize: alpha_bg = f32(sigmoid64(bg_opacity_raw)); num += alpha_bg *
    // f32(sigmoid64(bg_intensity_raw)); den += alpha_bg (rasterizer.py:175-177)
    *cbg = (float)sigmoid_f64(bg_raw[0]);
    *abg = (float)sigmoid_f64(bg_raw[1]);
}

__global__ void __launch_bounds__(kRasterThreads)
forward_kernel(const Rec *__restrict__ rec, const uint32_t *__restrict__ owner,
               const uint32_t *__restrict__ vals,
               const int2 *__restrict__ bin_range,
               const ugs_slice *__restrict__ slices,
               const double *__restrict__ bg_raw, float *__restrict__ num_out,
               float *__restrict__ den_out) {
    __shared__ float4 s0[kFwdBatch], s1[kFwdBatch], s2[kFwdBatch];
    __shared__ float sh_bg[2];
    const ugs_slice &sl = slices[blockIdx.y];
    const int ntile = sl.tiles_x * sl.tiles_y;
    const int t = blockIdx.x;
    if (t >= ntile) return;
    const int tx = t % sl.tiles_x, ty = t / sl.tiles_x;
    const PixelCoord pc = pixel_of_thread(tx, ty);
    const int2 rg = bin_range[sl.tile_base + t];
    if (threadIdx.x == 0) {
        float a, c;
        bg_values(bg_raw, &a, &c);
        sh_bg[0] = a;
        sh_bg[1] = c;
    }
    const float fu = (float)pc.u, fv = (float)pc.v;
    float num = 0.f, den = 0.f;
    for (int b0 = rg.x; b0 < rg.y; b0 += kFwdBatch) {
        const int nb = min(kFwdBatch, rg.y - b0);
        __syncthreads();
        if (threadIdx.x < nb) {
            const uint32_t r = __ldg(owner + __ldg(vals + b0 + threadIdx.x));
            const float4 *src = reinterpret_cast<const float4 *>(rec + r);
            s0[threadIdx.x] = __ldg(src);
            s1[threadIdx.x] = __ldg(src + 1);
            s2[threadIdx.x] = __ldg(src + 2);
        }
        __syncthreads();
        for (int j = 0; j < nb; ++j) {
            const float4 r2 = s2[j];
            const int wu = __float_as_int(r2.y), wv = __float_as_int(r2.z);
            if (warp_misses(wu, wv, pc)) continue;
            const float4 r0 = s0[j], r1 = s1[j];
            const float dx = (fu - r0.x) - r0.z;
            const float dy = (fv - r0.y) - r0.w;
            const float e = fmaf(fmaf(r1.x, dx, r1.y * dy), dx,
                                 fmaf(r1.z * dy, dy, r1.w));
            float w = ex2_approx(e);
            w = in_window(wu, wv, pc.u, pc.v) ? w : 0.f;
            num = fmaf(w, r2.x, num);
            den += w;
        }
    }
    __syncthreads();
    if (pc.u < sl.width && pc.v < sl.height) {
        const float abg = sh_bg[0], cbg = sh_bg[1];
        const int64_t p = sl.pix_base + (int64_t)pc.v * sl.width + pc.u;
        num_out[p] = num + abg * cbg;
        den_out[p] = den + abg;
    }
}

// Transpose-reduce of 8 per-lane values across the warp.  On return lanes
// with (lane & 3) == 0 hold the warp total of value (lane >> 2).
__device__ __forceinline__ float warp_reduce8(float a[8]) {
    const int lane = threadIdx.x & 31;
    float b[4], c[2];
    const bool h16 = lane & 16, h8 = lane & 8, h4 = lane & 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float send = h16 ? a[k] : a[k + 4];
        const float keep = h16 ? a[k + 4] : a[k];
        b[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const float send = h8 ? b[k] : b[k + 2];
        const float keep = h8 ? b[k + 2] : b[k];
        c[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    float d;
    {
        const float send = h4 ? c[0] : c[1];
        const float keep = h4 ? c[1] : c[0];
        d = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    d += __shfl_xor_sync(0xffffffffu, d, 2);
    d += __shfl_xor_sync(0xffffffffu, d, 1);
    return d;
}

__global__ void __launch_bounds__(kRasterThreads)
backward_kernel(const Rec *__restrict__ rec, const uint32_t *__restrict__ owner,
                const uint32_t *__restrict__ vals,
                const int2 *__restrict__ bin_range,
                const ugs_slice *__restrict__ slices,
                const float *__restrict__ num_in, const float *__restrict__ den_in,
                const float *__restrict__ dpix, const double *__restrict__ bg_raw,
                float *__restrict__ partial, float2 *__restrict__ bin_bg) {
    constexpr int kWarps = kRasterThreads / 32;
    __shared__ float4 s0[kBwdBatch], s1[kBwdBatch], s2[kBwdBatch];
    __shared__ uint32_t s_inst[kBwdBatch];
    __shared__ float part[kWarps][kBwdBatch][8];
    __shared__ float2 s_bg[kWarps];
    const ugs_slice &sl = slices[blockIdx.y];
    const int ntile = sl.tiles_x * sl.tiles_y;
    const int t = blockIdx.x;
    if (t >= ntile) return;
    const int tx = t % sl.tiles_x, ty = t / sl.tiles_x;
    const PixelCoord pc = pixel_of_thread(tx, ty);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int2 rg = bin_range[sl.tile_base + t];
    // per-pixel upstream terms: G = dpix/ssum, Gc = G * chat, chat = num/ssum
    float G = 0.f, Gc = 0.f, Gb = 0.f;
    if (pc.u < sl.width && pc.v < sl.height) {
        const int64_t p = sl.pix_base + (int64_t)pc.v * sl.width + pc.u;
        const float ssum = den_in[p];
        const float chat = __fdiv_rn(num_in[p], ssum);
        G = __fdiv_rn(dpix[p], ssum);
        Gc = G * chat;
        // background opacity term dpix*(c_bg - chat)/ssum, formed per pixel
        // as the reference does (gradients.py:110) to avoid cancellation
        Gb = G * ((float)sigmoid_f64(bg_raw[0]) - chat);
    }
    {   // background partials of this tile (sum G, sum G*(c_bg-chat)), fixed order
        float a = G, c = Gb;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (lane == 0) s_bg[warp] = make_float2(a, c);
    }
    const float fu = (float)pc.u, fv = (float)pc.v;
    for (int b0 = rg.x; b0 < rg.y; b0 += kBwdBatch) {
        const int nb = min(kBwdBatch, rg.y - b0);
        __syncthreads();
        if (threadIdx.x < nb) {
            const uint32_t inst = __ldg(vals + b0 + threadIdx.x);
            const uint32_t r = __ldg(owner + inst);
            const float4 *src = reinterpret_cast<const float4 *>(rec + r);
            s0[threadIdx.x] = __ldg(src);
            s1[threadIdx.x] = __ldg(src + 1);
            s2[threadIdx.x] = __ldg(src + 2);
            s_inst[threadIdx.x] = inst;
        }
        __syncthreads();
        for (int j = 0; j < nb; ++j) {
            const float4 r2 = s2[j];
            const int wu = __float_as_int(r2.y), wv = __float_as_int(r2.z);
            if (warp_misses(wu, wv, pc)) {
                if (lane < 8) part[warp][j][lane] = 0.f;
                continue;
            }
            const float4 r0 = s0[j], r1 = s1[j];
            const float dx = (fu - r0.x) - r0.z;
            const float dy = (fv - r0.y) - r0.w;
            const float e = fmaf(fmaf(r1.x, dx, r1.y * dy), dx,
                                 fmaf(r1.z * dy, dy, r1.w));
            float w = ex2_approx(e);
            w = in_window(wu, wv, pc.u, pc.v) ? w : 0.f;
            const float tq = fmaf(G, r2.x, -Gc) * w;   // dw * w
            const float tx_ = tq * dx, ty_ = tq * dy;
            float a[8];
            a[0] = G * w;
            a[1] = tq;
            a[2] = tx_;
            a[3] = ty_;
            a[4] = tx_ * dx;
            a[5] = tx_ * dy;
            a[6] = ty_ * dy;
            a[7] = 0.f;
            const float red = warp_reduce8(a);
            if ((lane & 3) == 0) part[warp][j][lane >> 2] = red;
        }
        __syncthreads();
        // fixed-order cross-warp sum, one (record, moment) per thread
        for (int idx = threadIdx.x; idx < nb * 8; idx += kRasterThreads) {
            const int j = idx >> 3, k = idx & 7;
            float sacc = 0.f;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) sacc += part[w][j][k];
            partial[(size_t)s_inst[j] * 8 + k] = sacc;
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

// Per slice (launched in slice order): sum a record's instance partials in
// order and chain to the raw parameters (ref gradients.py:84-103, moments ->
// d_mu = Lambda V, d_L = -M L; see the file comment).
__global__ void finalize_kernel(const Rec *__restrict__ rec,
                                const int32_t *__restrict__ rec_gid,
                                const int32_t *__restrict__ rec_inst,
                                const float *__restrict__ partial,
                                int64_t r_begin, int64_t r_end,
                                const ugs_slice *__restrict__ slice,
                                const float *__restrict__ means,
                                const float *__restrict__ l_raw, float beta,
                                int64_t n, float *__restrict__ grad,
                                uint8_t *__restrict__ touched, float scale) {
    const int64_t r = r_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= r_end) return;
    const ugs_slice &sl = *slice;
    double S[7] = {0, 0, 0, 0, 0, 0, 0};
    const int i0 = rec_inst[r], i1 = rec_inst[r + 1];
    for (int i = i0; i < i1; ++i) {
        const float4 pa = *reinterpret_cast<const float4 *>(partial + (size_t)i * 8);
        const float4 pb = *reinterpret_cast<const float4 *>(partial + (size_t)i * 8 + 4);
        S[0] += pa.x; S[1] += pa.y; S[2] += pa.z; S[3] += pa.w;
        S[4] += pb.x; S[5] += pb.y; S[6] += pb.z;
    }
    const int64_t g = rec_gid[r];
    const Rec R = rec[r];
    const Factor f = make_factor(l_raw, g, beta);
    const double mu[3] = {means[3 * g], means[3 * g + 1], means[3 * g + 2]};
    const double du[3] = {sl.du[0], sl.du[1], sl.du[2]};
    const double dv[3] = {sl.dv[0], sl.dv[1], sl.dv[2]};
    const double cu = (double)R.r0.x + (double)R.r0.z;
    const double cv = (double)R.r0.y + (double)R.r0.w;
    double es[3];
    for (int k = 0; k < 3; ++k)
        es[k] = ((double)sl.origin[k] - mu[k]) + cu * du[k] + cv * dv[k];
    const double Tc = S[0], S0 = S[1], Sx = S[2], Sy = S[3], Sxx = S[4],
                 Sxy = S[5], Syy = S[6];
    // V = sum t e ;  Mm = sum t e e^T     (dq = -t/2)
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
    const double L[3][3] = {{f.L00, 0.0, 0.0}, {f.L10, f.L11, 0.0}, {f.L20, f.L21, f.L22}};
    // Lambda = L L^T ; d_mu = Lambda V
    double LtV[3];
    for (int k = 0; k < 3; ++k) LtV[k] = L[0][k] * V[0] + L[1][k] * V[1] + L[2][k] * V[2];
    double dmu[3];
    for (int i = 0; i < 3; ++i) dmu[i] = L[i][0] * LtV[0] + L[i][1] * LtV[1] + L[i][2] * LtV[2];
    // d_L = -(Mm L), lower entries
    auto dL = [&](int i, int j) {
        return -(Mm[i][0] * L[0][j] + Mm[i][1] * L[1][j] + Mm[i][2] * L[2][j]);
    };
    const float *lr = l_raw + 6 * g;
    const double c = R.r2.x, a = R.r2.w;
    double gl[6];
    gl[0] = dL(0, 0) * 2.0 * (double)lr[0];
    gl[1] = dL(1, 1) * 2.0 * (double)lr[1];
    gl[2] = dL(2, 2) * 2.0 * (double)lr[2];
    gl[3] = dL(1, 0);
    gl[4] = dL(2, 0);
    gl[5] = dL(2, 1);
    const double gc = Tc * c * (1.0 - c);
    const double ga = S0 * (1.0 - a);   // (S0 / a) * a (1 - a)
    const double sc = (double)scale;
    float *gm = grad + 3 * g;
    for (int k = 0; k < 3; ++k) gm[k] += (float)(sc * dmu[k]);
    float *gL = grad + 3 * n + 6 * g;
    for (int k = 0; k < 6; ++k) gL[k] += (float)(sc * gl[k]);
    grad[9 * n + g] += (float)(sc * gc);
    grad[10 * n + g] += (float)(sc * ga);
    if (touched) touched[g] = 1;
}

// Background gradients of one slice: sum over its tiles in order.
__global__ void bg_finalize_kernel(const float2 *__restrict__ bin_bg, int tile_base,
                                   int ntile, const double *__restrict__ bg_raw,
                                   float *__restrict__ grad_bg, float scale) {
    __shared__ double sa[256], sc_[256];
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
    if (threadIdx.x == 0) {
        const double cbg = sigmoid_f64(bg_raw[0]), abg = sigmoid_f64(bg_raw[1]);
        const double sumG = sa[0], sumGb = sc_[0];
        const double d_cbg = (double)(float)abg * sumG;   // sum dpix*f32(a_bg)/ssum
        const double d_abg = sumGb;                       // sum dpix*(c_bg-chat)/ssum
        grad_bg[0] += (float)((double)scale * d_cbg * cbg * (1.0 - cbg));
        grad_bg[1] += (float)((double)scale * d_abg * abg * (1.0 - abg));
    }
}

}  // namespace

int launch_forward(const ugs_plan &p, const ugs_cloud &c, const uint32_t *vals,
                   float *num, float *den, cudaStream_t st) {
    if (p.S == 0) return UGS_OK;
    dim3 grid(p.max_tiles, p.S);
    stage_begin(const_cast<ugs_plan *>(&p), kStageForward, st);
    forward_kernel<<<grid, kRasterThreads, 0, st>>>(
        p.b.rec, p.b.owner, vals, p.b.bin_range, p.b.slices, c.bg_raw, num, den);
    UGS_LAUNCH_CHECK("forward_kernel");
    stage_end(const_cast<ugs_plan *>(&p), kStageForward, st);
    return UGS_OK;
}

int launch_backward(const ugs_plan &p, const ugs_cloud &c, const uint32_t *vals,
                    const float *num, const float *den, const float *dpix,
                    float *grad, uint8_t *touched, float scale,
                    cudaStream_t st) {
    if (p.S == 0) return UGS_OK;
    dim3 grid(p.max_tiles, p.S);
    ugs_plan *pm = const_cast<ugs_plan *>(&p);
    stage_begin(pm, kStageBackward, st);
    backward_kernel<<<grid, kRasterThreads, 0, st>>>(
        p.b.rec, p.b.owner, vals, p.b.bin_range, p.b.slices, num, den, dpix,
        c.bg_raw, p.b.partial, p.b.bin_bg);
    UGS_LAUNCH_CHECK("backward_kernel");
    stage_end(pm, kStageBackward, st);
    stage_begin(pm, kStageFinalize, st);
    for (int s = 0; s < p.S; ++s) {
        const int64_t r0 = p.h_slice_base[2 * s];
        const int64_t m = p.h_m[s];
        if (m > 0) {
            const int th = 128;
            finalize_kernel<<<(unsigned)((m + th - 1) / th), th, 0, st>>>(
                p.b.rec, p.b.rec_gid, p.b.rec_inst, p.b.partial, r0, r0 + m,
                p.b.slices + s, c.means, c.l_raw, (float)c.beta, c.n, grad, touched,
                scale);
            UGS_LAUNCH_CHECK("finalize_kernel");
        }
    }
    // background grads need the per-slice tile counts: read from the host copy
    for (int s = 0; s < p.S; ++s) {
        bg_finalize_kernel<<<1, 256, 0, st>>>(p.b.bin_bg, p.h_tile_base[s],
                                              p.h_ntile[s], c.bg_raw,
                                              grad + 11 * c.n, scale);
        UGS_LAUNCH_CHECK("bg_finalize_kernel");
    }
    stage_end(pm, kStageFinalize, st);
    return UGS_OK;
}

}  // namespace ugs
