// Diagnostics: FP32 FMA peak probe (the roofline denominator for the
// FP32-bound raster kernels is measured in the same run, on the same clocks).
#include "ugs_internal.cuh"

namespace ugs {
namespace {
__global__ void __launch_bounds__(256) fp32_peak_kernel(float *out, int iters) {
    float a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-7f + k;
    const float m = 0.9999999f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], m, c);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.678f) out[0] = s;   // keep the chains live
}
}  // namespace
}  // namespace ugs

extern "C" int ugs_fp32_peak_probe(float *out, int blocks, int iters, void *stream) {
    if (blocks < 1 || iters < 1) {
        ugs::set_error("ugs_fp32_peak_probe: blocks, iters must be >= 1");
        return UGS_ERR_INVALID;
    }
    ugs::fp32_peak_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, iters);
    UGS_LAUNCH_CHECK("fp32_peak_kernel");
    return UGS_OK;
}
