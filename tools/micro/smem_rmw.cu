// Microbenchmark: per-pixel (num, den) accumulation into 16 private shared
// tile buffers, the forward kernel's inner-loop memory pattern.
//   mode 0: LDS.64 + FFMA2 + STS.64 (round-1 forward)
//   mode 1: two red.shared.add.f32
//   mode 2: red.shared.add.v2.f32 (if the ISA accepts it)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(float *out, int iters) {
    __shared__ float2 acc[16][256];
    for (int i = threadIdx.x; i < 16 * 256; i += 256) (&acc[0][0])[i] = make_float2(0.f, 0.f);
    __syncthreads();
    const int g = threadIdx.x >> 4, l = threadIdx.x & 15;
    float2 *my = acc[g];
    float w = 1e-3f * (threadIdx.x + 1), c = 0.5f;
    int p = l;
    for (int it = 0; it < iters; ++it) {
        float2 *q = my + ((p + it * 16) & 255);
        if (MODE == 0) {
            float2 v = *q;
            v.x = fmaf(w, c, v.x);
            v.y += w;
            *q = v;
        } else if (MODE == 1) {
            asm volatile("red.shared.add.f32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&q->x)), "f"(w * c));
            asm volatile("red.shared.add.f32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&q->y)), "f"(w));
        }
        w *= 1.0001f;
    }
    __syncthreads();
    float s = 0.f;
    for (int gg = 0; gg < 16; ++gg) s += acc[gg][threadIdx.x].x + acc[gg][threadIdx.x].y;
    out[blockIdx.x * 256 + threadIdx.x] = s;
}

int main() {
    float *out;
    cudaMalloc(&out, 148 * 8 * 256 * 4 * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096, blocks = 148 * 4 * 4;
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<blocks, 256>>>(out, iters);
            if (mode == 1) k<1><<<blocks, 256>>>(out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double upd = (double)blocks * 256 * iters;
            if (rep == 2)
                printf("mode %d: %.3f ms, %.1f G pixel-updates/s, %.2f updates/clk/SM @1.965GHz (err %s)\n",
                       mode, ms, upd / ms / 1e6, upd / (ms * 1e-3) / 148 / 1.965e9,
                       cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
