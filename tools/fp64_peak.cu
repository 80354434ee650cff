// fp64_peak.cu -- measured FP64 roofline denominators on this GPU (not product code).
//   DFMA: 8 independent fma chains per thread, full occupancy.
//   DMMA: mma.sync m8n8k4 f64, 4 independent accumulators per warp, full occupancy.
// Prints one JSON line: {"dfma_tflops": ..., "dmma_tflops": ...}.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-9 + k;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += x[k];
    if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(double* out, int iters, double a, double b) {
    double c[CH][2];
#pragma unroll
    for (int k = 0; k < CH; k++) c[k][0] = c[k][1] = 0.0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < CH; k++) dmma(c[k][0], c[k][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < CH; k++) s += c[k][0] + c[k][1];
    if (s == 12345.678) out[0] = s;
}

template <class F>
float time_it(F f) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        f();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 4096, threads = 256, blocks = sms * 8;
    float ms = time_it([&] { k_dfma<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); });
    const double dfma = 2.0 * 8 * iters * (double)threads * blocks / (ms * 1e-3) / 1e12;
    float ms1 = time_it([&] { k_dmma<1><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); });
    float ms4 = time_it([&] { k_dmma<4><<<blocks, threads>>>(out, iters, 1.0000001, 1e-7); });
    const double warps = (double)threads / 32 * blocks;
    const double dmma1 = 2.0 * 256 * 1 * iters * warps / (ms1 * 1e-3) / 1e12;
    const double dmma4 = 2.0 * 256 * 4 * iters * warps / (ms4 * 1e-3) / 1e12;
    // latency: one warp per SM, one chain
    float msl = time_it([&] { k_dmma<1><<<sms, 32>>>(out, iters, 1.0000001, 1e-7); });
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double lat = msl * 1e-3 * clk * 1e3 / iters;
    printf("{\"dfma_tflops\": %.2f, \"dmma_tflops_1chain\": %.2f, \"dmma_tflops_4chain\": %.2f, "
           "\"dmma_latency_cycles\": %.1f, \"sms\": %d}\n", dfma, dmma1, dmma4, lat, sms);
    // DMMA throughput vs warps per SM (one CTA of W warps per SM, 13 independent accumulators per warp)
    for (int w : {4, 8, 12, 16, 32}) {
        float m = time_it([&] { k_dmma<13><<<sms, 32 * w>>>(out, iters / 4, 1.0000001, 1e-7); });
        printf("{\"warps_per_sm\": %d, \"chains\": 13, \"dmma_tflops\": %.2f}\n", w,
               2.0 * 256 * 13 * (iters / 4) * (double)w * sms / (m * 1e-3) / 1e12);
    }
    return 0;
}
