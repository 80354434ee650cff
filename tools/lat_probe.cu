// Dependent-chain latency (cycles per op) of the scalar ops on the batch kernel's critical path (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cstdint>

constexpr int N = 4096;

__global__ void probe(double* outd, unsigned long long* outu, long long* cyc, double a, unsigned long long k) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (double)((i * 7 + 1) & 1023);
    __syncthreads();
    double x = a;
    unsigned long long z = k;
    long long t0, t1;
    // DADD chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = x + 1e-300;
    t1 = clock64();
    cyc[0] = t1 - t0;
    // DMUL chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = x * 1.0000000001;
    t1 = clock64();
    cyc[1] = t1 - t0;
    // u64 multiply chain (mix64's z *= c)
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) z = z * 0xff51afd7ed558ccdull;
    t1 = clock64();
    cyc[2] = t1 - t0;
    // u64 -> f64 -> u64 round trip (uniform()'s convert + F2I)
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) z = (unsigned long long)((double)(z >> 11) * 0.5);
    t1 = clock64();
    cyc[3] = t1 - t0;
    // dependent shared-memory loads through a generic pointer
    const double* p = sm;
    int idx = (int)(k & 1023);
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) idx = (int)p[idx];
    t1 = clock64();
    cyc[4] = t1 - t0;
    // same with an explicit shared pointer
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) idx = (int)sm[idx];
    t1 = clock64();
    cyc[5] = t1 - t0;
    // DSETP + select (clamp) chain
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) x = x < 0.5 ? x + 1.0 : x - 0.25;
    t1 = clock64();
    cyc[6] = t1 - t0;
    // int -> double -> int (the FY index r = j + (int)(u * (dim - j)))
    int r = idx;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; i++) r = (int)((double)r * 0.999) + 1;
    t1 = clock64();
    cyc[7] = t1 - t0;
    outd[threadIdx.x] = x + idx + r;
    outu[threadIdx.x] = z;
}

int main() {
    double* d;
    unsigned long long* u;
    long long* c;
    cudaMalloc(&d, 8 * 32);
    cudaMalloc(&u, 8 * 32);
    cudaMallocManaged(&c, 8 * 8);
    for (int rep = 0; rep < 2; rep++) {
        probe<<<1, 32>>>(d, u, c, 1.5, 12345);
        cudaDeviceSynchronize();
    }
    const char* names[] = {"DADD", "DMUL", "u64 mul", "u64->f64->u64", "LD generic->smem", "LDS", "DSETP+sel",
                           "i->f64->i"};
    for (int i = 0; i < 8; i++) printf("%-18s %.1f cycles/op\n", names[i], (double)c[i] / N);
    return 0;
}
