// Probe: fp64 FMA throughput and latency on this GPU (B200 / sm_100a), and the
// int64 multiply rate, for the K3/K4 roofline notes. Throughput: every thread
// runs 8 independent DFMA chains; latency: one chain per warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rate_probe tools/fp64_rate_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void dfma_tput(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.0) out[0] = s;
}

__global__ void dfma_lat(double* out, int iters, double a, double b) {
    double x = threadIdx.x * 1e-3;
    for (int i = 0; i < iters; ++i) x = fma(x, a, b);
    if (x == 12345.0) out[0] = x;
}

__global__ void ffma_tput(float* out, int iters, float a, float b) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
    }
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.0f) out[0] = s;
}

__global__ void imul64_tput(uint64_t* out, int iters) {
    uint64_t x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = 6364136223846793005ULL * (x[k] ^ (x[k] >> 62)) + i;
    }
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s ^= x[k];
    if (s == 12345) out[0] = s;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* d;
    cudaMalloc(&d, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    const int iters = 4096;
    auto time = [&](auto launch) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        return ms;
    };
    const int blocks = sms * 8, threads = 256;
    ms = time([&] { dfma_tput<<<blocks, threads>>>(d, iters, 0.999, 1.0); });
    const double nf = 1.0 * blocks * threads * iters * 8;
    printf("DFMA throughput: %.2f T/s  (%.1f per SM per clock at %d MHz)\n", nf / ms / 1e9,
           nf / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    ms = time([&] { ffma_tput<<<blocks, threads>>>(reinterpret_cast<float*>(d), iters, 0.999f, 1.0f); });
    printf("FFMA throughput: %.2f T/s  (%.1f per SM per clock)\n", nf / ms / 1e9,
           nf / (ms * 1e-3) / sms / (clk * 1e3));
    ms = time([&] { imul64_tput<<<blocks, threads>>>(reinterpret_cast<uint64_t*>(d), iters); });
    printf("mt seeding step (xor-shift + 64-bit mul + add): %.2f G/s (%.2f per SM per clock)\n",
           nf / ms / 1e6, nf / (ms * 1e-3) / sms / (clk * 1e3));
    ms = time([&] { dfma_lat<<<1, 32>>>(d, iters * 16, 0.999, 1.0); });
    printf("DFMA dependent latency: %.1f cycles (one warp)\n", ms * 1e-3 * clk * 1e3 / (iters * 16));
    return 0;
}
