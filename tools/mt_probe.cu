// Probe: layouts of the single std::mt19937_64 stream for K8a (arrivals.cu).
// Generates N raw (untempered) words x_312.. with (A) the 160-thread kernel
// (thread = column, shared ring, one barrier per 2 steps) and (B) one warp,
// lane l owning columns 5l..5l+4 (neighbour words by shuffle, no barrier),
// checks both against a host std::mt19937_64 and times them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mt_probe tools/mt_probe.cu
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mt_mix(uint64_t xk, uint64_t xk1) {
    const uint64_t y = (xk & 0xFFFFFFFF80000000ULL) | (xk1 & 0x7FFFFFFFULL);
    return (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
}

__global__ void __launch_bounds__(160) mt_a(uint64_t seed, int64_t n, uint64_t* raw) {
    __shared__ uint64_t ring[4][156];
    const int c = threadIdx.x;
    if (c == 0) {
        uint64_t x = seed;
        ring[0][0] = x;
        for (int i = 1; i < 312; ++i) {
            x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
            ring[i / 156][i % 156] = x;
        }
    }
    __syncthreads();
    const bool active = c < 156;
    uint64_t x2 = active ? ring[0][c] : 0, x1 = active ? ring[1][c] : 0;
    const int64_t steps = (n + 155) / 156;
    for (int64_t s = 0; s < steps; s += 2) {
        const int a = static_cast<int>(s & 3), b = (a + 1) & 3, w0 = (a + 2) & 3, w1 = (a + 3) & 3;
        if (active) {
            uint64_t nb_a, nb_b;
            if (c < 155) { nb_a = ring[a][c + 1]; nb_b = ring[b][c + 1]; }
            else { nb_a = ring[b][0]; nb_b = ring[b][0] ^ mt_mix(ring[a][0], ring[a][1]); }
            const uint64_t y0 = x1 ^ mt_mix(x2, nb_a);
            const uint64_t y1 = y0 ^ mt_mix(x1, nb_b);
            ring[w0][c] = y0;
            ring[w1][c] = y1;
            const int64_t k0 = s * 156 + c;
            if (k0 < n) raw[k0] = y0;
            if (k0 + 156 < n) raw[k0 + 156] = y1;
            x2 = y0;
            x1 = y1;
        }
        __syncthreads();
    }
}

// (B) one warp; lane l owns columns 5l+j (j < 5, column < 156).
template <int kStage>
__global__ void __launch_bounds__(32) mt_b(uint64_t seed, int64_t n, uint64_t* raw) {
    __shared__ uint64_t init[312];
    __shared__ __align__(16) uint64_t stage[kStage > 0 ? kStage : 1][156];
    const int l = threadIdx.x;
    if (l == 0) {
        uint64_t x = seed;
        init[0] = x;
        for (int i = 1; i < 312; ++i) {
            x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
            init[i] = x;
        }
    }
    __syncwarp();
    uint64_t x2[5], x1[5];   // column 5l+j at steps s, s+1
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const int c = 5 * l + j;
        x2[j] = c < 156 ? init[c] : 0;
        x1[j] = c < 156 ? init[156 + c] : 0;
    }
    const int64_t steps = (n + 155) / 156;
    for (int64_t s = 0; s < steps; ++s) {
        // x_{m-311} for column c = 5l+j is column c+1 at step s, except c = 155
        // (lane 31, j = 0): column 0 at step s+1
        const uint64_t right = __shfl_down_sync(0xffffffffu, x2[0], 1);   // column 5l+5 at s
        const uint64_t col0_next = __shfl_sync(0xffffffffu, x1[0], 0);     // column 0 at s+1
        uint64_t y[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            uint64_t nb = j < 4 ? x2[j + 1] : right;
            if (l == 31 && j == 0) nb = col0_next;
            y[j] = x1[j] ^ mt_mix(x2[j], nb);
        }
        const int64_t base = (s) * 156;   // raw index of step s+2 column 0 (raw[k] = x_{312+k})
        if (kStage == 0) {
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const int c = 5 * l + j;
                if (c < 156 && base + c < n) raw[base + c] = y[j];
            }
        } else {
            const int slot = static_cast<int>(s % kStage);
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const int c = 5 * l + j;
                if (c < 156) stage[slot][c] = y[j];
            }
            if (slot == kStage - 1 || s + 1 == steps) {
                __syncwarp();
                const int64_t first = (s - slot) * 156;
                const int cnt = (slot + 1) * 156;
                const uint64_t* src = &stage[0][0];
                for (int k = l; k < cnt; k += 32)
                    if (first + k < n) raw[first + k] = src[k];
                __syncwarp();
            }
        }
#pragma unroll
        for (int j = 0; j < 5; ++j) { x2[j] = x1[j]; x1[j] = y[j]; }
    }
}

// (C) 160 threads, FOUR steps per barrier: thread t computes column t of
// steps s+2..s+5 from the last two steps (A = step s, B = step s+1, shared),
// recomputing the few neighbour words (column t+1 of steps s+2/s+3, column 0 of
// the next step for t >= 154) it needs instead of waiting for their owners.
template <int kStore>
__global__ void __launch_bounds__(160) mt_c(uint64_t seed, int64_t n, uint64_t* raw) {
    __shared__ uint64_t buf[2][2][156];   // [set][A/B][column]
    __shared__ __align__(16) uint64_t stage[2][624];
    const int t = threadIdx.x;
    if (t == 0) {
        uint64_t x = seed;
        buf[0][0][0] = x;
        for (int i = 1; i < 312; ++i) {
            x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
            buf[0][i / 156][i % 156] = x;
        }
    }
    __syncthreads();
    const int64_t steps = (n + 155) / 156;
    int set = 0;
    for (int64_t s = 0; s < steps; s += 4) {
        const uint64_t* A = buf[set][0];
        const uint64_t* B = buf[set][1];
        if (t < 156) {
            auto w2 = [&](int c) { return B[c] ^ mt_mix(A[c], c < 155 ? A[c + 1] : B[0]); };
            const uint64_t w2_0 = (t >= 154) ? w2(0) : 0;
            auto w3 = [&](int c, uint64_t w2c) {
                return w2c ^ mt_mix(B[c], c < 155 ? B[c + 1] : w2_0);
            };
            const uint64_t W2 = w2(t);
            const uint64_t W3 = w3(t, W2);
            uint64_t n2, n3;   // column t+1 (or the next step's column 0) of steps s+2, s+3
            if (t < 155) {
                n2 = w2(t + 1);
                n3 = w3(t + 1, n2);
            } else {
                n2 = w3(0, w2_0);                                  // W3(0)
                const uint64_t w2_1 = w2(1);
                n3 = n2 ^ mt_mix(w2_0, w2_1);                      // W4(0)
            }
            const uint64_t W4 = W3 ^ mt_mix(W2, n2);
            const uint64_t W5 = W4 ^ mt_mix(W3, n3);
            const int64_t k0 = s * 156 + t;
            if (kStore == 0) {
                if (k0 < n) raw[k0] = W2;
                if (k0 + 156 < n) raw[k0 + 156] = W3;
                if (k0 + 312 < n) raw[k0 + 312] = W4;
                if (k0 + 468 < n) raw[k0 + 468] = W5;
            } else if (kStore == 1) {
                if ((k0 & 63) == 0 && k0 < n) raw[k0] = W2 ^ W3 ^ W4 ^ W5;
            } else {
                stage[set][t] = W2;
                stage[set][t + 156] = W3;
                stage[set][t + 312] = W4;
                stage[set][t + 468] = W5;
            }
            buf[set ^ 1][0][t] = W4;
            buf[set ^ 1][1][t] = W5;
        }
        if (kStore == 2) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncthreads();
        if (kStore == 2 && t == 0) {
            const int64_t first = s * 156;
            const int64_t cnt = n - first < 624 ? n - first : 624;
            if (cnt > 0) {
                const uint32_t src = static_cast<uint32_t>(__cvta_generic_to_shared(&stage[set][0]));
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                             :: "l"(raw + first), "r"(src), "r"(static_cast<uint32_t>(cnt * 8)) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            }
        }
        set ^= 1;
    }
    if (kStore == 2 && t == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const int64_t n = 1000000;
    const uint64_t seed = 0x1234567887654321ULL;
    std::mt19937_64 eng(seed);
    // raw words are untempered; compare tempered outputs instead via host temper
    auto temper = [](uint64_t z) {
        z ^= (z >> 29) & 0x5555555555555555ULL;
        z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
        z ^= (z << 37) & 0xFFF7EEE000000000ULL;
        z ^= z >> 43;
        return z;
    };
    std::vector<uint64_t> want(n);
    for (int64_t i = 0; i < n; ++i) want[i] = eng();
    uint64_t* d;
    cudaMalloc(&d, n * 8);
    std::vector<uint64_t> got(n);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        cudaMemset(d, 0, n * 8);
        launch();
        cudaDeviceSynchronize();
        cudaMemcpy(got.data(), d, n * 8, cudaMemcpyDeviceToHost);
        int64_t bad = 0;
        for (int64_t i = 0; i < n; ++i) bad += temper(got[i]) != want[i];
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %8.3f ms per 1M words, mismatches %lld, err %s\n", name, ms / 5, (long long)bad,
               cudaGetErrorString(cudaGetLastError()));
    };
    run("A 160 threads, ring", [&] { mt_a<<<1, 160>>>(seed, n, d); });
    run("C 160 threads, 4 steps/barrier", [&] { mt_c<0><<<1, 160>>>(seed, n, d); });
    run("C, stores off (compute only)", [&] { mt_c<1><<<1, 160>>>(seed, n, d); });
    run("C, bulk stores from smem", [&] { mt_c<2><<<1, 160>>>(seed, n, d); });
    run("B one warp, direct stores", [&] { mt_b<0><<<1, 32>>>(seed, n, d); });
    run("B one warp, staged x4", [&] { mt_b<4><<<1, 32>>>(seed, n, d); });
    run("B one warp, staged x8", [&] { mt_b<8><<<1, 32>>>(seed, n, d); });
    return 0;
}
