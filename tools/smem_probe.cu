// Microbenchmark: shared-memory port sharing between the tensor core's operand
// reads (tcgen05.mma, SS mode, M128 N256 K16, A SW128 + B SW64 as in
// disc_kernel), bulk-TMA writes of 16 KB stages from L2, and st.shared.v4 from
// warps -- all on every SM for a fixed window of ~400K cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2411_15381_b200/csrc tools/smem_probe.cu -o /tmp/smem_probe && /tmp/smem_probe
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace sm100;

constexpr long long kWindow = 400000;   // cycles

__device__ __forceinline__ uint64_t desc_k_sw64(uint32_t smem_addr) {
    const uint64_t lo = ((smem_addr >> 4) & 0x3FFFu) | (1u << 16);
    const uint64_t hi = (512u >> 4) | (1u << 14) | (4u << 29);
    return lo | (hi << 32);
}

struct Res {
    long long mma, tma_bytes, sts_bytes, cycles;
};

// smem: A 16 KB @0 | B 32 KB @16K | TMA ring 8 x 16 KB @48K | st.shared area 32 KB @176K
__global__ void __launch_bounds__(256, 1) probe(int do_mma, int ring, int sts_warps,
                                                const uint8_t* blob, Res* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t full[8], mma_bar, never;
    __shared__ uint32_t tmem_base;
    __shared__ unsigned long long s_tma, s_sts, s_mma;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sbase = smem_u32(smem);
    for (int i = threadIdx.x; i < (48 << 10) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < 8; ++s) mbar_init(&full[s], 1);
        mbar_init(&mma_bar, 1);
        mbar_init(&never, 1);
        s_tma = s_sts = s_mma = 0;
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<512>(&tmem_base);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    const long long t0 = clock64();
    if (warp == 0 && lane == 0 && do_mma) {
        const uint64_t ad = desc_k_sw128(sbase);
        const uint32_t idesc = idesc_bf16_f32(128, 256);
        long long n = 0;
        uint32_t ph = 0;
        while (clock64() - t0 < kWindow) {
            for (int it = 0; it < 16; ++it)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint64_t bd = desc_k_sw64(sbase + 16384 + (k >> 1) * 16384);
                    umma_bf16(tmem, ad + 2 * k, bd + 2 * (k & 1), idesc, 1u);
                }
            n += 64;
            umma_commit(&mma_bar);      // keep the queue bounded: wait every 64 MMAs
            mbar_wait(&mma_bar, ph);
            ph ^= 1;
        }
        s_mma = n;
        mbar_arrive(&never);
    } else if (warp == 1 && lane == 0 && ring > 0) {
        const uint64_t policy = policy_evict_last();
        long long bytes = 0;
        int s = 0, t = 0;
        uint32_t ph = 0;
        for (int i = 0; i < ring; ++i, ++t) {
            mbar_arrive_expect_tx(&full[i], 16384);
            bulk_g2s_hint(smem + (48 << 10) + i * 16384, blob + size_t(t % 88) * 16384, 16384,
                          &full[i], policy);
        }
        while (clock64() - t0 < kWindow) {
            mbar_wait(&full[s], ph);
            bytes += 16384;
            mbar_arrive_expect_tx(&full[s], 16384);
            bulk_g2s_hint(smem + (48 << 10) + s * 16384, blob + size_t(t % 88) * 16384, 16384,
                          &full[s], policy);
            ++t;
            if (++s == ring) { s = 0; ph ^= 1; }
        }
        for (int i = 0; i < ring; ++i) {   // drain
            mbar_wait(&full[s], ph);
            if (++s == ring) { s = 0; ph ^= 1; }
        }
        s_tma = bytes;
    } else if (warp >= 2 && warp < 2 + (sts_warps & 15)) {
        const uint32_t base = sbase + (176 << 10) + (threadIdx.x - 64) * 16;
        long long bytes = 0;
        const int kind = sts_warps >> 4;   // 0 st.shared, 1 cp.async 16 B from L2, 2 ldg+sts, 3 HBM stream (ld.nc)
        const int tid = threadIdx.x - 64;
        int t = 0;
        while (clock64() - t0 < kWindow) {
            if (kind == 0) {
#pragma unroll
                for (int r = 0; r < 16; ++r) st_shared_v4(base + (r & 3) * 3072 * 2, r, r, r, r);
            } else if (kind == 1) {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const uint8_t* src = blob + (size_t(t % 88) * 16384 + ((r * 192 + tid) * 16) % 16384);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                     base + (r & 3) * 3072 * 2),
                                 "l"(src)
                                 : "memory");
                }
                asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 2;" ::: "memory");
                ++t;
            } else if (kind == 4) {
                // spin on an mbarrier phase that completes only at the end of the window
                mbar_wait(&never, 0);
                break;
            } else if (kind == 3) {
                // stream a 4 GB buffer from HBM: 16 x 16 B per thread, like the A-builder
                const uint8_t* big = blob + (size_t(88) << 14);
                uint4 v[16];
                const size_t base_off = ((size_t(blockIdx.x) * 1000003 + size_t(t) * 6144 + tid * 16) % (size_t(3) << 30)) & ~size_t(15);
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = ld_global_nc_v4(big + (base_off + size_t(r) * 3072 * 16) % (size_t(3) << 30));
                uint32_t acc = 0;
#pragma unroll
                for (int r = 0; r < 16; ++r) acc ^= v[r].x ^ v[r].w;
                if (acc == 0x12345678u) st_shared_v4(base, acc, acc, acc, acc);
                ++t;
            } else {
                uint4 v[16];
#pragma unroll
                for (int r = 0; r < 16; ++r)
                    v[r] = ld_global_nc_v4(blob + (size_t(t % 88) * 16384 + ((r * 192 + tid) * 16) % 16384));
#pragma unroll
                for (int r = 0; r < 16; ++r)
                    st_shared_v4(base + (r & 3) * 3072 * 2, v[r].x, v[r].y, v[r].z, v[r].w);
                ++t;
            }
            bytes += 256;
        }
        if (kind == 1) asm volatile("cp.async.wait_all;" ::: "memory");
        atomicAdd(&s_sts, static_cast<unsigned long long>(bytes));
    }
    const long long t1 = clock64();
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        out[blockIdx.x].mma = s_mma;
        out[blockIdx.x].tma_bytes = s_tma;
        out[blockIdx.x].sts_bytes = s_sts;
        out[blockIdx.x].cycles = t1 - t0;
    }
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

int main() {
    const int smem = 208 << 10;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    uint8_t* blob = nullptr;
    cudaMalloc(&blob, 88 * 16384 + (size_t(3) << 30) + (1 << 20));
    cudaMemset(blob, 0, 88 * 16384 + (size_t(3) << 30));
    Res* d = nullptr;
    cudaMalloc(&d, sizeof(Res) * 148);
    struct Cfg { int mma, ring, sts; } cfgs[] = {
        {1, 4, 0}, {1, 4, 64 + 2}, {1, 4, 64 + 4}, {1, 4, 64 + 6}};
    for (const Cfg& c : cfgs) {
        probe<<<148, 256, smem>>>(c.mma, c.ring, c.sts, blob, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
        }
        Res h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double mma = 0, tma = 0, sts = 0;
        for (int i = 0; i < 148; ++i) {
            mma += double(h[i].mma) / h[i].cycles;
            tma += double(h[i].tma_bytes) / h[i].cycles;
            sts += double(h[i].sts_bytes) / h[i].cycles;
        }
        mma /= 148;
        tma /= 148;
        sts /= 148;
        printf("mma=%d ring=%d lsu=%d (kind %d) | cycles/MMA %6.1f (operand B/clk %5.1f) | TMA "
               "B/clk %5.1f | st.shared B/clk %5.1f\n",
               c.mma, c.ring, c.sts & 15, c.sts >> 4, mma > 0 ? 1.0 / mma : 0.0, mma * 12288, tma, sts);
    }
    return 0;
}
