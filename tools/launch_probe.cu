// Kernel-boundary cost of the discriminator's launch shape, isolated: a
// near-empty kernel launched 200 times back to back in a CUDA graph, per
// launch time for (cluster 2 / none) x (227 KB / 0 dynamic smem) x (480 / 128
// threads), with and without a 1-CTA kernel between launches (the finalize
// step), and with programmatic dependent launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/lp tools/launch_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void body(int spin) {
    extern __shared__ unsigned char sm[];
    if (spin && threadIdx.x == 0) {
        long long t0 = clock64();
        while (clock64() - t0 < spin) {
        }
        if (blockDim.x == 0) sm[0] = 1;   // never: keeps the smem symbol
    }
}
__global__ void small() {}
__global__ void body_pdl(int spin) {
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ unsigned char sm[];
    if (spin && threadIdx.x == 0) {
        long long t0 = clock64();
        while (clock64() - t0 < spin) {
        }
        if (blockDim.x == 0) sm[0] = 1;   // never: keeps the smem symbol
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

float run(int cluster, int smem, int threads, bool with_small, bool pdl, int spin) {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaFuncSetAttribute(body, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(body_pdl, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 200; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        int na = 0;
        if (cluster > 1) {
            at[na].id = cudaLaunchAttributeClusterDimension;
            at[na].val.clusterDim.x = cluster;
            at[na].val.clusterDim.y = 1;
            at[na].val.clusterDim.z = 1;
            ++na;
        }
        if (pdl) {
            at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[na].val.programmaticStreamSerializationAllowed = 1;
            ++na;
        }
        cfg.attrs = at;
        cfg.numAttrs = na;
        if (pdl) cudaLaunchKernelEx(&cfg, body_pdl, spin);
        else cudaLaunchKernelEx(&cfg, body, spin);
        if (with_small) small<<<1, 256, 0, s>>>();
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ge;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
        printf("instantiate failed: %s\n", cudaGetErrorString(cudaGetLastError()));
        return -1;
    }
    cudaGraphLaunch(ge, s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(s);
    return ms * 1000.0f / 200;
}

int main() {
    const int spin = 20000;   // ~10 us of work per CTA
    for (int spin_on = 0; spin_on < 2; ++spin_on)
        for (int cl : {1, 2})
            for (int sm : {0, 227 * 1024})
                for (int th : {128, 480})
                    for (int ws : {0, 1}) {
                        printf("spin %5d cluster %d smem %6d threads %3d +small %d: %6.2f us/launch",
                               spin_on * spin, cl, sm, th, ws,
                               run(cl, sm, th, ws, false, spin_on * spin));
                        if (!ws) printf("   pdl: %6.2f", run(cl, sm, th, ws, true, spin_on * spin));
                        printf("\n");
                    }
    return 0;
}
