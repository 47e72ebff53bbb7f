// Microbenchmark: K-SET round hand-off latency on B200 (per round, us), for the
// protocols the executor can use between rounds k-1 and k:
//   0 sc      : __syncthreads; tid0 fence.sc.gpu (__threadfence) + atomicAdd; tid0 polls
//               ld.acquire (+__nanosleep 200 ns on CTAs != 0); __syncthreads   (round-1 code)
//   1 rel     : __syncthreads; tid0 red.release.gpu; tid0 polls ld.acquire, no sleep; __syncthreads
//   2 warp    : every warp: __syncwarp; lane0 red.release.gpu; lane0 of every warp polls; __syncwarp
//   3 cluster : barrier.cluster.arrive.release / wait.acquire (g == cluster size)
// "data" variants add one dependent access per round: thread t of CTA b reads the word
// CTA (b+1)%g wrote in round k-1 (an L2 hit) and writes its own for round k.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/handoff tools/handoff.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
    uint32_t v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void red_rel(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MODE, bool DATA>
__global__ void handoff(uint32_t* done, int rounds, uint64_t* trace, uint32_t* data, int nwarps_sig) {
    const int b = blockIdx.x, g = gridDim.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int W = blockDim.x / 32;
    uint32_t acc = 0;
    for (int k = 0; k < rounds; ++k) {
        if (k > 0) {
            if (MODE == 0) {
                if (tid == 0) { uint32_t s = 0; while (ld_acq(&done[k - 1]) < (uint32_t)g) if (++s > 16) __nanosleep(b == 0 ? 20 : 200); }
                __syncthreads();
            } else if (MODE == 1) {
                if (tid == 0) while (ld_acq(&done[k - 1]) < (uint32_t)g) { }
                __syncthreads();
            } else if (MODE == 2) {
                if (lane == 0) while (ld_acq(&done[k - 1]) < (uint32_t)(g * W)) { }
                __syncwarp();
            }
        }
        if (b == 0 && tid == 0) trace[k] = gt();
        if (DATA) {
            // read what the neighbour CTA wrote last round, write ours (dependent chain)
            const uint32_t src = (uint32_t)((b + 1) % g) * blockDim.x + tid;
            const uint32_t v = k ? *(volatile uint32_t*)&data[(size_t)((k - 1) & 1) * g * blockDim.x + src] : 0;
            acc += v;
            data[(size_t)(k & 1) * g * blockDim.x + (size_t)b * blockDim.x + tid] = v + 1;
        }
        if (MODE == 0) {
            __syncthreads();
            if (tid == 0) { __threadfence(); atomicAdd(&done[k], 1u); }
        } else if (MODE == 1) {
            __syncthreads();
            if (tid == 0) red_rel(&done[k], 1u);
        } else if (MODE == 2) {
            __syncwarp();
            if (lane == 0) red_rel(&done[k], 1u);
        } else {
            asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        }
    }
    if (acc == 0xFFFFFFFFu) trace[0] = acc;
}

template <int MODE, bool DATA>
void run(uint32_t* done, uint64_t* tr, uint32_t* data, int g, int threads, const char* name) {
    const int R = 400;
    cudaMemset(done, 0, R * 4 * 2);
    cudaMemset(data, 0, (size_t)2 * g * threads * 4);
    int rounds = R, ns = 0;
    void* args[] = {&done, &rounds, &tr, &data, &ns};
    cudaError_t e;
    if (MODE == 3) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(g);
        lc.blockDim = dim3(threads);
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = g; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
        lc.attrs = &at; lc.numAttrs = 1;
        if (g > 8) cudaFuncSetAttribute((const void*)handoff<MODE, DATA>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        e = cudaLaunchKernelExC(&lc, (const void*)handoff<MODE, DATA>, args);
    } else {
        e = cudaLaunchCooperativeKernel((void*)handoff<MODE, DATA>, dim3(g), dim3(threads), args, 0, 0);
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    std::vector<uint64_t> h(R);
    cudaMemcpy(h.data(), tr, R * 8, cudaMemcpyDeviceToHost);
    printf("%-8s data %d threads %4d g %3d: %6.3f us/round (%s)\n", name, (int)DATA, threads, g,
           (h[R - 1] - h[20]) / 1e3 / (R - 21), cudaGetErrorString(e));
}

int main() {
    uint32_t *done, *data; uint64_t* tr;
    cudaMalloc(&done, 400 * 4 * 2); cudaMalloc(&tr, 400 * 8); cudaMalloc(&data, 2 * 148 * 1024 * 4);
    for (int threads : {128, 1024}) {
        for (int g : {2, 8, 16, 32, 148}) {
            run<0, false>(done, tr, data, g, threads, "sc");
            run<1, false>(done, tr, data, g, threads, "rel");
            run<2, false>(done, tr, data, g, threads, "warp");
            run<0, true>(done, tr, data, g, threads, "sc");
            run<1, true>(done, tr, data, g, threads, "rel");
            run<2, true>(done, tr, data, g, threads, "warp");
            if (g <= 16) { run<3, false>(done, tr, data, g, threads, "cluster"); run<3, true>(done, tr, data, g, threads, "cluster"); }
        }
    }
    return 0;
}
