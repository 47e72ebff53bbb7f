// Microbenchmark: round hand-off latency between CTAs through per-round counters
// (the K-SET executor's protocol), with and without the executor's extras.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) {
    uint32_t v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}

__global__ void pingpong(uint32_t* done, int rounds, int g, uint64_t* trace, int mode) {
    const int b = blockIdx.x;
    if (b >= g) return;
    for (int k = 0; k < rounds; ++k) {
        if (k > 0) {
            if (threadIdx.x == 0) while (ld_acq(&done[k - 1]) < (uint32_t)g) { }
            __syncthreads();
        }
        if (b == 0 && threadIdx.x == 0) trace[k] = gt();
        __syncthreads();
        if (threadIdx.x == 0) {
            if (mode == 0) { __threadfence(); atomicAdd(&done[k], 1u); }
            else { asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&done[k]) : "memory"); }
        }
    }
}

int main() {
    const int R = 200;
    uint32_t* done; uint64_t* tr;
    cudaMalloc(&done, R * 4 * 64); cudaMalloc(&tr, R * 8);
    for (int threads : {128, 1024}) for (int g : {2, 8, 32, 148}) for (int mode : {0, 1}) {
        cudaMemset(done, 0, R * 4 * 64);
        int rounds = R;
        void* args[] = {&done, &rounds, &g, &tr, &mode};
        cudaLaunchCooperativeKernel((void*)pingpong, dim3(g), dim3(threads), args, 0, 0);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<uint64_t> h(R);
        cudaMemcpy(h.data(), tr, R * 8, cudaMemcpyDeviceToHost);
        printf("threads %4d g %3d mode %d: %.2f us/round (%s)\n", threads, g, mode,
               (h[R - 1] - h[10]) / 1e3 / (R - 11), cudaGetErrorString(e));
    }
    return 0;
}
