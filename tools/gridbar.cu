// Microbenchmark: cost of the two-level tree grid barrier (common.cuh grid_sync).
#include <cstdio>
#include <vector>
#include "../paper_1103_3105_b200/csrc/common.cuh"
using namespace gputx;

__global__ void bar_kernel(GridBar* bar, int rounds, uint64_t* trace) {
    for (int k = 0; k < rounds; ++k) {
        if (blockIdx.x == 0 && threadIdx.x == 0) trace[k] = globaltimer_ns();
        grid_sync(bar);
    }
}

int main() {
    const int R = 300;
    GridBar* bar; uint64_t* tr;
    cudaMalloc(&bar, sizeof(GridBar)); cudaMalloc(&tr, R * 8);
    for (int threads : {256, 1024}) for (int g : {2, 16, 148, 296}) {
        if (threads == 1024 && g > 148) continue;
        cudaMemset(bar, 0, sizeof(GridBar));
        int rounds = R;
        void* args[] = {&bar, &rounds, &tr};
        cudaError_t e = cudaLaunchCooperativeKernel((void*)bar_kernel, dim3(g), dim3(threads), args, 0, 0);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        std::vector<uint64_t> h(R);
        cudaMemcpy(h.data(), tr, R * 8, cudaMemcpyDeviceToHost);
        printf("threads %4d grid %3d: %.2f us/barrier (%s)\n", threads, g, (h[R - 1] - h[10]) / 1e3 / (R - 11),
               cudaGetErrorString(e));
    }
}
