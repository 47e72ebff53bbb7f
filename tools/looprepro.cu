// Standalone copy of the K-SET executor's round loop (no transaction bodies) on a
// TM-1-like round schedule, to bisect the multi-CTA hand-off latency.
#include <cstdio>
#include <vector>
#include "../paper_1103_3105_b200/csrc/common.cuh"
using namespace gputx;

constexpr uint32_t CH = 2048;

template <int KB>
__global__ void __launch_bounds__(KB) loop_kernel(const uint32_t* off, const uint16_t* g, uint32_t* done, uint32_t nk,
                                                  uint64_t* trace, uint32_t mode) {
    const uint32_t b = blockIdx.x, tid = threadIdx.x;
    __shared__ uint16_t sg[CH];
    __shared__ uint32_t soff[CH + 1];
    uint32_t cb = 0xFFFFFFFFu;
    auto load_chunk = [&](uint32_t base) {
        __syncthreads();
        for (uint32_t i = tid; i < CH; i += KB) sg[i] = base + i < nk ? __ldg(&g[base + i]) : (uint16_t)0;
        for (uint32_t i = tid; i <= CH; i += KB) soff[i] = base + i <= nk ? __ldcg(&off[base + i]) : 0u;
        __syncthreads();
        cb = base;
    };
    auto G = [&](uint32_t kk) -> uint32_t {
        if (kk < cb || kk >= cb + CH) load_chunk(kk - kk % CH);
        return sg[kk - cb];
    };
    uint32_t k = 0;
    while (k < nk && G(k) <= b) ++k;
    if (k >= nk) return;
    uint32_t prev = 0xFFFFFFFFu, gprev = 0;
    while (k < nk) {
        const uint32_t gk = G(k);
        if (k > 0) {
            const bool mine = (prev == k - 1) && gprev == 1;
            if (!mine) {
                if (tid == 0) {
                    const uint32_t need = prev == k - 1 ? gprev : __ldg(&g[k - 1]);
                    uint32_t spins = 0;
                    while (ld_acquire(&done[k - 1]) < need) ++spins;
                    if (b < 2) trace[8 * k + 4 + b] = spins;
                }
                __syncthreads();
            }
        }
        if (b < 2 && tid == 0) trace[8 * k + 2 * b] = globaltimer_ns();
        uint32_t k2 = k + 1;
        if (mode & 1) { while (k2 < nk && __ldg(&g[k2]) <= b) ++k2; }
        else { while (k2 < nk && G(k2) <= b) ++k2; }
        __syncthreads();
        const bool next_shared = b > 0 || ((k + 1 < nk) && G(k + 1) > 1);
        if (tid == 0 && (gk > 1 || next_shared)) {
            __threadfence();
            atomicAdd(&done[k], 1u);
        }
        if (b < 2 && tid == 0) trace[8 * k + 2 * b + 1] = globaltimer_ns();
        prev = k;
        gprev = gk;
        k = k2;
    }
}

int main() {
    // TM-1 NURand-like: 24 rounds with 2 CTAs, then 171 rounds with 1
    const uint32_t nk = 195;
    std::vector<uint16_t> hg(nk, 1);
    for (int k = 0; k < 24; ++k) hg[k] = 2;
    std::vector<uint32_t> hoff(nk + 1);
    for (uint32_t k = 0; k <= nk; ++k) hoff[k] = k * 100;
    uint16_t* g; uint32_t *off, *done; uint64_t* tr;
    cudaMalloc(&g, nk * 2); cudaMalloc(&off, (nk + 1) * 4); cudaMalloc(&done, nk * 4); cudaMalloc(&tr, nk * 64);
    cudaMemcpy(g, hg.data(), nk * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(off, hoff.data(), (nk + 1) * 4, cudaMemcpyHostToDevice);
    for (uint32_t mode : {0u, 1u}) {
        cudaMemset(done, 0, nk * 4);
        cudaMemset(tr, 0, nk * 64);
        uint32_t nk_ = nk;
        void* args[] = {&off, &g, &done, &nk_, &tr, &mode};
        cudaError_t e = cudaLaunchCooperativeKernel((void*)loop_kernel<1024>, dim3(2), dim3(1024), args, 0, 0);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        std::vector<uint64_t> h(nk * 8);
        cudaMemcpy(h.data(), tr, nk * 64, cudaMemcpyDeviceToHost);
        double wide = 0, narrow = 0;
        for (uint32_t k = 0; k + 1 < nk; ++k) {
            double dt = (double)(h[8 * (k + 1)] - h[8 * k]) / 1e3;
            if (k < 24) wide += dt; else narrow += dt;
        }
        printf("mode %u: wide %.2f us/round (spins r5 %llu), narrow %.2f us/round (%s)\n", mode, wide / 24,
               (unsigned long long)h[8 * 5 + 4], narrow / (nk - 25), cudaGetErrorString(e));
    }
}
