// Runs the library's kset_exec_kernel<TM-1> in isolation (fake schedule, diag=13: no
// transaction bodies) to separate code generation from memory state.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1103_3105_b200/csrc/kernels.cuh"
using namespace gputx;

__global__ void touch(uint16_t* g, uint32_t* done, uint32_t nk, const uint16_t* src) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nk; k += gridDim.x * blockDim.x) {
        g[k] = src[k];
        done[k] = 0;
    }
}

int main() {
    uint32_t nk = 195;
    const uint32_t T = 7, n = 1000000;
    std::vector<uint16_t> hg(nk, 1);
    for (int k = 0; k < 24; ++k) hg[k] = 2;
    std::vector<uint32_t> hoff((nk + 1) * T + 1);
    for (uint32_t k = 0; k <= nk * T; ++k) hoff[k] = (uint32_t)((uint64_t)k * n / (nk * T));
    if (getenv("SCHED")) {
        FILE* f = fopen(getenv("SCHED"), "rb");
        fread(&nk, 4, 1, f);
        hoff.assign(nk * T + 1 + T, 0);
        fread(hoff.data(), 4, nk * T + 1, f);
        for (uint32_t i = nk * T + 1; i < hoff.size(); ++i) hoff[i] = hoff[nk * T];
        hg.assign(nk, 1);
        fread(hg.data(), 2, nk, f);
        fclose(f);
        printf("loaded real schedule: nk %u\n", nk);
    }
    uint16_t* g; uint32_t *off, *done, *sc, *perm, *pp; uint8_t* ptype; uint64_t* tr;
    cudaMalloc(&g, nk * 2); cudaMalloc(&off, hoff.size() * 4); cudaMalloc(&done, nk * 4);
    cudaMalloc(&sc, 64 * 4); cudaMalloc(&perm, n * 4); cudaMalloc(&pp, n * 32); cudaMalloc(&ptype, n);
    cudaMalloc(&tr, nk * 64);
    cudaMemcpy(g, hg.data(), nk * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(off, hoff.data(), hoff.size() * 4, cudaMemcpyHostToDevice);
    std::vector<uint32_t> hsc(64, 0);
    hsc[SC_MAXD] = nk - 1;
    cudaMemcpy(sc, hsc.data(), 64 * 4, cudaMemcpyHostToDevice);
    cudaMemset(perm, 0, n * 4); cudaMemset(pp, 0, n * 32); cudaMemset(ptype, 0, n);
    DevDb db{};
    uint8_t* big;
    cudaMalloc(&big, 1ull << 30);
    std::vector<void*> hog;
    if (getenv("HOG_GB")) {
        for (int i = 0; i < atoi(getenv("HOG_GB")); ++i) { void* p; cudaMalloc(&p, 1ull << 30); cudaMemset(p, 0, 1ull << 30); hog.push_back(p); }
    }
    cudaStream_t nb;
    cudaStreamCreateWithFlags(&nb, cudaStreamNonBlocking);
    uint16_t* gsrc; cudaMalloc(&gsrc, nk * 2); cudaMemcpy(gsrc, hg.data(), nk * 2, cudaMemcpyHostToDevice);
    for (uint32_t diag : {13u, 141u, 13u + 4096u, 13u + 8192u, 13u + 16384u}) {
        if (diag & 4096u) { cudaMemset(big, 1, 1ull << 30); }
        cudaMemset(done, 0, nk * 4);
        if (diag & 16384u) touch<<<592, 256>>>(g, done, nk, gsrc);
        uint32_t TT = T;
        uint32_t C0 = 0;
        void* args[] = {&db, &perm, &off, &TT, &g, &done, &sc, &ptype, &pp, &tr, &diag, &C0};
        cudaError_t e = cudaLaunchCooperativeKernel((void*)kset_exec_kernel<S_TM1, 8, 1024>, dim3(2), dim3(1024), args, 0,
                                                    (diag & 8192u) ? nb : (cudaStream_t)0);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        std::vector<uint64_t> h(nk * 8);
        cudaMemcpy(h.data(), tr, nk * 64, cudaMemcpyDeviceToHost);
        double wide = 0, narrow = 0;
        for (uint32_t k = 0; k + 1 < nk; ++k) {
            double dt = (double)(h[8 * (k + 1)] - h[8 * k]) / 1e3;
            if (k < 24) wide += dt; else narrow += dt;
        }
        printf("diag %u: wide %.2f us/round (polls r5 %llu), narrow %.2f us/round (%s)\n", diag, wide / 24,
               (unsigned long long)h[8 * 5 + 4], narrow / (nk - 25), cudaGetErrorString(e));
    }
}
