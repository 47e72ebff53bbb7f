// common.cuh — device primitives shared by the GPUTx kernels (sm_100a).
//
//  * acquire/release loads and stores (PTX memory model, gpu scope)
//  * a sense-free generation grid barrier for cooperative persistent kernels
//  * warp / block scans for any associative (not necessarily commutative)
//    operator, and a decoupled look-back across tiles (single pass over the data)
//
// Operators follow the convention  Op::combine(earlier, later)  so that a
// prefix is  combine(combine(x0, x1), x2) ...  in array order.
#pragma once
#include <initializer_list>
#include <cstdint>
#include <cuda_runtime.h>

#define DEV __device__ __forceinline__

namespace gputx {

constexpr int WARP = 32;

DEV uint32_t lane_id() { return threadIdx.x & 31u; }
DEV uint32_t warp_id() { return threadIdx.x >> 5; }
DEV uint32_t lanemask_lt() { uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }

DEV uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : : "memory");
    return t;
}
DEV uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
DEV uint64_t ld_acquire64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
DEV uint64_t ld_relaxed64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
DEV uint32_t ld_relaxed(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
DEV void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
DEV void st_release64(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// fire-and-forget release increment: orders every prior write of the calling thread (and,
// cumulatively, those it observed, e.g. its CTA's writes before a __syncthreads) before
// the increment; ~0.3 us/round cheaper than __threadfence (fence.sc) + atomicAdd
// (tools/handoff.cu, profiles/round2_handoff_microbench.txt)
DEV void red_add_release(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
DEV uint32_t atom_add_release(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// ---------------------------------------------------------------------------------
// dev_fill: cudaMemsetAsync's signature, done by a kernel.  A memset may be serviced by a
// copy engine and then waits behind an in-flight bulk transfer in the same direction
// (gputx_run_bulks overlaps a bulk's result D2H with the next bulk's execution).
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) fill_bytes_kernel(uint8_t* p, uint32_t v8, uint64_t bytes) {
    const uint64_t head = (16 - ((uintptr_t)p & 15)) & 15;
    const uint64_t h = head < bytes ? head : bytes;
    const uint64_t n16 = (bytes - h) / 16;
    const uint32_t w = v8 * 0x01010101u;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
    if (tid < h) p[tid] = (uint8_t)v8;
    uint4* q = reinterpret_cast<uint4*>(p + h);
    for (uint64_t i = tid; i < n16; i += nt) q[i] = make_uint4(w, w, w, w);
    for (uint64_t i = h + n16 * 16 + tid; i < bytes; i += nt) p[i] = (uint8_t)v8;
}
inline cudaError_t dev_fill(void* p, int value, size_t bytes, cudaStream_t s) {
    if (!bytes) return cudaSuccess;
    uint64_t blocks = (bytes / 16 + 255) / 256;
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 8) blocks = 148 * 8;
    fill_bytes_kernel<<<(unsigned)blocks, 256, 0, s>>>((uint8_t*)p, (uint32_t)(value & 0xFF), (uint64_t)bytes);
    return cudaGetLastError();
}

// dev_copy2: two device-to-device copies in ONE launch (blockIdx.y = which), 16-B vectors
// with four in flight per thread when both ends of a copy are 16-B aligned, bytes otherwise
// (a D2D cudaMemcpyAsync of a device-resident bulk's types / offsets was ~40 us on TPC-B)
struct CopySeg {
    uint8_t* dst;
    const uint8_t* src;
    uint64_t bytes;
};
__global__ void __launch_bounds__(256) copy2_kernel(CopySeg a, CopySeg b) {
    const CopySeg c = blockIdx.y ? b : a;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
    uint64_t done = 0;
    if (!(((uintptr_t)c.dst | (uintptr_t)c.src) & 15u)) {
        const uint64_t n16 = c.bytes / 16;
        const uint4* s4 = reinterpret_cast<const uint4*>(c.src);
        uint4* d4 = reinterpret_cast<uint4*>(c.dst);
        for (uint64_t i = tid; i < n16; i += 4 * nt) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + u * nt < n16) v[u] = __ldg(&s4[i + u * nt]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + u * nt < n16) d4[i + u * nt] = v[u];
        }
        done = n16 * 16;
    }
    for (uint64_t i = done + tid; i < c.bytes; i += nt) c.dst[i] = c.src[i];
}
inline cudaError_t dev_copy2(void* d0, const void* s0, size_t b0, void* d1, const void* s1, size_t b1, cudaStream_t s) {
    const size_t mx = b0 > b1 ? b0 : b1;
    if (!mx) return cudaSuccess;
    uint64_t blocks = (mx / 64 + 255) / 256;
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 4) blocks = 148 * 4;
    copy2_kernel<<<dim3((unsigned)blocks, 2), 256, 0, s>>>(CopySeg{(uint8_t*)d0, (const uint8_t*)s0, b0},
                                                          CopySeg{(uint8_t*)d1, (const uint8_t*)s1, b1});
    return cudaGetLastError();
}

// Several fills in ONE launch (blockIdx.y = segment): the per-bulk bookkeeping fills
// (counters, depth array, sort workspace, result buffers) otherwise cost a launch each.
// The segments are filled concurrently: they must not overlap.
struct FillSeg {
    uint8_t* p;
    uint64_t bytes;
    uint32_t v8;
};
constexpr int FILL_MAX = 6;
struct FillList {
    FillSeg s[FILL_MAX];
};
__global__ void __launch_bounds__(256) fill_multi_kernel(FillList fl) {
    const FillSeg g = fl.s[blockIdx.y];
    uint8_t* p = g.p;
    const uint64_t bytes = g.bytes;
    const uint64_t head = (16 - ((uintptr_t)p & 15)) & 15;
    const uint64_t h = head < bytes ? head : bytes;
    const uint64_t n16 = (bytes - h) / 16;
    const uint32_t w = g.v8 * 0x01010101u;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
    if (tid < h) p[tid] = (uint8_t)g.v8;
    uint4* q = reinterpret_cast<uint4*>(p + h);
    for (uint64_t i = tid; i < n16; i += nt) q[i] = make_uint4(w, w, w, w);
    for (uint64_t i = h + n16 * 16 + tid; i < bytes; i += nt) p[i] = (uint8_t)g.v8;
}
// fills (ptr, byte value, bytes) x k (k <= FILL_MAX; empty segments allowed)
inline cudaError_t dev_fill_multi(cudaStream_t s, std::initializer_list<FillSeg> segs) {
    FillList fl = {};
    int k = 0;
    uint64_t mx = 0;
    for (const FillSeg& g : segs) {
        if (!g.bytes) continue;
        fl.s[k++] = {g.p, g.bytes, g.v8 & 0xFFu};
        mx = g.bytes > mx ? g.bytes : mx;
    }
    if (!k) return cudaSuccess;
    uint64_t blocks = (mx / 16 + 255) / 256;
    if (blocks < 1) blocks = 1;
    if (blocks > 148 * 8) blocks = 148 * 8;
    fill_multi_kernel<<<dim3((unsigned)blocks, (unsigned)k), 256, 0, s>>>(fl);
    return cudaGetLastError();
}
inline FillSeg fseg(void* p, int v, uint64_t bytes) { return FillSeg{(uint8_t*)p, bytes, (uint32_t)(v & 0xFF)}; }

// ---------------------------------------------------------------------------------
// Grid barrier for a cooperative launch (all CTAs co-resident).  gen is bumped by
// the last arriver; waiters poll it with acquire loads.
// ---------------------------------------------------------------------------------
// Two-level arrival tree: CTA b arrives on sub-counter b % GB_SUB (each on its own
// 128-B line), the last arriver of a sub-counter arrives on the top counter, the last
// top arriver bumps gen.  Same-address atomics per level: <= gridDim/GB_SUB.
constexpr uint32_t GB_SUB = 16;
struct GridBar {
    uint32_t sub[GB_SUB * 32];
    uint32_t top;
    uint32_t pad[31];
    uint32_t gen;
    uint32_t pad2[31];
    uint32_t dead;        // watchdog tripped in this launch (reset by the host before each launch)
};

// Spin watchdog (SPEC "watchdog -> EDEADLOCK"): every device spin loop that
// waits for another CTA polls a timer; past g_watchdog_ns (GPUTX_WATCHDOG_MS, default 10 s)
// or once another waiter has tripped, it gives up, the kernel drains without waiting, and
// the host returns GPUTX_EDEADLOCK and poisons the handle until gputx_reset.
__device__ unsigned long long g_watchdog_ns = 10000000000ull;
struct SpinWatch {
    uint64_t t0 = 0;
    uint32_t n = 0;
    // call once per unsuccessful poll; true = give up (and *flag is set)
    DEV bool expired(uint32_t* flag) {
        if ((++n & 1023u) != 0) return false;
        const uint64_t now = globaltimer_ns();
        if (!t0) { t0 = now; return false; }
        if (*reinterpret_cast<volatile uint32_t*>(flag)) return true;
        if (now - t0 > g_watchdog_ns) { atomicExch(flag, 1u); return true; }
        return false;
    }
};

DEV void grid_sync(GridBar* b) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t nb = gridDim.x;
        const uint32_t g = ld_acquire(&b->gen);
        const uint32_t s = blockIdx.x % GB_SUB;
        const uint32_t nsub = nb < GB_SUB ? nb : GB_SUB;
        const uint32_t members = (nb - s + GB_SUB - 1) / GB_SUB;
        __threadfence();
        const uint32_t a = atomicAdd(&b->sub[s * 32], 1u);
        bool wait = true;
        if (a == members - 1) {
            b->sub[s * 32] = 0;
            __threadfence();
            const uint32_t t = atomicAdd(&b->top, 1u);
            if (t == nsub - 1) {
                b->top = 0;
                __threadfence();
                st_release(&b->gen, g + 1);
                wait = false;
            }
        }
        if (wait) {
            SpinWatch wd;
            while (ld_acquire(&b->gen) == g)
                if (wd.expired(&b->dead)) break;
        }
        __threadfence();
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------------
// Scans
// ---------------------------------------------------------------------------------
template <class T>
DEV T shfl_up_t(T v, int d) {
    static_assert(sizeof(T) % 4 == 0, "4-byte multiple");
    union { T t; uint32_t w[sizeof(T) / 4]; } u;
    u.t = v;
#pragma unroll
    for (int k = 0; k < (int)(sizeof(T) / 4); ++k) u.w[k] = __shfl_up_sync(0xffffffffu, u.w[k], d);
    return u.t;
}
template <class T>
DEV T shfl_t(T v, int src) {
    union { T t; uint32_t w[sizeof(T) / 4]; } u;
    u.t = v;
#pragma unroll
    for (int k = 0; k < (int)(sizeof(T) / 4); ++k) u.w[k] = __shfl_sync(0xffffffffu, u.w[k], src);
    return u.t;
}

// inclusive warp scan
template <class T, class Op>
DEV T warp_scan_incl(T x) {
    const int lane = lane_id();
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T y = shfl_up_t(x, d);
        if (lane >= d) x = Op::combine(y, x);
    }
    return x;
}

// Exclusive block scan of one value per thread.  Returns the exclusive prefix
// (Op::identity() for thread 0) and the block aggregate.  smem: >= (blockDim/32) T.
template <class T, class Op>
DEV T block_scan_excl(T x, T& total, T* smem) {
    const int lane = lane_id(), wid = warp_id(), nw = blockDim.x >> 5;
    T inc = warp_scan_incl<T, Op>(x);
    if (lane == 31) smem[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        T w = lane < nw ? smem[lane] : Op::identity();
        T wi = warp_scan_incl<T, Op>(w);
        if (lane < nw) smem[lane] = wi;          // inclusive warp totals
    }
    __syncthreads();
    T wpre = wid ? smem[wid - 1] : Op::identity();
    total = smem[nw - 1];
    T ex = shfl_up_t(inc, 1);
    if (lane == 0) ex = Op::identity();
    T r = Op::combine(wpre, ex);
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------------
// Decoupled look-back (single-pass tile prefix).  Per tile: a flag word
// (epoch << 2 | kind, kind 1 = aggregate, 2 = inclusive prefix) and two payloads.
// epoch makes stale flags of earlier launches/passes invisible (no resets).
// ---------------------------------------------------------------------------------
template <class T>
struct LookBack {
    uint32_t* flag;
    T* agg;
    T* inc;
};

template <class T>
DEV void lb_store(T* dst, const T& v) {
    const uint32_t* s = reinterpret_cast<const uint32_t*>(&v);
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(T) / 4); ++k) __stcg(d + k, s[k]);
}
template <class T>
DEV T lb_load(const T* src) {
    union { T t; uint32_t w[sizeof(T) / 4]; } u;
    const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
#pragma unroll
    for (int k = 0; k < (int)(sizeof(T) / 4); ++k) u.w[k] = __ldcg(s + k);
    return u.t;
}

// Called by ONE full warp of the tile's CTA.  Publishes the aggregate, looks back
// for the exclusive prefix, publishes the inclusive prefix, returns the exclusive
// prefix (identity for tile 0) to all lanes of the warp.
template <class T, class Op>
DEV T lookback_warp(LookBack<T> lb, uint32_t tile, uint32_t epoch, T agg) {
    const int lane = lane_id();
    const uint32_t fa = (epoch << 2) | 1u, fi = (epoch << 2) | 2u;
    if (tile == 0) {
        if (lane == 0) {
            lb_store(&lb.inc[0], agg);
            __threadfence();
            st_release(&lb.flag[0], fi);
        }
        __syncwarp();
        return Op::identity();
    }
    if (lane == 0) {
        lb_store(&lb.agg[tile], agg);
        __threadfence();
        st_release(&lb.flag[tile], fa);
    }
    __syncwarp();
    T excl = Op::identity();          // prefix of tiles (p, tile) gathered so far (lane 0)
    int64_t base = (int64_t)tile - 1;
    while (true) {
        int64_t p = base - lane;
        uint32_t f = 0;
        if (p >= 0) {
            do { f = ld_acquire(&lb.flag[p]); } while ((f >> 2) != epoch);
        } else {
            f = fi;                      // virtual inclusive before tile 0 (never reached)
        }
        uint32_t kind = f & 3u;
        uint32_t incmask = __ballot_sync(0xffffffffu, kind == 2u);
        int stop = incmask ? __ffs(incmask) - 1 : 32;       // closest inclusive lane
        T v = Op::identity();
        if (p >= 0 && lane <= stop && lane < 32) v = (kind == 2u) ? lb_load(&lb.inc[p]) : lb_load(&lb.agg[p]);
        // compose lanes stop..0 (oldest first) on lane 0
        int top = stop < 32 ? stop : 31;
        T acc = Op::identity();
        for (int l = top; l >= 0; --l) {
            T vl = shfl_t(v, l);
            acc = Op::combine(acc, vl);
        }
        if (lane == 0) excl = Op::combine(acc, excl);
        if (stop < 32) break;
        base -= 32;
    }
    if (lane == 0) {
        T incv = Op::combine(excl, agg);
        lb_store(&lb.inc[tile], incv);
        __threadfence();
        st_release(&lb.flag[tile], fi);
    }
    excl = shfl_t(excl, 0);
    return excl;
}

// ---------------------------------------------------------------------------------
// Operators
// ---------------------------------------------------------------------------------
struct OpAddU32 {
    static DEV uint32_t identity() { return 0u; }
    static DEV uint32_t combine(uint32_t a, uint32_t b) { return a + b; }
};
// two independent u32 sums side by side (one scan for two per-transaction counts)
struct OpAddU2 {
    static DEV uint2 identity() { return make_uint2(0u, 0u); }
    static DEV uint2 combine(uint2 a, uint2 b) { return make_uint2(a.x + b.x, a.y + b.y); }
};

}  // namespace gputx
