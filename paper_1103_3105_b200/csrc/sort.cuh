// sort.cuh — stable LSD radix sort of u64 keys on a bit range, onesweep style:
// one histogram pass over the keys for all digit passes, then per 8-bit digit pass a
// single kernel that ranks a 4096-key tile (warp multi-split from per-bit ballots),
// obtains the tile's global digit offsets by decoupled look-back, stages the tile in
// shared memory in digit order and writes it out coalesced.
//
// The paper groups access records "firstly on v and then on id" with a sort
// (§4.2) and partitions PART's transactions with a radix sort
// (§5.2).  Records are emitted in timestamp order, so a STABLE sort on
// the item (resp. partition) bits alone yields (item, ts) order.
#pragma once
#include "common.cuh"

namespace gputx {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;
constexpr int RS_WK = 32 * RS_ITEMS;               // keys per warp
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;     // 4096 keys per tile
constexpr int RS_MAXPASS = 5;
constexpr int RS_HIST_GRID = 148 * 8;            // (296 blocks: 160 us for 12 M keys, latency-bound)
constexpr int RS_HU = 8;                           // histogram: keys in flight per thread
constexpr int RS_LB = 8;                           // look-back window (tiles per round trip)

struct SortWs {
    uint32_t* hist;        // [RS_MAXPASS][256]
    uint64_t* status;      // [max_tiles][256]  (epoch:30 | kind:2) << 32 | value
    uint32_t* tickets;     // [64]
    uint64_t max_tiles;
    uint32_t items;        // keys per thread of a pass tile (8, 12 or 16; 0 = RS_ITEMS)
};

__global__ void __launch_bounds__(256) rs_hist_kernel(const uint64_t* __restrict__ keys,
                                                      const uint32_t* __restrict__ n_ptr, uint32_t lo,
                                                      uint32_t nbits, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[RS_MAXPASS][256];
    const uint32_t npass = (nbits + 7) / 8;
    for (uint32_t i = threadIdx.x; i < RS_MAXPASS * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint32_t n = *n_ptr;
    // RS_HU keys per thread in flight (grid-stride apart): one DRAM round trip per RS_HU keys
    // instead of one per key (12 M keys: 219 us latency-bound with one)
    const uint32_t nr = (n + 31) & ~31u, stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < nr; base += stride * RS_HU) {
        uint64_t k[RS_HU];
#pragma unroll
        for (int u = 0; u < RS_HU; ++u) {
            const uint64_t i = (uint64_t)base + (uint64_t)u * stride;
            k[u] = i < n ? __ldg(&keys[i]) : 0;
        }
#pragma unroll
        for (int u = 0; u < RS_HU; ++u) {
            const uint64_t i = (uint64_t)base + (uint64_t)u * stride;
            if (i - lane_id() >= nr) break;                 // warp-uniform (stride and nr are multiples of 32)
            const bool valid = i < n;
            for (uint32_t p = 0; p < npass; ++p) {
                const uint32_t w = min(8u, nbits - 8 * p);
                const uint32_t d = valid ? (uint32_t)(k[u] >> (lo + 8 * p)) & ((1u << w) - 1) : 0x100u;
                // a digit the whole warp shares (the high passes of clustered item ids): one
                // add; else one shared-memory atomic per lane (no __match_any_sync: its
                // throughput, not the loads, bounded this kernel)
                const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
                if (__all_sync(0xffffffffu, d == d0)) {
                    if (lane_id() == 0 && d0 < 256) atomicAdd(&h[p][d0], 32u);
                } else if (d < 256) {
                    atomicAdd(&h[p][d], 1u);
                }
            }
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < npass * 256; i += blockDim.x) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(&hist[i], v);
    }
}

// exclusive scan of each pass's 256 counts (one block per pass)
__global__ void __launch_bounds__(256) rs_scan_kernel(uint32_t* hist) {
    __shared__ uint32_t sm[8];
    uint32_t* h = hist + blockIdx.x * 256;
    uint32_t v = h[threadIdx.x], tot;
    uint32_t ex = block_scan_excl<uint32_t, OpAddU32>(v, tot, sm);
    h[threadIdx.x] = ex;
}

// lanes holding the same 9-bit value (digit, or 0x100 past the end) as this lane: the
// __match_any_sync result from 9 ballots (MATCH's issue rate bounded the passes)
DEV uint32_t rs_peers(uint32_t d) {
    uint32_t peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 9; ++b) {
        const bool bit = (d >> b) & 1u;
        const uint32_t bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
    }
    return peers;
}

DEV uint64_t rs_pack(uint32_t epoch, uint32_t kind, uint32_t v) {
    return ((uint64_t)((epoch << 2) | kind) << 32) | v;
}

template <int ITEMS>
__global__ void __launch_bounds__(RS_THREADS) rs_pass_kernel(const uint64_t* __restrict__ in,
                                                             uint64_t* __restrict__ out,
                                                             const uint32_t* __restrict__ n_ptr,
                                                             uint32_t shift, uint32_t mask,
                                                             const uint32_t* __restrict__ base,
                                                             uint64_t* status, uint32_t epoch,
                                                             uint32_t* ticket) {
    __shared__ uint32_t whist[RS_WARPS][256];
    __shared__ uint32_t tstart[256];
    __shared__ uint32_t gbase[256];
    __shared__ uint32_t scan_sm[8];
    constexpr int WK = 32 * ITEMS, TILE = RS_THREADS * ITEMS;
    __shared__ uint64_t stage[TILE];
    __shared__ uint32_t s_tile;

    const uint32_t n = *n_ptr;
    const uint32_t ntiles = (n + TILE - 1) / TILE;
    const uint32_t tid = threadIdx.x, lane = lane_id(), wid = warp_id();
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    for (uint32_t i = tid; i < RS_WARPS * 256; i += RS_THREADS) (&whist[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) return;
    const uint64_t tbase = (uint64_t)tile * TILE;

    uint64_t key[ITEMS];
    uint16_t loc[ITEMS];
    const uint64_t wbase = tbase + wid * WK;
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const uint64_t i = wbase + j * 32 + lane;
        key[j] = i < n ? __ldg(&in[i]) : ~0ull;
    }
    const uint32_t lmask = lanemask_lt();
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const uint64_t i = wbase + j * 32 + lane;
        const uint32_t d = i < n ? (uint32_t)(key[j] >> shift) & mask : 0x100u;
        const uint32_t peers = rs_peers(d);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if ((int)lane == leader && d < 256) {
            old = whist[wid][d];
            whist[wid][d] = old + __popc(peers);
        }
        old = __shfl_sync(0xffffffffu, old, leader);
        loc[j] = (uint16_t)(old + __popc(peers & lmask));
        __syncwarp();          // the next key's leader (another lane) reads this count
    }
    __syncthreads();
    // per digit: exclusive prefix over warps (in key order), tile count
    const uint32_t d = tid;                     // RS_THREADS == 256 digits
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
        const uint32_t c = whist[w][d];
        whist[w][d] = cnt;
        cnt += c;
    }
    // decoupled look-back per digit across tiles
    uint64_t* st = status + (uint64_t)tile * 256 + d;
    uint32_t excl = 0;
    if (tile == 0) {
        st_release64(st, rs_pack(epoch, 2, cnt));
    } else {
        st_release64(st, rs_pack(epoch, 1, cnt));
        // windowed look-back: RS_LB predecessors' (flag | count) words per round trip (each
        // word is self-contained, so relaxed loads suffice and stay in flight together)
        int64_t p = (int64_t)tile - 1;
        bool found = false;
        while (!found) {
            uint64_t sv[RS_LB];
#pragma unroll
            for (int i = 0; i < RS_LB; ++i)
                sv[i] = p - i >= 0 ? ld_relaxed64(status + (uint64_t)(p - i) * 256 + d) : rs_pack(epoch, 2, 0);
#pragma unroll
            for (int i = 0; i < RS_LB; ++i) {
                if (found) continue;
                while ((uint32_t)(sv[i] >> 34) != epoch) sv[i] = ld_relaxed64(status + (uint64_t)(p - i) * 256 + d);
                excl += (uint32_t)sv[i];
                found = ((sv[i] >> 32) & 3u) == 2u;
            }
            p -= RS_LB;
        }
        st_release64(st, rs_pack(epoch, 2, excl + cnt));
    }
    gbase[d] = base[d] + excl;
    uint32_t tot;
    tstart[d] = block_scan_excl<uint32_t, OpAddU32>(cnt, tot, scan_sm);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
        const uint64_t i = wbase + j * 32 + lane;
        if (i < n) {
            const uint32_t dj = (uint32_t)(key[j] >> shift) & mask;
            stage[tstart[dj] + whist[wid][dj] + loc[j]] = key[j];
        }
    }
    __syncthreads();
    const uint32_t tn = (n - tbase) < (uint64_t)TILE ? (uint32_t)(n - tbase) : (uint32_t)TILE;
    for (uint32_t i = tid; i < tn; i += RS_THREADS) {
        const uint64_t k = stage[i];
        const uint32_t dk = (uint32_t)(k >> shift) & mask;
        out[gbase[dk] + (i - tstart[dk])] = k;
    }
}

// Sorts n (device value, <= n_max) keys of a[] on bits [lo, lo+nbits).  Returns the
// buffer holding the result (a or b).  epoch is advanced by the passes used.
inline uint64_t* radix_sort_u64(uint64_t* a, uint64_t* b, const uint32_t* n_dev, uint64_t n_max, uint32_t lo,
                                uint32_t nbits, SortWs& ws, uint32_t& epoch, cudaStream_t s) {
    if (n_max == 0 || nbits == 0) return a;
    const uint32_t npass = (nbits + 7) / 8;
    dev_fill_multi(s, {fseg(ws.hist, 0, sizeof(uint32_t) * RS_MAXPASS * 256), fseg(ws.tickets, 0, sizeof(uint32_t) * 64)});
    rs_hist_kernel<<<RS_HIST_GRID, 256, 0, s>>>(a, n_dev, lo, nbits, ws.hist);
    rs_scan_kernel<<<npass, 256, 0, s>>>(ws.hist);
    const uint32_t tile = RS_THREADS * (ws.items ? ws.items : RS_ITEMS);
    const uint32_t grid = (uint32_t)((n_max + tile - 1) / tile);
    uint64_t* src = a;
    uint64_t* dst = b;
    for (uint32_t p = 0; p < npass; ++p) {
        const uint32_t w = nbits - 8 * p < 8 ? nbits - 8 * p : 8;
        ++epoch;
        auto fn = ws.items == 8 ? rs_pass_kernel<8> : ws.items == 12 ? rs_pass_kernel<12> : rs_pass_kernel<RS_ITEMS>;
        fn<<<grid, RS_THREADS, 0, s>>>(src, dst, n_dev, lo + 8 * p, (1u << w) - 1, ws.hist + p * 256,
                                       ws.status, epoch, ws.tickets + p);
        uint64_t* t = src; src = dst; dst = t;
    }
    return src;
}

}  // namespace gputx
