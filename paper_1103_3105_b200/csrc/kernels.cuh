// kernels.cuh — the bulk-generation and bulk-execution kernels (sm_100a).
//
//   ingest      validate signatures, resolve split lookups, insert-row counts
//   scan        exclusive prefix sums (single pass, decoupled look-back)
//   emit        per-transaction access records  key = item<<30 | idx<<6 | j<<2 | W
//   rank        iterated segmented max-plus scan to the depth fixpoint         (corrected, DESIGN.md R-S1)
//   group       counting sort of transactions by (depth, type)
//   kset_exec   persistent k-set round loop, no locks                          (§5.3)
//   part_*      fragment map, partition bounds, one thread per partition       (§5.2)
//   tpl_*       counter-lock keys from the sorted records, ts-ordered 2PL      (App. C Fig. 11)
#pragma once
#include "common.cuh"
#include "schema.cuh"

namespace gputx {

// ---- device scalar slots (u32) -------------------------------------------------------
enum {
    SC_ERR = 0, SC_BADIDX, SC_NREC, SC_NFRAG, SC_MAXD, SC_ZERO, SC_PASSES, SC_CHG0, SC_CHG1, SC_CHG2,
    SC_KNEXT, SC_TICKET, SC_DEADLOCK, SC_MAXCHAIN, SC_NKEYS, SC_NKEYS1, SC_COMMITTED, SC_NOCONV,
    SC_COUNT = 32
};
enum { E_TYPE = 1, E_UNREG = 2, E_LEN = 3, E_RANGE = 4, E_OFF = 5 };

// TM-1 sub_nbr hash (shared host/device)
__host__ __device__ inline uint64_t nbr_hash(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

DEV void report_err(uint32_t* sc, uint32_t code, uint32_t idx) {
    atomicMin(&sc[SC_BADIDX], idx);
    atomicMax(&sc[SC_ERR], code);
}

// =====================================================================================
// ingest: validate in place, resolve static lookups, count insert rows
// =====================================================================================
template <int S>
__global__ void __launch_bounds__(256) ingest_kernel(DevDb db, uint32_t* pw, uint32_t n_words, uint32_t type_mask,
                                                     uint32_t* ins_cnt, uint32_t ins_stride, uint32_t* sc) {
    const uint32_t n = db.n;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t t = db.type[i];
        const uint32_t o0 = db.poff[i], o1 = db.poff[i + 1];
        if (i == 0 && o0 != 0) { report_err(sc, E_OFF, i); continue; }
        if (i == n - 1 && o1 != n_words) { report_err(sc, E_OFF, i); continue; }
        if (o1 < o0 || o1 > n_words) { report_err(sc, E_OFF, i); continue; }
        if (t >= db.ntypes) { report_err(sc, E_TYPE, i); continue; }
        if (!((type_mask >> t) & 1u)) { report_err(sc, E_UNREG, i); continue; }
        uint32_t* p = pw + o0;
        const uint32_t len = o1 - o0;
        if (S == S_TPCB) {
            const uint32_t B = db.dims[0], T = db.dims[1], A = db.dims[2];
            if (len != 4) { report_err(sc, E_LEN, i); continue; }
            if (p[0] >= B * A || p[1] >= B * T || p[2] >= B) { report_err(sc, E_RANGE, i); continue; }
        } else if (S == S_TM1) {
            const uint32_t P = db.dims[0];
            const uint8_t need[7] = {1, 4, 2, 4, 3, 7, 4};
            if (len != need[t]) { report_err(sc, E_LEN, i); continue; }
            if (t <= 3) {
                if (p[0] < 1 || p[0] > P) { report_err(sc, E_RANGE, i); continue; }
                if ((t == 1 || t == 3) && (p[1] < 1 || p[1] > 4)) { report_err(sc, E_RANGE, i); continue; }
                if (t == 2 && (p[1] < 1 || p[1] > 4)) { report_err(sc, E_RANGE, i); continue; }
                if (t == 1 && (p[2] > 16 || (p[2] & 7))) { report_err(sc, E_RANGE, i); continue; }
            } else {
                if (t >= 5 && (p[2] < 1 || p[2] > 4 || p[3] > 16 || (p[3] & 7))) { report_err(sc, E_RANGE, i); continue; }
                // the lookup half of the split transaction: sub_nbr -> s_id
                const uint64_t nbr = (uint64_t)p[0] | ((uint64_t)p[1] << 32);
                uint32_t sid = 0;
                uint64_t h = nbr_hash(nbr) & db.hmask;
                while (true) {
                    const uint64_t k = __ldg(&db.hkeys[h]);
                    if (k == 0) break;
                    if (k == nbr) { sid = __ldg(&db.hvals[h]); break; }
                    h = (h + 1) & db.hmask;
                }
                p[0] = sid;
                p[1] = 0;
            }
        } else {
            const uint32_t W = db.dims[0], D = db.dims[1], C = db.dims[2], I = db.dims[3];
            if (t == 0) {
                if (len < 4) { report_err(sc, E_LEN, i); continue; }
                const uint32_t cnt = p[3];
                if (cnt < 1 || cnt > 15 || len != 4 + 3 * cnt) { report_err(sc, E_LEN, i); continue; }
                if (p[0] >= W || p[1] >= D || p[2] >= C) { report_err(sc, E_RANGE, i); continue; }
                bool bad = false, abort = false;
                for (uint32_t l = 0; l < cnt; ++l) {
                    bad |= p[4 + 3 * l] > I || p[5 + 3 * l] >= W || p[6 + 3 * l] < 1 || p[6 + 3 * l] > 1000;
                    abort |= p[4 + 3 * l] >= I;
                }
                if (bad) { report_err(sc, E_RANGE, i); continue; }
                if (!abort) {
                    ins_cnt[T_ORDER * ins_stride + i] = 1;
                    ins_cnt[T_NEWORDER * ins_stride + i] = 1;
                    ins_cnt[T_OLINE * ins_stride + i] = cnt;
                }
            } else {
                if (len != 7) { report_err(sc, E_LEN, i); continue; }
                if (p[0] >= W || p[1] >= D || p[2] >= W || p[3] >= D || p[4] > 1 || p[6] > 0x7FFFFFFFu) {
                    report_err(sc, E_RANGE, i); continue;
                }
                if (p[4] == 1) {
                    // the lookup half of the split Payment: (cw, cd, c_last) -> c_id,
                    // row ceil(n/2) of the customers with that last name ordered by c_first
                    if (p[5] >= 1000) { report_err(sc, E_RANGE, i); continue; }
                    const uint64_t g = ((uint64_t)p[2] * D + p[3]) * 1000 + p[5];
                    const uint32_t lo = __ldg(&db.name_off[g]), hi = __ldg(&db.name_off[g + 1]);
                    if (hi == lo) {
                        p[4] = 2;
                    } else {
                        p[5] = __ldg(&db.name_sorted[lo + (hi - lo + 1) / 2 - 1]);
                        p[4] = 0;
                    }
                } else if (p[5] >= C) {
                    report_err(sc, E_RANGE, i); continue;
                }
                if (p[4] != 2) ins_cnt[T_HIST * ins_stride + i] = 1;
            }
        }
    }
}

// =====================================================================================
// exclusive scan of u32 (n from device), in place allowed; out[n] = total
// =====================================================================================
constexpr int SC_THREADS = 256, SC_ITEMS = 16, SC_TILE = SC_THREADS * SC_ITEMS;

__global__ void __launch_bounds__(SC_THREADS) scan_kernel(const uint32_t* in, uint32_t* out, const uint32_t* n_ptr,
                                                          uint32_t n_host, LookBack<uint32_t> lb, uint32_t epoch,
                                                          uint32_t* ticket, uint32_t* total_out) {
    __shared__ uint32_t sm[8];
    __shared__ uint32_t s_tile, s_pre;
    const uint32_t n = n_ptr ? *n_ptr : n_host;
    const uint32_t ntiles = (n + SC_TILE) / SC_TILE;      // covers index n (the total)
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) return;
    const uint64_t b = (uint64_t)tile * SC_TILE + threadIdx.x * SC_ITEMS;
    uint32_t v[SC_ITEMS];
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        v[k] = (b + k < n) ? in[b + k] : 0u;
        s += v[k];
    }
    uint32_t tot;
    uint32_t ex = block_scan_excl<uint32_t, OpAddU32>(s, tot, sm);
    if (warp_id() == 0) {
        uint32_t pre = lookback_warp<uint32_t, OpAddU32>(lb, tile, epoch, tot);
        if (lane_id() == 0) s_pre = pre;
    }
    __syncthreads();
    uint32_t run = s_pre + ex;
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        if (b + k <= n) out[b + k] = run;
        if (total_out && b + k == n) *total_out = run;
        run += v[k];
    }
}

// =====================================================================================
// emit access records
// =====================================================================================
template <int S>
__global__ void __launch_bounds__(256) emit_count_kernel(DevDb db, uint32_t* cnt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < db.n; i += gridDim.x * blockDim.x) {
        Rec r[MAX_REC];
        cnt[i] = footprint<S>(db, db.type[i], db.pw + db.poff[i], r);
    }
}

template <int S>
__global__ void __launch_bounds__(256) emit_write_kernel(DevDb db, const uint32_t* __restrict__ off, uint64_t* keys) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < db.n; i += gridDim.x * blockDim.x) {
        Rec r[MAX_REC];
        const int k = footprint<S>(db, db.type[i], db.pw + db.poff[i], r);
        uint64_t* dst = keys + off[i];
        for (int j = 0; j < k; ++j) dst[j] = make_key(r[j].item, i, j, r[j].w);
    }
}

// =====================================================================================
// rank: iterated segmented max-plus scan
//   per item group, in ts order, state (a, m) from (-1, -1):
//     write: L = max(d, m+1); (a, m) <- (L, L)
//     read : L = max(d, a+1); (a, m) <- (a, max(m, L))
//   D[idx] <- max(D[idx], L); repeat passes until nothing changes.
// Each record is a 2x3 max-plus affine map on (a, m, 1); a group head's map is the
// constant it produces from (-1, -1), so one UNsegmented scan of maps is exact.
// =====================================================================================
constexpr int NEG = -(1 << 29);
struct Xf { int aa, am, ac, ma, mm, mc; };
DEV int clneg(int x) { return x < NEG ? NEG : x; }
struct OpXf {
    static DEV Xf identity() { return Xf{0, NEG, NEG, NEG, 0, NEG}; }
    static DEV Xf combine(const Xf& F, const Xf& G) {     // F first, then G
        Xf H;
        H.aa = clneg(max(G.aa + F.aa, G.am + F.ma));
        H.am = clneg(max(G.aa + F.am, G.am + F.mm));
        H.ac = clneg(max(max(G.aa + F.ac, G.am + F.mc), G.ac));
        H.ma = clneg(max(G.ma + F.aa, G.mm + F.ma));
        H.mm = clneg(max(G.ma + F.am, G.mm + F.mm));
        H.mc = clneg(max(max(G.ma + F.ac, G.mm + F.mc), G.mc));
        return H;
    }
};
DEV Xf rec_xf(bool head, uint32_t w, int d) {
    if (head) return w ? Xf{NEG, NEG, d, NEG, NEG, d} : Xf{NEG, NEG, -1, NEG, NEG, d};
    return w ? Xf{NEG, 1, d, NEG, 1, d} : Xf{0, NEG, NEG, 1, 0, d};
}

constexpr int RK_THREADS = 256, RK_ITEMS = 8, RK_TILE = RK_THREADS * RK_ITEMS;

__global__ void __launch_bounds__(RK_THREADS) rank_kernel(const uint64_t* __restrict__ keys, const uint32_t* nrec_ptr,
                                                          uint32_t* D, LookBack<Xf> lb, uint32_t epoch0,
                                                          GridBar* bar, uint32_t* sc, uint32_t max_passes) {
    __shared__ uint64_t stage[RK_TILE];
    __shared__ Xf sm[8];
    __shared__ Xf s_pre;
    __shared__ uint64_t s_prev;
    __shared__ int s_chg;
    const uint32_t nrec = *nrec_ptr;
    const uint32_t ntiles = (nrec + RK_TILE - 1) / RK_TILE;
    const uint32_t tid = threadIdx.x;
    for (uint32_t pass = 0;; ++pass) {
        const uint32_t epoch = epoch0 + pass;
        if (blockIdx.x == 0 && tid == 0) sc[SC_CHG0 + (pass + 1) % 3] = 0;
        if (tid == 0) s_chg = 0;
        for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const uint64_t tb = (uint64_t)tile * RK_TILE;
            __syncthreads();
            for (uint32_t i = tid; i < RK_TILE; i += RK_THREADS)
                stage[i] = (tb + i < nrec) ? __ldg(&keys[tb + i]) : ~0ull;
            if (tid == 0) s_prev = tb ? __ldg(&keys[tb - 1]) : ~0ull;
            __syncthreads();
            int dv[RK_ITEMS];
            uint32_t hw = 0;                   // bit 2k: head, bit 2k+1: write
            Xf agg = OpXf::identity();
#pragma unroll
            for (int k = 0; k < RK_ITEMS; ++k) {
                const uint32_t pos = tid * RK_ITEMS + k;
                const uint64_t key = stage[pos];
                dv[k] = 0;
                if (tb + pos < nrec) {
                    const uint64_t prev = pos ? stage[pos - 1] : s_prev;
                    const bool head = (tb + pos == 0) || key_item(prev) != key_item(key);
                    const uint32_t w = key_w(key);
                    const int d = (int)__ldcg(&D[key_idx(key)]);
                    dv[k] = d;
                    hw |= (head ? 1u : 0u) << (2 * k);
                    hw |= w << (2 * k + 1);
                    agg = OpXf::combine(agg, rec_xf(head, w, d));
                }
            }
            Xf tot;
            Xf ex = block_scan_excl<Xf, OpXf>(agg, tot, sm);
            if (warp_id() == 0) {
                Xf pre = lookback_warp<Xf, OpXf>(lb, tile, epoch, tot);
                if (lane_id() == 0) s_pre = pre;
            }
            __syncthreads();
            Xf cur = OpXf::combine(s_pre, ex);
            bool chg = false;
#pragma unroll
            for (int k = 0; k < RK_ITEMS; ++k) {
                const uint32_t pos = tid * RK_ITEMS + k;
                if (tb + pos < nrec) {
                    const bool head = (hw >> (2 * k)) & 1u;
                    const uint32_t w = (hw >> (2 * k + 1)) & 1u;
                    const int d = dv[k];
                    const int a = head ? -1 : cur.ac, m = head ? -1 : cur.mc;
                    const int L = w ? max(d, m + 1) : max(d, a + 1);
                    if (L > d) {
                        const uint32_t old = atomicMax(&D[key_idx(stage[pos])], (uint32_t)L);
                        chg |= old < (uint32_t)L;
                    }
                    cur = OpXf::combine(cur, rec_xf(head, w, d));
                }
            }
            if (chg) s_chg = 1;
        }
        __syncthreads();
        if (tid == 0 && s_chg) sc[SC_CHG0 + pass % 3] = 1;
        grid_sync(bar);
        const uint32_t c = __ldcg(&sc[SC_CHG0 + pass % 3]);
        if (!c || pass + 1 >= max_passes) {
            if (blockIdx.x == 0 && tid == 0) {
                sc[SC_PASSES] = pass + 1;
                sc[SC_NOCONV] = c ? 1u : 0u;
            }
            return;
        }
    }
}

// =====================================================================================
// group by (depth, type)
// =====================================================================================
__global__ void __launch_bounds__(256) depth_reduce_kernel(const uint32_t* D, uint32_t n, uint32_t* sc) {
    uint32_t mx = 0, z = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t d = D[i];
        mx = max(mx, d);
        z += d == 0;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        z += __shfl_xor_sync(0xffffffffu, z, o);
    }
    if (lane_id() == 0) {
        atomicMax(&sc[SC_MAXD], mx);
        atomicAdd(&sc[SC_ZERO], z);
    }
}

__global__ void group_nkeys_kernel(uint32_t* sc, uint32_t T) {
    sc[SC_NKEYS] = (sc[SC_MAXD] + 1) * T;
    sc[SC_NKEYS1] = (sc[SC_MAXD] + 1) * T + 1;
}

__global__ void __launch_bounds__(256) zero_dev_kernel(uint32_t* a, const uint32_t* n_ptr) {
    const uint32_t n = *n_ptr;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = 0;
}

__global__ void __launch_bounds__(256) group_hist_kernel(const uint32_t* D, const uint8_t* type, uint32_t n, uint32_t T,
                                                         uint32_t* cnt) {
    for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < n; i0 += gridDim.x * blockDim.x) {
        const uint32_t i = i0 + threadIdx.x;
        const uint32_t key = i < n ? D[i] * T + type[i] : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        if (key != 0xFFFFFFFFu && lane_id() == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&cnt[key], __popc(peers));
    }
}

__global__ void __launch_bounds__(256) group_scatter_kernel(const uint32_t* D, const uint8_t* type, uint32_t n, uint32_t T,
                                                            uint32_t* cnt, const uint32_t* off, uint32_t* perm) {
    for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < n; i0 += gridDim.x * blockDim.x) {
        const uint32_t i = i0 + threadIdx.x;
        const uint32_t key = i < n ? D[i] * T + type[i] : 0xFFFFFFFFu;
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(peers) - 1;
        const uint32_t c = __popc(peers);
        uint32_t old = 0;
        if (key != 0xFFFFFFFFu && (int)lane_id() == leader) old = atomicSub(&cnt[key], c);
        old = __shfl_sync(0xffffffffu, old, leader);
        if (key != 0xFFFFFFFFu) perm[off[key] + old - c + __popc(peers & lanemask_lt())] = i;
    }
}

// =====================================================================================
// K-SET executor: persistent, one round per k-set (Property 1: no locks).  A run of
// narrow k-sets (<= narrow_max) executes inside CTA 0 separated by __syncthreads;
// wide k-sets are spread over the grid, separated by a grid barrier.
// =====================================================================================
template <int S>
__global__ void __launch_bounds__(256) kset_exec_kernel(DevDb db, const uint32_t* __restrict__ perm,
                                                        const uint32_t* __restrict__ off, uint32_t T, GridBar* bar,
                                                        uint32_t* sc, uint32_t narrow_max) {
    const uint32_t nk = __ldcg(&sc[SC_MAXD]) + 1;
    const uint32_t tid = threadIdx.x;
    const uint32_t gstride = gridDim.x * blockDim.x;
    uint32_t k = 0;
    while (k < nk) {
        uint32_t lo = __ldcg(&off[k * T]), hi = __ldcg(&off[(k + 1) * T]);
        if (hi - lo <= narrow_max) {
            if (blockIdx.x == 0) {
                while (true) {
                    for (uint32_t j = lo + tid; j < hi; j += blockDim.x) exec_txn<S>(db, __ldg(&perm[j]));
                    __syncthreads();
                    ++k;
                    if (k >= nk) break;
                    lo = hi;
                    hi = __ldcg(&off[(k + 1) * T]);
                    if (hi - lo > narrow_max) break;
                }
                if (tid == 0) sc[SC_KNEXT] = k;
            }
            grid_sync(bar);
            k = __ldcg(&sc[SC_KNEXT]);
            grid_sync(bar);                    // everyone has read KNEXT before it can change
        } else {
            for (uint32_t j = lo + blockIdx.x * blockDim.x + tid; j < hi; j += gstride) exec_txn<S>(db, __ldg(&perm[j]));
            grid_sync(bar);
            ++k;
        }
    }
}

// =====================================================================================
// PART
// =====================================================================================
template <int S>
__global__ void __launch_bounds__(256) frag_count_kernel(DevDb db, uint32_t* cnt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < db.n; i += gridDim.x * blockDim.x)
        cnt[i] = fragments<S>(db, i, nullptr);
}
template <int S>
__global__ void __launch_bounds__(256) frag_emit_kernel(DevDb db, const uint32_t* off, uint64_t* keys) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < db.n; i += gridDim.x * blockDim.x)
        fragments<S>(db, i, keys + off[i]);
}
__global__ void __launch_bounds__(256) part_bounds_kernel(const uint64_t* frags, const uint32_t* nf_ptr, uint32_t nparts,
                                                          uint32_t* part_off) {
    const uint32_t nf = *nf_ptr;
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
    if (nf == 0) {
        for (uint32_t p = g; p <= nparts; p += gs) part_off[p] = 0;
        return;
    }
    for (uint32_t k = g; k <= nf; k += gs) {
        const int64_t pid = k < nf ? (int64_t)(frags[k] >> 32) : (int64_t)nparts;
        const int64_t prev = k ? (int64_t)(frags[k - 1] >> 32) : -1;
        for (int64_t p = prev + 1; p <= pid; ++p) part_off[p] = k;
    }
}
template <int S>
__global__ void __launch_bounds__(128) part_exec_kernel(DevDb db, const uint64_t* __restrict__ frags,
                                                        const uint32_t* __restrict__ part_off, uint32_t nparts, uint32_t* sc) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nparts) return;
    const uint32_t lo = part_off[p], hi = part_off[p + 1];
    for (uint32_t j = lo; j < hi; ++j) exec_frag<S>(db, __ldg(&frags[j]));
    if (hi - lo) atomicMax(&sc[SC_MAXCHAIN], hi - lo);
}

// =====================================================================================
// TPL
// =====================================================================================
struct Pair { uint32_t h, w; };
struct OpPair {
    static DEV Pair identity() { return Pair{0u, 0u}; }
    static DEV Pair combine(const Pair& a, const Pair& b) { return Pair{max(a.h, b.h), max(a.w, b.w)}; }
};

// Counter-lock keys (DESIGN.md R-S5): in group order, a write's key is its position in
// the group; a read's key is the position of the first record of its run of reads.
// A record may enter when lock >= key; it releases +1 after its transaction.
__global__ void __launch_bounds__(RK_THREADS) tpl_keys_kernel(const uint64_t* __restrict__ keys, const uint32_t* nrec_ptr,
                                                              const uint32_t* __restrict__ rec_off, uint32_t* lkey,
                                                              uint32_t* lock, LookBack<Pair> lb, uint32_t epoch,
                                                              uint32_t* ticket) {
    __shared__ Pair sm[8];
    __shared__ Pair s_pre;
    __shared__ uint32_t s_tile;
    const uint32_t nrec = *nrec_ptr;
    const uint32_t ntiles = (nrec + RK_TILE - 1) / RK_TILE;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) return;
    const uint64_t b = (uint64_t)tile * RK_TILE + threadIdx.x * RK_ITEMS;
    uint64_t kk[RK_ITEMS];
    Pair agg = OpPair::identity();
    uint32_t hflags = 0;
#pragma unroll
    for (int k = 0; k < RK_ITEMS; ++k) {
        const uint64_t i = b + k;
        if (i < nrec) {
            kk[k] = __ldg(&keys[i]);
            const bool head = i == 0 || key_item(__ldg(&keys[i - 1])) != key_item(kk[k]);
            hflags |= (head ? 1u : 0u) << k;
            Pair e{head ? (uint32_t)i + 1 : 0u, key_w(kk[k]) ? (uint32_t)i + 1 : 0u};
            agg = OpPair::combine(agg, e);
        } else {
            kk[k] = 0;
        }
    }
    Pair tot;
    Pair ex = block_scan_excl<Pair, OpPair>(agg, tot, sm);
    if (warp_id() == 0) {
        Pair pre = lookback_warp<Pair, OpPair>(lb, tile, epoch, tot);
        if (lane_id() == 0) s_pre = pre;
    }
    __syncthreads();
    Pair cur = OpPair::combine(s_pre, ex);
#pragma unroll
    for (int k = 0; k < RK_ITEMS; ++k) {
        const uint64_t i = b + k;
        if (i < nrec) {
            const bool head = (hflags >> k) & 1u;
            const uint32_t lw_ex = cur.w;                  // index+1 of last write before i
            const uint32_t w = key_w(kk[k]);
            cur = OpPair::combine(cur, Pair{head ? (uint32_t)i + 1 : 0u, w ? (uint32_t)i + 1 : 0u});
            const uint32_t H = cur.h - 1;                  // group head index
            uint32_t key;
            if (w) key = (uint32_t)i - H;
            else key = (lw_ex > H) ? lw_ex - H : 0u;
            lkey[rec_off[key_idx(kk[k])] + key_j(kk[k])] = key;
            if (head) lock[key_item(kk[k])] = 0;
        }
    }
}

constexpr uint32_t SPIN_LIMIT = 1u << 26;

template <int S>
__global__ void __launch_bounds__(128) tpl_exec_kernel(DevDb db, const uint32_t* __restrict__ rec_off,
                                                       const uint32_t* __restrict__ lkey, uint32_t* lock, uint32_t* sc) {
    __shared__ uint32_t s_base;
    if (threadIdx.x == 0) s_base = atomicAdd(&sc[SC_TICKET], blockDim.x);   // ts-ordered dispatch
    __syncthreads();
    const uint32_t idx = s_base + threadIdx.x;
    if (idx >= db.n) return;
    Rec r[MAX_REC];
    const int k = footprint<S>(db, db.type[idx], db.pw + db.poff[idx], r);
    const uint32_t ro = rec_off[idx];
    // growing phase: enter every lock in turn (keys order conflicting records by ts)
    for (int j = 0; j < k; ++j) {
        const uint32_t key = __ldg(&lkey[ro + j]);
        uint32_t* lw = &lock[r[j].item];
        uint32_t spins = 0;
        while (ld_acquire(lw) < key) {
            if (++spins > SPIN_LIMIT) { atomicExch(&sc[SC_DEADLOCK], 1u); break; }
            if (spins > 64) __nanosleep(64);
        }
    }
    exec_txn<S>(db, idx);
    __threadfence();
    // shrinking phase
    for (int j = 0; j < k; ++j) atomicAdd(&lock[r[j].item], 1u);
}

}  // namespace gputx
