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
    SC_KNEXT, SC_TICKET, SC_DEADLOCK, SC_MAXCHAIN, SC_NKEYS, SC_NKEYS1, SC_COMMITTED, SC_NOCONV, SC_XTOTAL,
    SC_RRSPLIT,       // 19: root-local rank fell back to the grid scan (a root too large for one warp)
    SC_COUNT = 48      // (slots 20-31: SC_INS0, SC_DEST0; 32: SC_CROSS; 33: SC_NOCLUSTER; ... 40: SC_OUTBYTES)
};
enum { E_TYPE = 1, E_UNREG = 2, E_LEN = 3, E_RANGE = 4, E_OFF = 5, E_TS = 6, E_OWNER = 7, E_WORDS = 8, E_POISON = 9 };
constexpr int SC_INS0 = 20;       // [20, 24): insert rows per table (ingest)
constexpr int SC_CROSS = 32;      // c: transactions with fragments in > 1 PART partition
constexpr int SC_NOCLUSTER = 33;  // K-SET: launched without the requested cluster shape (counter hand-offs used)
constexpr int SC_ERRPK = 34;      // [34, 36): u64 (first bad idx << 8 | its code); all-ones = none
constexpr int SC_SPARSE = 36;     // TPC-B ingest: transactions without a history row (withdrawals, peers')
constexpr int SC_P2P = 37;        // [37, 39): peer exchange: records received, overflow bits
constexpr int SC_OUTBYTES = 40;   // GPUTX_FLAG_PACKED_OUT: bytes of the bulk's packed output records
constexpr int SC_NTXN = 41;       // transactions in the submitted bulk (device copy of n, ingest)
constexpr int SC_NCHAIN = 42;     // spine-streaming rank: chains

// TM-1 sub_nbr hash (shared host/device)
__host__ __device__ inline uint64_t nbr_hash(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
    return x;
}

// The first bad transaction and ITS error code, packed (idx << 8 | code) in one 64-bit
// word so that one atomicMin keeps them together (separate min/max words paired
// the lowest index with another transaction's code); SC_ERR flags "some error".
DEV void report_err(uint32_t* sc, uint32_t code, uint32_t idx) {
    atomicMin(reinterpret_cast<unsigned long long*>(&sc[SC_ERRPK]), ((unsigned long long)idx << 8) | code);
    atomicOr(&sc[SC_ERR], 1u);
}

// =====================================================================================
// ingest: validate in place, resolve static lookups, count insert rows
// =====================================================================================
// A device-resident bulk's parameter words, copied with the count read on the device
// (param_off[n]) -- no host round trip to size the copy; more than max_words -> E_WORDS
__global__ void __launch_bounds__(256) copy_pw_kernel(const uint32_t* __restrict__ src, const uint32_t* nw_ptr,
                                                      uint32_t* dst, uint32_t max_words, uint32_t* sc) {
    uint32_t nw = __ldg(nw_ptr);
    if (nw > max_words) {
        if (blockIdx.x == 0 && threadIdx.x == 0) report_err(sc, E_WORDS, 0);
        nw = max_words;
    }
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    uint32_t done = 0;
    if (!((uintptr_t)src & 15u)) {
        // 16-B vectors, four in flight per thread (one 4-B word per thread and iteration was
        // latency-bound: ~100 us for TPC-B's 64 MB of words)
        const uint32_t n4 = nw / 4;
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint4* d4 = reinterpret_cast<uint4*>(dst);                  // (cudaMalloc'ed)
        for (uint32_t i = g; i < n4; i += 4 * stride) {
            uint4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + u * stride < n4) v[u] = __ldg(&s4[i + u * stride]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + u * stride < n4) d4[i + u * stride] = v[u];
        }
        done = n4 * 4;
    }
    for (uint32_t i = done + g; i < nw; i += stride) dst[i] = __ldg(&src[i]);
}

// nw_ptr (optional): the word count on the device; n_words is then its upper bound
template <int S>
__global__ void __launch_bounds__(256) ingest_kernel(DevDb db, uint32_t* pw, uint32_t n_words, const uint32_t* nw_ptr,
                                                     uint32_t type_mask, uint32_t* ins_cnt, uint32_t ins_stride,
                                                     uint32_t* sc, uint8_t* xflag, uint32_t* out_size,
                                                     uint32_t* rec_cnt) {
    const uint32_t n = db.n;
    if (blockIdx.x == 0 && threadIdx.x == 0) sc[SC_NTXN] = n;
    if (db.poison && __ldcg(db.poison)) {             // an earlier bulk of this run failed
        if (blockIdx.x == 0 && threadIdx.x == 0) report_err(sc, E_POISON, 0);
        return;
    }
    if (nw_ptr) n_words = min(__ldg(nw_ptr), n_words);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        // an invalid transaction keeps no records and no output bytes (a deferred verdict
        // runs the rest of the bulk's generation on the valid ones)
        if (out_size) out_size[i] = 0;
        if (rec_cnt) rec_cnt[i] = 0;
        const uint32_t t = db.type[i];
        // sharded: a peer's transaction (NOT_HOME) only runs its fragments on this shard
        const bool home = !db.src || db.src[i] != NOT_HOME;
        if (db.ts && i + 1 < n && db.ts[i] >= db.ts[i + 1]) { report_err(sc, E_TS, i); continue; }
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
            // WITHDRAW: a local account (its rollback must not span partitions / shards) and a
            // positive amount
            if (t == 1 && (p[0] / A != p[2] || (int32_t)p[3] <= 0)) { report_err(sc, E_RANGE, i); continue; }
        } else if (S == S_MICRO) {
            if (len != 1) { report_err(sc, E_LEN, i); continue; }
            if (p[0] >= db.dims[0]) { report_err(sc, E_RANGE, i); continue; }
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
                if (!abort && home) {
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
                if (p[4] != 2 && home) ins_cnt[T_HIST * ins_stride + i] = 1;
            }
        }
        if (out_size) out_size[i] = out_bytes<S>(t, p);            // packed outputs (scanned at submit)
        if (rec_cnt) {                                                // access records (emit's count pass)
            Rec rr[MAX_REC];
            rec_cnt[i] = footprint_local<S>(db, t, p, rr);
        }
        if (S == S_TPCB) {                                           // history rows (deposits) via ins_off
            ins_cnt[i] = (home && t == 0) ? 1u : 0u;
            if (!(home && t == 0)) atomicAdd(&sc[SC_SPARSE], 1u);       // some row is not at its idx
        }
        if (db.nshards > 1) {
            // the home root must be this shard's iff the transaction was submitted here
            const uint64_t root = S == S_TPCB ? p[2] : S == S_TPCC ? p[0] : (uint64_t)(p[0] ? p[0] - 1 : db.root_lo);
            if (home != root_local(db, root)) { report_err(sc, E_OWNER, i); continue; }
            xflag[i] = (!home || fragments_local<S>(db, i, nullptr) != fragments<S>(db, i, nullptr)) ? 1 : 0;
        }
    }
}

// =====================================================================================
// exclusive scan of u32 (n from device), in place allowed; out[n] = total
// =====================================================================================
constexpr int SC_THREADS = 256, SC_ITEMS = 16, SC_TILE = SC_THREADS * SC_ITEMS;

// a thread's 16 consecutive u32 (a run starts at a multiple of 16 elements; the caller checks
// the array's 16-B alignment) as four 16-B accesses
__device__ __forceinline__ void load16(const uint32_t* p, uint32_t (&v)[SC_ITEMS]) {
#pragma unroll
    for (int q = 0; q < SC_ITEMS / 4; ++q) {
        const uint4 x = reinterpret_cast<const uint4*>(p)[q];
        v[4 * q] = x.x; v[4 * q + 1] = x.y; v[4 * q + 2] = x.z; v[4 * q + 3] = x.w;
    }
}
__device__ __forceinline__ void store16(uint32_t* p, const uint32_t (&v)[SC_ITEMS]) {
#pragma unroll
    for (int q = 0; q < SC_ITEMS / 4; ++q)
        reinterpret_cast<uint4*>(p)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
}

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
    // the thread's 16 values as 4 x 16-B accesses (arrays at a 16-B boundary; the per-table
    // insert offsets of TPC-C sit at (n + 1)-word strides and take the scalar path)
    const bool full = b + SC_ITEMS <= n && !(((uintptr_t)in | (uintptr_t)out) & 15);
    if (full) {
        load16(in + b, v);
    } else {
#pragma unroll
        for (int k = 0; k < SC_ITEMS; ++k) v[k] = (b + k < n) ? in[b + k] : 0u;
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) s += v[k];
    uint32_t tot;
    uint32_t ex = block_scan_excl<uint32_t, OpAddU32>(s, tot, sm);
    if (warp_id() == 0) {
        uint32_t pre = lookback_warp<uint32_t, OpAddU32>(lb, tile, epoch, tot);
        if (lane_id() == 0) s_pre = pre;
    }
    __syncthreads();
    uint32_t run = s_pre + ex;
    if (full) {
#pragma unroll
        for (int k = 0; k < SC_ITEMS; ++k) {
            const uint32_t x = v[k];
            v[k] = run;
            run += x;
        }
        store16(out + b, v);
        return;
    }
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        if (b + k <= n) out[b + k] = run;
        if (total_out && b + k == n) *total_out = run;
        run += v[k];
    }
}

// scan_kernel over two u32 arrays at once (packed-output sizes and access-record counts,
// both per transaction, both computed at ingest): outX[n] / outY[n] = totals
__global__ void __launch_bounds__(SC_THREADS) scan2_kernel(const uint32_t* inX, const uint32_t* inY, uint32_t* outX,
                                                           uint32_t* outY, uint32_t n, LookBack<uint2> lb,
                                                           uint32_t epoch, uint32_t* ticket, uint32_t* totX,
                                                           uint32_t* totY) {
    __shared__ uint2 sm[8];
    __shared__ uint32_t s_tile;
    __shared__ uint2 s_pre;
    const uint32_t ntiles = (n + SC_TILE) / SC_TILE;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) return;
    const uint64_t b = (uint64_t)tile * SC_TILE + threadIdx.x * SC_ITEMS;
    uint32_t vx[SC_ITEMS], vy[SC_ITEMS];
    const bool full = b + SC_ITEMS <= n && !(((uintptr_t)inX | (uintptr_t)inY | (uintptr_t)outX | (uintptr_t)outY) & 15);
    if (full) {
        load16(inX + b, vx);
        load16(inY + b, vy);
    } else {
#pragma unroll
        for (int k = 0; k < SC_ITEMS; ++k) {
            vx[k] = b + k < n ? inX[b + k] : 0u;
            vy[k] = b + k < n ? inY[b + k] : 0u;
        }
    }
    uint2 sum = make_uint2(0u, 0u);
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) sum = OpAddU2::combine(sum, make_uint2(vx[k], vy[k]));
    uint2 tot;
    uint2 ex = block_scan_excl<uint2, OpAddU2>(sum, tot, sm);
    if (warp_id() == 0) {
        uint2 pre = lookback_warp<uint2, OpAddU2>(lb, tile, epoch, tot);
        if (lane_id() == 0) s_pre = pre;
    }
    __syncthreads();
    uint2 run = OpAddU2::combine(s_pre, ex);
    if (full) {
#pragma unroll
        for (int k = 0; k < SC_ITEMS; ++k) {
            const uint32_t x = vx[k], y = vy[k];
            vx[k] = run.x;
            vy[k] = run.y;
            run.x += x;
            run.y += y;
        }
        store16(outX + b, vx);
        store16(outY + b, vy);
        return;
    }
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        if (b + k <= n) { outX[b + k] = run.x; outY[b + k] = run.y; }
        if (b + k == n) { *totX = run.x; *totY = run.y; }
        run = OpAddU2::combine(run, make_uint2(vx[k], vy[k]));
    }
}

// =====================================================================================
// emit access records
// =====================================================================================
template <int S>
__global__ void __launch_bounds__(256) emit_count_kernel(DevDb db, uint32_t* cnt) {
    const bool failed = bulk_failed(db);
    if (failed && db.poison && blockIdx.x == 0 && threadIdx.x == 0) *db.poison = 1u;   // stop the run
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < db.n; i += gridDim.x * blockDim.x) {
        Rec r[MAX_REC];
        cnt[i] = failed ? 0 : footprint_local<S>(db, db.type[i], db.pw + db.poff[i], r);
    }
}

template <int S>
__global__ void __launch_bounds__(256) emit_write_kernel(DevDb db, const uint32_t* __restrict__ off, uint64_t* keys) {
    // a failed bulk (guarded modes): only the transactions that kept records are valid ones
    const bool failed = bulk_failed(db);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < db.n; i += gridDim.x * blockDim.x) {
        if (failed && off[i + 1] == off[i]) continue;
        Rec r[MAX_REC];
        const int k = footprint_local<S>(db, db.type[i], db.pw + db.poff[i], r);
        uint64_t* dst = keys + off[i];
        for (int j = 0; j < k; ++j) dst[j] = make_key(r[j].item, db.idx_base + i, j, r[j].w);
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
// Record maps on the state (a, m) = (max depth of the last writer and the adds since it,
// max depth of the last writer and the reads since it); mode 0 read, 1 write, 2 add
// (ADD rule: adds of one item do not conflict with each other).  Without adds a is
// the last writer's depth, m the max since it, and these are the R/W maps.
//   read : a' = a,                 m' = max(m, a+1, d)      level max(d, a+1)
//   add  : a' = max(a, m+1, d),    m' = m                   level max(d, m+1)
//   write: a' = m' = max(a+1, m+1, d)                       level max(d, max(a, m)+1)
// A group head starts from (-1, -1).
DEV Xf rec_xf(bool head, uint32_t mode, int d) {
    if (head) return mode == 0 ? Xf{NEG, NEG, -1, NEG, NEG, d}
                   : mode == 2 ? Xf{NEG, NEG, d, NEG, NEG, -1} : Xf{NEG, NEG, d, NEG, NEG, d};
    return mode == 0 ? Xf{0, NEG, NEG, 1, 0, d} : mode == 2 ? Xf{0, 1, d, NEG, 0, NEG} : Xf{1, 1, d, 1, 1, d};
}
DEV int rec_level(bool head, uint32_t mode, int d, const Xf& cur) {
    const int a = head ? -1 : cur.ac, m = head ? -1 : cur.mc;
    return mode == 0 ? max(d, a + 1) : mode == 2 ? max(d, m + 1) : max(d, max(a, m) + 1);
}
// per-record bits of a lane's RK_ITEMS records: bit 3k head, bits 3k+1..3k+2 mode,
// bit 24+k valid
DEV uint32_t rk_bits(bool head, uint32_t mode, int k) {
    return ((head ? 1u : 0u) | (mode << 1)) << (3 * k) | 1u << (24 + k);
}
DEV bool rk_valid(uint32_t hw, int k) { return (hw >> (24 + k)) & 1u; }
DEV bool rk_head(uint32_t hw, int k) { return (hw >> (3 * k)) & 1u; }
DEV uint32_t rk_mode(uint32_t hw, int k) { return (hw >> (3 * k + 1)) & 3u; }

constexpr int RK_THREADS = 256, RK_ITEMS = 8, RK_TILE = RK_THREADS * RK_ITEMS;
constexpr int RK_WT = 32 * RK_ITEMS;      // records per warp-tile (the rank pass's unit of work)
constexpr uint32_t RK_LOCAL_DEFAULT = 4;   // in-tile Gauss-Seidel sweeps per pass (default)

// One pass over the sorted records = reduce, then scan:
//   A. every CTA owns a contiguous range of tiles; it composes the maps of its records
//      (with the current D) into one aggregate and publishes it;
//   B. grid barrier;
//   C. each CTA composes the aggregates of the CTAs before it -> the state entering
//      its range (no look-back chain);
//   D. it sweeps its tiles in order: block scan of the maps, L per record, atomicMax
//      into D; a tile that raised something is re-swept with its own new values (up to
//      local_max times; items of one root key are adjacent, so chains close on chip).
// Every L computed is a lower bound of the true depth, so chaotic/in-tile updates
// reach the same fixpoint; a pass in which nothing is raised proves it.
struct RkTile {
    uint32_t hw;       // bit 2k: head, bit 2k+1: write, bit 16+k: valid
};

DEV uint32_t rk_load(const uint64_t* __restrict__ keys, uint32_t nrec, uint32_t tile, uint64_t* stage,
                     uint64_t* s_prev) {
    const uint64_t tb = (uint64_t)tile * RK_TILE;
    const uint32_t tid = threadIdx.x;
    __syncthreads();
    for (uint32_t i = tid; i < RK_TILE; i += RK_THREADS) stage[i] = (tb + i < nrec) ? __ldg(&keys[tb + i]) : ~0ull;
    if (tid == 0) *s_prev = tb ? __ldg(&keys[tb - 1]) : ~0ull;
    __syncthreads();
    uint32_t hw = 0;
#pragma unroll
    for (int k = 0; k < RK_ITEMS; ++k) {
        const uint32_t pos = tid * RK_ITEMS + k;
        if (tb + pos < nrec) {
            const uint64_t key = stage[pos];
            const uint64_t prev = pos ? stage[pos - 1] : *s_prev;
            const bool head = (tb + pos == 0) || key_item(prev) != key_item(key);
            hw |= rk_bits(head, key_mode(key), k);
        }
    }
    return hw;
}

// Dirty-tile worklist across the passes of one rank launch.  A tile's map aggregate
// depends only on the depths of its records' transactions, and its sweep only on those
// and its incoming state.  So a tile is re-swept only if one of its transactions was
// raised since its last sweep (`dirty` bit, set by the raiser) or its incoming state
// changed (`carD`); a clean tile reuses its memoised aggregate `aggA`.  To mark, the
// raiser needs the tiles of all records of a transaction: `recpos` (sorted position of
// record rec_off[t] + j), built in the prologue.
constexpr uint32_t RANK_TRACE_SLOTS = 8 * 1024;      // 8 timestamps per pass (diagnostics)
struct RkMemo {
    Xf* aggA;
    Xf* carD;
    uint32_t* dirty;
    uint32_t* recpos;
    const uint32_t* rec_off;
};

DEV bool xf_eq(const Xf& a, const Xf& b) {
    return a.aa == b.aa && a.am == b.am && a.ac == b.ac && a.ma == b.ma && a.mm == b.mm && a.mc == b.mc;
}

DEV void rk_gather(const uint64_t* stage, uint32_t hw, const uint32_t* D, int* dv) {
#pragma unroll
    for (int k = 0; k < RK_ITEMS; ++k)
        dv[k] = rk_valid(hw, k) ? (int)__ldcg(&D[key_idx(stage[threadIdx.x * RK_ITEMS + k])]) : 0;
}

DEV Xf rk_compose(uint32_t hw, const int* dv) {
    Xf agg = OpXf::identity();
#pragma unroll
    for (int k = 0; k < RK_ITEMS; ++k)
        if (rk_valid(hw, k)) agg = OpXf::combine(agg, rec_xf(rk_head(hw, k), rk_mode(hw, k), dv[k]));
    return agg;
}

DEV bool rk_is_dirty(const uint32_t* dirty, uint32_t tile) {
    return (__ldcg(&dirty[tile >> 5]) >> (tile & 31)) & 1u;
}

// transaction t was raised by a thread sweeping tile `self`: mark the other tiles holding
// its records (`self` is swept again until it raises nothing)
DEV void rk_mark(const RkMemo& memo, uint32_t t, uint32_t self) {
    __threadfence();                          // the raise is visible before the mark
    const uint32_t r0 = __ldg(&memo.rec_off[t]), r1 = __ldg(&memo.rec_off[t + 1]);
    for (uint32_t r = r0; r < r1; ++r) {
        const uint32_t tl = __ldcg(&memo.recpos[r]) / RK_WT;
        if (tl != self && !rk_is_dirty(memo.dirty, tl)) atomicOr(&memo.dirty[tl >> 5], 1u << (tl & 31));
    }
}

// One warp-tile (RK_WT records) into this warp's stage; returns the head/write/valid bits
// of the lane's RK_ITEMS records.
DEV uint32_t rk_wload(const uint64_t* __restrict__ keys, uint32_t nrec, uint32_t wt, uint64_t* stage) {
    const uint64_t tb = (uint64_t)wt * RK_WT;
    const uint32_t lane = lane_id();
    __syncwarp();
#pragma unroll
    for (int k = 0; k < RK_ITEMS; ++k) {
        const uint32_t i = k * 32 + lane;            // coalesced
        stage[i] = (tb + i < nrec) ? __ldg(&keys[tb + i]) : ~0ull;
    }
    const uint64_t prev = tb ? __ldg(&keys[tb - 1]) : ~0ull;
    __syncwarp();
    uint32_t hw = 0;
#pragma unroll
    for (int k = 0; k < RK_ITEMS; ++k) {
        const uint32_t pos = lane * RK_ITEMS + k;
        if (tb + pos < nrec) {
            const uint64_t key = stage[pos];
            const uint64_t pk = pos ? stage[pos - 1] : prev;
            const bool head = (tb + pos == 0) || key_item(pk) != key_item(key);
            hw |= rk_bits(head, key_mode(key), k);
        }
    }
    return hw;
}

DEV void rk_wgather(const uint64_t* stage, uint32_t hw, const uint32_t* D, int* dv) {
    const uint32_t lane = lane_id();
#pragma unroll
    for (int k = 0; k < RK_ITEMS; ++k)
        dv[k] = rk_valid(hw, k) ? (int)__ldcg(&D[key_idx(stage[lane * RK_ITEMS + k])]) : 0;
}

// exclusive warp scan of maps; total to every lane
DEV Xf rk_wscan(Xf x, Xf& total) {
    const Xf inc = warp_scan_incl<Xf, OpXf>(x);
    total = shfl_t(inc, 31);
    Xf ex = shfl_up_t(inc, 1);
    if (lane_id() == 0) ex = OpXf::identity();
    return ex;
}

// Warp-granular passes: every warp owns a contiguous range of warp-tiles and walks it as
// an independent chain (warp shuffles only, no block barrier in the tile loop), so an SM
// has 16 independent load/scan/atomic chains in flight instead of 2.
__device__ __forceinline__ void rank_generic(const uint64_t* __restrict__ keys, const uint32_t* nrec_ptr, uint32_t* D,
                                             LookBack<Xf> lb, uint32_t epoch0, GridBar* bar, uint32_t* sc,
                                             uint32_t max_passes, uint32_t local_max, uint32_t use_dirty, RkMemo memo,
                                             uint64_t* trace) {
    // trace (diagnostics): per pass p, [8p] pass start (CTA 0), [8p+1] last CTA done with A,
    // [8p+2] CTA 0 past barrier 1, [8p+3] last CTA done with D, [8p+4] CTA 0 past barrier 2,
    // [8p+5] warp-tiles swept, [8p+6] sweeps
    auto tmax = [&](uint32_t pass, uint32_t slot) {
        if (trace && threadIdx.x == 0 && pass < RANK_TRACE_SLOTS / 8)
            atomicMax(reinterpret_cast<unsigned long long*>(&trace[8 * pass + slot]), (unsigned long long)globaltimer_ns());
    };
    constexpr uint32_t NW = RK_THREADS / 32;
    __shared__ uint64_t stage_all[NW * RK_WT];
    __shared__ Xf sm[8];
    __shared__ Xf wagg[NW];
    __shared__ int s_chg;
    __shared__ uint32_t s_swept, s_sweeps;
    Xf* cta_agg = lb.agg;                  // one aggregate per CTA
    const uint32_t nrec = *nrec_ptr;
    const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
    uint64_t* stage = stage_all + wid * RK_WT;
    const uint32_t nwt = (nrec + RK_WT - 1) / RK_WT;
    const uint32_t per = (nwt + gridDim.x * NW - 1) / (gridDim.x * NW);
    const uint32_t gw = blockIdx.x * NW + wid;
    const uint32_t w0 = min(nwt, gw * per), w1 = min(nwt, w0 + per);
    // prologue (complete before the first marks, which come after pass 0's barriers)
    for (uint64_t p = (uint64_t)w0 * RK_WT + lane; p < min((uint64_t)w1 * RK_WT, (uint64_t)nrec); p += 32) {
        const uint64_t k = __ldg(&keys[p]);
        memo.recpos[__ldg(&memo.rec_off[key_idx(k)]) + key_j(k)] = (uint32_t)p;
    }
    for (uint32_t pass = 0;; ++pass) {
        const bool all = pass < 2 || !use_dirty;   // passes 0 and 1 sweep everything; marks start in pass 1
        if (blockIdx.x == 0 && tid == 0) sc[SC_CHG0 + (pass + 1) % 3] = 0;
        if (blockIdx.x == 0) tmax(pass, 0);
        if (tid == 0) { s_chg = 0; s_swept = 0; s_sweeps = 0; }
        // A: aggregate of this warp's range, then of the CTA's
        Xf mine = OpXf::identity();
        for (uint32_t wt = w0; wt < w1; ++wt) {
            Xf tot;
            // the bit can be set concurrently by other warps: lane 0 reads it for the warp
            const uint32_t dirty = all ? 1u : __shfl_sync(0xffffffffu, lane == 0 ? (uint32_t)rk_is_dirty(memo.dirty, wt) : 0u, 0);
            if (!dirty) {
                tot = memo.aggA[wt];
            } else {
                const uint32_t hw = rk_wload(keys, nrec, wt, stage);
                int dv[RK_ITEMS];
                rk_wgather(stage, hw, D, dv);
                rk_wscan(rk_compose(hw, dv), tot);
            }
            mine = OpXf::combine(mine, tot);
        }
        if (lane == 0) wagg[wid] = mine;
        __syncthreads();
        if (tid == 0) {
            Xf c = OpXf::identity();
            for (uint32_t j = 0; j < NW; ++j) c = OpXf::combine(c, wagg[j]);
            lb_store(&cta_agg[blockIdx.x], c);
        }
        tmax(pass, 1);
        grid_sync(bar);
        if (blockIdx.x == 0) tmax(pass, 2);
        // C: state entering this warp's range = the CTA aggregates before it, then the
        // warp aggregates of this CTA before it
        Xf carry = OpXf::identity();
        for (uint32_t c0 = 0; c0 < blockIdx.x; c0 += RK_THREADS) {
            const Xf x = (c0 + tid < blockIdx.x) ? lb_load(&cta_agg[c0 + tid]) : OpXf::identity();
            Xf tot;
            block_scan_excl<Xf, OpXf>(x, tot, sm);
            carry = OpXf::combine(carry, tot);
        }
        for (uint32_t j = 0; j < wid; ++j) carry = OpXf::combine(carry, wagg[j]);
        // D: sweep the warp-tiles in order
        uint32_t swept = 0, sweeps = 0;
        bool wchg = false;
        for (uint32_t wt = w0; wt < w1; ++wt) {
            const uint32_t dirty = all ? 1u : __shfl_sync(0xffffffffu, lane == 0 ? (uint32_t)rk_is_dirty(memo.dirty, wt) : 0u, 0);
            if (!dirty && xf_eq(carry, memo.carD[wt])) {           // same inputs and state: settled
                carry = OpXf::combine(carry, memo.aggA[wt]);
                continue;
            }
            if (lane == 0) {
                if (dirty) atomicAnd(&memo.dirty[wt >> 5], ~(1u << (wt & 31)));
                __threadfence();           // clear before gathering: a later raise re-marks
            }
            __syncwarp();
            const uint32_t hw = rk_wload(keys, nrec, wt, stage);
            ++swept;
            Xf last_tot = OpXf::identity();
            bool settled = false;
            uint32_t raised = 0;           // bit k: record k's transaction raised in this tile
            for (uint32_t it = 0; it < local_max; ++it) {
                ++sweeps;
                int dv[RK_ITEMS];
                rk_wgather(stage, hw, D, dv);
                Xf tot;
                const Xf ex = rk_wscan(rk_compose(hw, dv), tot);
                last_tot = tot;
                Xf cur = OpXf::combine(carry, ex);
                int L[RK_ITEMS];
#pragma unroll
                for (int k = 0; k < RK_ITEMS; ++k) {
                    L[k] = 0;
                    if (rk_valid(hw, k)) {
                        const bool head = rk_head(hw, k);
                        const uint32_t mode = rk_mode(hw, k);
                        L[k] = rec_level(head, mode, dv[k], cur);
                        cur = OpXf::combine(cur, rec_xf(head, mode, dv[k]));
                    }
                }
                // raises as fire-and-forget reductions (RED.MAX): a raise is detected from the
                // gathered value (L > dv) instead of the atomic's return, so the sweep does not
                // wait a round trip per tile; a raise another warp made meanwhile at most costs
                // one more sweep (the next gather sees it: every value is a lower bound)
                bool chg = false;
#pragma unroll
                for (int k = 0; k < RK_ITEMS; ++k)
                    if (L[k] > dv[k]) {
                        atomicMax(&D[key_idx(stage[lane * RK_ITEMS + k])], (uint32_t)L[k]);
                        chg = true;
                        raised |= 1u << k;
                    }
                if (!__any_sync(0xffffffffu, chg)) {
                    // this sweep raised nothing: its aggregate and incoming state are the
                    // tile's fixpoint until a record's transaction is raised
                    if (lane == 0) { memo.carD[wt] = carry; memo.aggA[wt] = tot; }
                    settled = true;
                    break;
                }
                wchg = true;
            }
            if (!settled && lane == 0) {   // sweep cap hit: sweep again next pass
                memo.aggA[wt] = last_tot;
                atomicOr(&memo.dirty[wt >> 5], 1u << (wt & 31));
            }
            if (use_dirty && pass >= 1 && raised) {     // mark the other tiles of the raised transactions
                __threadfence();           // the raises are visible before the marks
#pragma unroll
                for (int k = 0; k < RK_ITEMS; ++k)
                    if ((raised >> k) & 1u) rk_mark(memo, key_idx(stage[lane * RK_ITEMS + k]), wt);
            }
            carry = OpXf::combine(carry, last_tot);
        }
        if (lane == 0 && wchg) s_chg = 1;
        if (trace && lane == 0) { atomicAdd(&s_swept, swept); atomicAdd(&s_sweeps, sweeps); }
        __syncthreads();
        if (tid == 0 && s_chg) sc[SC_CHG0 + pass % 3] = 1;
        if (trace && tid == 0 && pass < RANK_TRACE_SLOTS / 8) {
            atomicAdd(reinterpret_cast<unsigned long long*>(&trace[8 * pass + 5]), (unsigned long long)s_swept);
            atomicAdd(reinterpret_cast<unsigned long long*>(&trace[8 * pass + 6]), (unsigned long long)s_sweeps);
        }
        tmax(pass, 3);
        grid_sync(bar);
        if (blockIdx.x == 0) tmax(pass, 4);
        const uint32_t c = __ldcg(&sc[SC_CHG0 + pass % 3]);
        if (!c || pass + 1 >= max_passes || __ldcg(&bar->dead)) {
            if (blockIdx.x == 0 && tid == 0 && __ldcg(&bar->dead)) sc[SC_DEADLOCK] = 1u;
            if (blockIdx.x == 0 && tid == 0) {
                sc[SC_PASSES] = pass + 1;
                sc[SC_NOCONV] = c ? 1u : 0u;
            }
            return;
        }
    }
}

// -------------------------------------------------------------------------------------
// Windowed rank (TPC-C).  The records are sorted by (window, item, ts),
// a window being 2^WB consecutive timestamps, and the fixpoint is iterated one window
// after the other: a group head inside window w starts from the state (a, m) its item
// had at the end of window w-1 (wst[item], (-1, -1) before the first access) instead
// of (-1, -1).  A transaction's records all lie in its own window, and every earlier
// access to an item lies in an earlier window or earlier in the same group, so the
// per-window fixpoint with the carried states is the exact depth (SA-5 "exact" on every
// configuration).  TPC-C's whole-bulk iteration needs ~230 grid passes over all 7 M
// records because its longest paths hop between items hundreds of times; windowed, each
// pass touches one window's ~115 k records (L2-resident) and a window converges in
// <= ~25 passes.  After a window converges one more sweep writes the states of its
// groups' last records to wst.
// -------------------------------------------------------------------------------------
DEV Xf rkw_const(int a, int m) { return Xf{NEG, NEG, a, NEG, NEG, m}; }
// a head's map: the record's map applied after the carried state (a constant)
DEV Xf rkw_xf(bool head, uint32_t mode, int d, int2 c) {
    const Xf x = rec_xf(false, mode, d);
    return head ? OpXf::combine(rkw_const(c.x, c.y), x) : x;
}
DEV int rkw_level(bool head, uint32_t mode, int d, const Xf& cur, int2 c) {
    return rec_level(false, mode, d, head ? rkw_const(c.x, c.y) : cur);
}
// warp-tile [tb, tb + RK_WT) of window [ws, we) into the warp's stage: head/mode/valid
// bits (the window's first record is a head), the records' depths and the heads'
// carried states
DEV uint32_t rkw_load(const uint64_t* __restrict__ keys, uint32_t ws, uint32_t we, uint32_t tb, uint64_t* stage,
                      const uint32_t* D, const int2* wst, int* dv, int2* cs) {
    const uint32_t lane = lane_id();
    __syncwarp();
#pragma unroll
    for (int k = 0; k < RK_ITEMS; ++k) {
        const uint32_t i = k * 32 + lane;
        stage[i] = tb + i < we ? __ldg(&keys[tb + i]) : ~0ull;
    }
    const uint64_t prev = tb > ws ? __ldg(&keys[tb - 1]) : ~0ull;
    __syncwarp();
    uint32_t hw = 0;
#pragma unroll
    for (int k = 0; k < RK_ITEMS; ++k) {
        const uint32_t pos = lane * RK_ITEMS + k;
        dv[k] = 0;
        cs[k] = make_int2(-1, -1);
        if (tb + pos < we) {
            const uint64_t key = stage[pos];
            const uint64_t pk = pos ? stage[pos - 1] : prev;
            const bool head = tb + pos == ws || key_item(pk) != key_item(key);
            hw |= rk_bits(head, key_mode(key), k);
            dv[k] = (int)__ldcg(&D[key_idx(key)]);
            if (head) cs[k] = __ldcg(&wst[key_item(key)]);
        }
    }
    return hw;
}
DEV Xf rkw_compose(uint32_t hw, const int* dv, const int2* cs) {
    Xf agg = OpXf::identity();
#pragma unroll
    for (int k = 0; k < RK_ITEMS; ++k)
        if (rk_valid(hw, k)) agg = OpXf::combine(agg, rkw_xf(rk_head(hw, k), rk_mode(hw, k), dv[k], cs[k]));
    return agg;
}

// CL: launched as ONE thread-block cluster (gridDim.x = cluster size): the barriers
// between the phases of a pass are hardware cluster barriers (release/acquire at
// cluster scope) instead of grid barriers -- a window's passes are latency-bound, so
// fewer SMs with a cheaper barrier win.
template <bool CL>
DEV void rkw_sync(GridBar* bar) {
    if (CL) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else grid_sync(bar);
}
template <bool CL>
__global__ void __launch_bounds__(RK_THREADS, 2) rank_window_kernel(const uint64_t* __restrict__ keys,
                                                                 const uint32_t* __restrict__ seg, uint32_t nwin,
                                                                 uint32_t* D, int2* wst, LookBack<Xf> lb, GridBar* bar,
                                                                 uint32_t* sc, uint32_t max_passes, uint32_t local_max) {
    constexpr uint32_t NW = RK_THREADS / 32;
    __shared__ uint64_t stage_all[NW * RK_WT];
    __shared__ Xf sm[8];
    __shared__ Xf wagg[NW];
    __shared__ int s_chg;
    Xf* cta_agg = lb.agg;
    const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
    uint64_t* stage = stage_all + wid * RK_WT;
    const uint32_t gw = blockIdx.x * NW + wid;
    uint32_t gpass = 0;
    bool noconv = false;
    for (uint32_t w = 0; w < nwin; ++w) {
        const uint32_t ws = __ldcg(&seg[w]), we = __ldcg(&seg[w + 1]);
        if (ws >= we) continue;                          // (uniform: every CTA reads the same seg)
        const uint32_t nwt = (we - ws + RK_WT - 1) / RK_WT;
        const uint32_t per = (nwt + gridDim.x * NW - 1) / (gridDim.x * NW);
        const uint32_t w0 = min(nwt, gw * per), w1 = min(nwt, w0 + per);
        Xf carry0 = OpXf::identity();                    // state entering this warp's range
        // Passes alternate between "fresh" (phase A recomputes every range aggregate from
        // the current depths; 2 barriers) and "reuse" (the aggregates each warp composed
        // while sweeping in the previous pass are published at its end; 1 barrier, no
        // phase A).  Reused aggregates may be stale (another warp raised a shared
        // transaction since) but are lower bounds, so the relaxation stays sound; the
        // window is converged only after a FRESH pass raises nothing.
        bool fresh = true;
        for (uint32_t pass = 0;; ++pass, ++gpass) {
            if (blockIdx.x == 0 && tid == 0) sc[SC_CHG0 + (gpass + 1) % 3] = 0;
            if (tid == 0) s_chg = 0;
            if (fresh) {
                // A: aggregate of this warp's range, then of the CTA's
                Xf mine = OpXf::identity();
                for (uint32_t wt = w0; wt < w1; ++wt) {
                    int dv[RK_ITEMS];
                    int2 cs[RK_ITEMS];
                    const uint32_t hw = rkw_load(keys, ws, we, ws + wt * RK_WT, stage, D, wst, dv, cs);
                    Xf tot;
                    rk_wscan(rkw_compose(hw, dv, cs), tot);
                    mine = OpXf::combine(mine, tot);
                }
                if (lane == 0) wagg[wid] = mine;
                __syncthreads();
                if (tid == 0) {
                    Xf c = OpXf::identity();
                    for (uint32_t j = 0; j < NW; ++j) c = OpXf::combine(c, wagg[j]);
                    lb_store(&cta_agg[blockIdx.x], c);
                }
                rkw_sync<CL>(bar);
            }
            // C: state entering this warp's range
            Xf carry = OpXf::identity();
            for (uint32_t c0 = 0; c0 < blockIdx.x; c0 += RK_THREADS) {
                const Xf x = (c0 + tid < blockIdx.x) ? lb_load(&cta_agg[c0 + tid]) : OpXf::identity();
                Xf tot;
                block_scan_excl<Xf, OpXf>(x, tot, sm);
                carry = OpXf::combine(carry, tot);
            }
            for (uint32_t j = 0; j < wid; ++j) carry = OpXf::combine(carry, wagg[j]);
            carry0 = carry;
            // D: sweep the warp-tiles in order, raising depths (RED.MAX)
            bool wchg = false;
            Xf mine_d = OpXf::identity();
            for (uint32_t wt = w0; wt < w1; ++wt) {
                Xf last_tot = OpXf::identity();
                for (uint32_t it = 0; it < local_max; ++it) {
                    int dv[RK_ITEMS];
                    int2 cs[RK_ITEMS];
                    const uint32_t hw = rkw_load(keys, ws, we, ws + wt * RK_WT, stage, D, wst, dv, cs);
                    Xf tot;
                    const Xf ex = rk_wscan(rkw_compose(hw, dv, cs), tot);
                    last_tot = tot;
                    Xf cur = OpXf::combine(carry, ex);
                    bool chg = false;
#pragma unroll
                    for (int k = 0; k < RK_ITEMS; ++k) {
                        if (!rk_valid(hw, k)) continue;
                        const bool head = rk_head(hw, k);
                        const uint32_t mode = rk_mode(hw, k);
                        const int L = rkw_level(head, mode, dv[k], cur, cs[k]);
                        cur = OpXf::combine(cur, rkw_xf(head, mode, dv[k], cs[k]));
                        if (L > dv[k]) {
                            atomicMax(&D[key_idx(stage[lane * RK_ITEMS + k])], (uint32_t)L);
                            chg = true;
                        }
                    }
                    if (!__any_sync(0xffffffffu, chg)) break;
                    wchg = true;
                }
                carry = OpXf::combine(carry, last_tot);
                mine_d = OpXf::combine(mine_d, last_tot);
            }
            if (lane == 0 && wchg) s_chg = 1;
            __syncthreads();                           // every warp is past C and D
            if (lane == 0) wagg[wid] = mine_d;         // (the next pass may reuse them)
            __syncthreads();
            if (tid == 0) {
                if (s_chg) sc[SC_CHG0 + gpass % 3] = 1;
                Xf cc = OpXf::identity();
                for (uint32_t j = 0; j < NW; ++j) cc = OpXf::combine(cc, wagg[j]);
                lb_store(&cta_agg[blockIdx.x], cc);
            }
            rkw_sync<CL>(bar);
            const uint32_t c = __ldcg(&sc[SC_CHG0 + gpass % 3]);
            if ((!c && fresh) || pass + 1 >= max_passes || __ldcg(&bar->dead)) {
                noconv |= c != 0;
                ++gpass;
                break;
            }
            fresh = !c;                                // nothing raised on reused aggregates: verify
        }
        // the window's final states: the last record of each group writes its item's
        // state (D did not change in the last pass, so carry0 and the sweep are exact)
        {
            Xf carry = carry0;
            for (uint32_t wt = w0; wt < w1; ++wt) {
                const uint32_t tb = ws + wt * RK_WT;
                int dv[RK_ITEMS];
                int2 cs[RK_ITEMS];
                const uint32_t hw = rkw_load(keys, ws, we, tb, stage, D, wst, dv, cs);
                const uint64_t after = tb + RK_WT < we ? __ldg(&keys[tb + RK_WT]) : ~0ull;
                Xf tot;
                const Xf ex = rk_wscan(rkw_compose(hw, dv, cs), tot);
                Xf cur = OpXf::combine(carry, ex);
                int2 outv[RK_ITEMS];
                uint32_t tail = 0;
#pragma unroll
                for (int k = 0; k < RK_ITEMS; ++k) {
                    if (!rk_valid(hw, k)) continue;
                    cur = OpXf::combine(cur, rkw_xf(rk_head(hw, k), rk_mode(hw, k), dv[k], cs[k]));
                    const uint32_t pos = lane * RK_ITEMS + k;
                    const uint64_t nk = pos + 1 < RK_WT ? stage[pos + 1] : after;
                    if (tb + pos + 1 >= we || key_item(nk) != key_item(stage[pos])) {
                        tail |= 1u << k;
                        outv[k] = make_int2(cur.ac, cur.mc);
                    }
                }
#pragma unroll
                for (int k = 0; k < RK_ITEMS; ++k)
                    if ((tail >> k) & 1u) __stcg(&wst[key_item(stage[lane * RK_ITEMS + k])], outv[k]);
                carry = OpXf::combine(carry, tot);
            }
        }
        rkw_sync<CL>(bar);                                   // states visible to the next window
        if (__ldcg(&bar->dead)) break;                      // watchdog: drain
    }
    if (blockIdx.x == 0 && tid == 0) {
        sc[SC_PASSES] = gpass;
        sc[SC_NOCONV] = noconv ? 1u : 0u;
        if (__ldcg(&bar->dead)) sc[SC_DEADLOCK] = 1u;
    }
}

// seg[w] = first sorted record of window w (records sorted by (window, item, ts))
__global__ void __launch_bounds__(256) win_bounds_kernel(const uint64_t* __restrict__ keys, const uint32_t* nrec_ptr,
                                                         uint32_t wb, uint32_t nwin, uint32_t* seg) {
    const uint32_t nrec = *nrec_ptr;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k <= nrec; k += gridDim.x * blockDim.x) {
        const int64_t w = k < nrec ? (int64_t)(key_idx(__ldg(&keys[k])) >> wb) : (int64_t)nwin;
        const int64_t pw = k ? (int64_t)(key_idx(__ldg(&keys[k - 1])) >> wb) : -1;
        for (int64_t q = pw + 1; q <= w; ++q) seg[q] = k;
    }
}

__global__ void __launch_bounds__(RK_THREADS, 2) rank_kernel(const uint64_t* __restrict__ keys, const uint32_t* nrec_ptr,
                                                          uint32_t* D, LookBack<Xf> lb, uint32_t epoch0,
                                                          GridBar* bar, uint32_t* sc, uint32_t max_passes,
                                                          uint32_t local_max, uint32_t use_dirty, RkMemo memo,
                                                          uint64_t* trace) {
    rank_generic(keys, nrec_ptr, D, lb, epoch0, bar, sc, max_passes, local_max, use_dirty, memo, trace);
}

// Root-local rank (TM-1): every warp owns a range of whole roots (a root = all items of
// one subscriber, adjacent in the sorted records) and sweeps it until it raises nothing.
// A transaction whose records all lie in one root is settled by its root alone, so when
// no transaction crosses roots the first pass reaches the fixpoint everywhere and the
// second only confirms it; transactions that do cross roots are still exact: passes
// repeat (grid barrier between them) until one raises nothing.  This replaces ~12 grid
// passes over CTA-sized ranges (hot NURand subscribers spanning several ranges) by
// warp-local sweeps with no inter-warp dependence.
template <int S>
DEV uint64_t rr_root(const DevDb& db, uint64_t key) { return item_root<S>(db, key_item(key)); }

// first record at or after p that starts a root (p itself if p == 0 or p >= nrec);
// searches at most `limit` records (4 x 32 loads in flight per step) and returns
// 0xFFFFFFFF if the root continues past them
template <int S>
DEV uint32_t rr_align(const DevDb& db, const uint64_t* __restrict__ keys, uint32_t nrec, uint32_t p, uint32_t limit) {
    if (p == 0 || p >= nrec) return min(p, nrec);
    const uint64_t r0 = rr_root<S>(db, __ldg(&keys[p - 1]));
    const uint32_t end = (uint32_t)min((uint64_t)nrec, (uint64_t)p + limit);
    for (uint32_t b = p; b < end; b += 128) {
        uint64_t k[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t i = b + 32 * j + lane_id();
            k[j] = i < end ? __ldg(&keys[i]) : 0ull;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t i = b + 32 * j + lane_id();
            const uint32_t m = __ballot_sync(0xffffffffu, i < end && rr_root<S>(db, k[j]) != r0);
            if (m) return b + 32 * j + __ffs(m) - 1;
        }
    }
    return end == nrec ? nrec : 0xFFFFFFFFu;
}

//
// A root holding many times a warp's share of the records (a hot branch: TPC-B with
// hot-branch skew puts ~10% of all records in branch 0) would serialise the pass on one
// warp, so the kernel first checks the aligned ranges: if any exceeds RR_SPLIT x the
// even share, every CTA runs the grid-wide scan (rank_generic) instead.
constexpr uint32_t RR_SPLIT = 8;
template <int S>
__global__ void __launch_bounds__(RK_THREADS) rank_root_kernel(DevDb db, const uint64_t* __restrict__ keys,
                                                               const uint32_t* nrec_ptr, uint32_t* D, GridBar* bar,
                                                               uint32_t* sc, uint32_t max_passes, uint64_t* trace,
                                                               LookBack<Xf> lb, uint32_t epoch0, uint32_t local_max,
                                                               uint32_t use_dirty, RkMemo memo) {
    constexpr uint32_t NW = RK_THREADS / 32;
    __shared__ uint64_t stage_all[NW * RK_WT];
    __shared__ int s_chg;
    const uint32_t nrec = *nrec_ptr;
    const uint32_t tid = threadIdx.x, lane = lane_id(), wid = tid >> 5;
    uint64_t* stage = stage_all + wid * RK_WT;
    const uint32_t TW = gridDim.x * NW, gw = blockIdx.x * NW + wid;
    const uint32_t chunk = (nrec + TW - 1) / TW;
    const uint32_t lim = RR_SPLIT * max(chunk, RK_WT);
    const uint32_t r0 = rr_align<S>(db, keys, nrec, gw * chunk, lim);
    const uint32_t r1 = rr_align<S>(db, keys, nrec, (gw + 1) * chunk, lim);
    if (lane == 0 && (r0 == 0xFFFFFFFFu || r1 == 0xFFFFFFFFu || r1 - r0 > lim)) atomicOr(&sc[SC_RRSPLIT], 1u);
    grid_sync(bar);
    if (__ldcg(&sc[SC_RRSPLIT])) {
        rank_generic(keys, nrec_ptr, D, lb, epoch0, bar, sc, max_passes, local_max, use_dirty, memo, trace);
        return;
    }
    for (uint32_t pass = 0;; ++pass) {
        if (blockIdx.x == 0 && tid == 0) sc[SC_CHG0 + (pass + 1) % 3] = 0;
        if (tid == 0) s_chg = 0;
        if (trace && blockIdx.x == 0 && tid == 0 && pass < RANK_TRACE_SLOTS / 8) trace[8 * pass] = globaltimer_ns();
        __syncthreads();
        bool wchg = false;
        uint32_t sweeps = 0;
        for (;; ++sweeps) {
            bool raised = false;
            Xf carry = OpXf::identity();
            for (uint32_t c = r0; c < r1; c += RK_WT) {
                // chunk [c, min(c + RK_WT, r1)) into the warp's stage
                __syncwarp();
#pragma unroll
                for (int k = 0; k < RK_ITEMS; ++k) {
                    const uint32_t i = k * 32 + lane;
                    stage[i] = c + i < r1 ? __ldg(&keys[c + i]) : ~0ull;
                }
                const uint64_t prev = c ? __ldg(&keys[c - 1]) : ~0ull;
                __syncwarp();
                uint32_t hw = 0;
#pragma unroll
                for (int k = 0; k < RK_ITEMS; ++k) {
                    const uint32_t pos = lane * RK_ITEMS + k;
                    if (c + pos < r1) {
                        const uint64_t key = stage[pos];
                        const uint64_t pk = pos ? stage[pos - 1] : prev;
                        const bool head = (c + pos == 0) || key_item(pk) != key_item(key);
                        hw |= rk_bits(head, key_mode(key), k);
                    }
                }
                int dv[RK_ITEMS];
                rk_wgather(stage, hw, D, dv);
                Xf tot;
                const Xf ex = rk_wscan(rk_compose(hw, dv), tot);
                Xf cur = OpXf::combine(carry, ex);
                int L[RK_ITEMS];
#pragma unroll
                for (int k = 0; k < RK_ITEMS; ++k) {
                    L[k] = 0;
                    if (rk_valid(hw, k)) {
                        const bool head = rk_head(hw, k);
                        const uint32_t mode = rk_mode(hw, k);
                        L[k] = rec_level(head, mode, dv[k], cur);
                        cur = OpXf::combine(cur, rec_xf(head, mode, dv[k]));
                    }
                }
                bool chg = false;                  // RED.MAX raises (see rank_generic)
#pragma unroll
                for (int k = 0; k < RK_ITEMS; ++k)
                    if (L[k] > dv[k]) {
                        atomicMax(&D[key_idx(stage[lane * RK_ITEMS + k])], (uint32_t)L[k]);
                        chg = true;
                    }
                raised |= __any_sync(0xffffffffu, chg);
                carry = OpXf::combine(carry, tot);
            }
            if (!raised) break;
            wchg = true;
            if (sweeps + 1 >= max_passes) break;
        }
        if (lane == 0 && wchg) s_chg = 1;
        if (trace && lane == 0 && pass < RANK_TRACE_SLOTS / 8)
            atomicMax(reinterpret_cast<unsigned long long*>(&trace[8 * pass + 6]), (unsigned long long)sweeps);
        __syncthreads();
        if (tid == 0 && s_chg) sc[SC_CHG0 + pass % 3] = 1;
        if (trace && tid == 0 && pass < RANK_TRACE_SLOTS / 8)
            atomicMax(reinterpret_cast<unsigned long long*>(&trace[8 * pass + 3]), (unsigned long long)globaltimer_ns());
        grid_sync(bar);
        if (trace && blockIdx.x == 0 && tid == 0 && pass < RANK_TRACE_SLOTS / 8) trace[8 * pass + 4] = globaltimer_ns();
        const uint32_t c = __ldcg(&sc[SC_CHG0 + pass % 3]);
        if (!c || pass + 1 >= max_passes || __ldcg(&bar->dead)) {
            if (blockIdx.x == 0 && tid == 0 && __ldcg(&bar->dead)) sc[SC_DEADLOCK] = 1u;
            if (blockIdx.x == 0 && tid == 0) {
                sc[SC_PASSES] = pass + 1;
                sc[SC_NOCONV] = c ? 1u : 0u;
            }
            return;
        }
    }
}

// Root-stream rank (TM-1): every TM-1 transaction touches the items of ONE subscriber
// (PAPER.md:451-453), so the T-dependency graph is a disjoint union of per-subscriber
// graphs -- finer: per (subscriber, item component), TM1_COMP_BITS in schema.cuh.  The
// records are sorted on the (subscriber, component) bits only (stable: (root, ts)
// order, a transaction's records adjacent), and the streaming depth recurrence runs
// over each root's records in ts order (SURVEY.md §8(c) "Depth oracle"):
//   d(t) = max over t's records of (write ? Md[x] + 1 : Wd[x] + 1), 0 without records;
//   then write: Wd[x] = Md[x] = d(t);  read: Md[x] = max(Md[x], d(t)).
// Exact in one pass (the streaming order is a topological order of the root's graph).
// A root has <= 8 item slots (item & 7); their state (Wd, Md) lives in registers
// (constant-indexed, selected by a 3-level tree).  This replaces the iterated scan's
// repeated sweeps of hot NURand subscribers (13 sweeps in the first pass, round 1).
constexpr int RS_STREAM_THREADS = 128;
constexpr int RS_CHUNK = 8;
constexpr uint32_t RS_LONG = 32;                           // longer roots: warp walk
constexpr int RS_STREAM_TILE = RS_STREAM_THREADS * 8;     // records scanned for heads per CTA
constexpr uint32_t TM1_ROOT_SLOTS = 1u << TM1_COMP_BITS;

struct Tm1RootState {
    int W[TM1_ROOT_SLOTS], M[TM1_ROOT_SLOTS];
    uint32_t wm = 0, rm = 0;                 // the open transaction's written / read slots
    int d = 0;                               // and its depth so far
    DEV Tm1RootState() {
#pragma unroll
        for (int j = 0; j < (int)TM1_ROOT_SLOTS; ++j) W[j] = M[j] = -1;
    }
    DEV static int sel(const int* a, uint32_t x) {
        const int l = x & 2u ? (x & 1u ? a[3] : a[2]) : (x & 1u ? a[1] : a[0]);
        const int h = x & 2u ? (x & 1u ? a[7] : a[6]) : (x & 1u ? a[5] : a[4]);
        return x & 4u ? h : l;
    }
    // one record (slot x, write w) of the open transaction; nothing when !valid
    DEV void access(uint32_t x, bool w, bool valid) {
        const int v = (w ? sel(M, x) : sel(W, x)) + 1;
        d = valid ? max(d, v) : d;
        const uint32_t b = valid ? 1u << x : 0u;
        wm |= w ? b : 0u;
        rm |= w ? 0u : b;
    }
    // the open transaction closes when c: its depth updates its slots (branch-free)
    DEV void close(bool c) {
#pragma unroll
        for (int j = 0; j < (int)TM1_ROOT_SLOTS; ++j) {
            const bool wj = c && (wm >> j & 1u), rj = c && (rm >> j & 1u);
            W[j] = wj ? d : W[j];
            M[j] = wj ? d : (rj ? max(M[j], d) : M[j]);
        }
        d = c ? 0 : d;
        wm = c ? 0u : wm;
        rm = c ? 0u : rm;
    }
};
DEV uint64_t tm1_root(uint64_t k) { return key_item(k) >> TM1_COMP_BITS; }
DEV uint32_t tm1_slot(uint64_t k) { return (uint32_t)key_item(k) & (TM1_ROOT_SLOTS - 1); }

// Each CTA first lists the root heads (first record of a root) of its tile of
// RS_STREAM_TILE sorted records in position order (block scan), so a root ends at the
// next head.  A root whose records all belong to one transaction has depth 0 (skipped:
// D is zero-filled); other roots up to RS_LONG records are walked one per thread, longer
// ones (hot NURand subscribers, up to ~660 records) one per warp: the warp loads 32
// consecutive keys per instruction, two chunks ahead, every lane decodes its own record
// (slot, mode, first-of-transaction) and the recurrence runs branch-free over the 32
// broadcast records in every lane, so only its ~20-cycle state dependence is serial.
__global__ void __launch_bounds__(RS_STREAM_THREADS) rank_stream_tm1_kernel(const uint64_t* __restrict__ keys,
                                                                           const uint32_t* nrec_ptr, uint32_t* D,
                                                                           uint32_t* sc) {
    constexpr int PER = RS_STREAM_TILE / RS_STREAM_THREADS;
    __shared__ uint32_t heads[RS_STREAM_TILE + 1];
    __shared__ uint32_t longs[RS_STREAM_TILE];
    __shared__ uint32_t scan_sm[RS_STREAM_THREADS / 32];
    __shared__ uint32_t s_nl;
    __shared__ int2 wstate[RS_STREAM_THREADS / 32][TM1_ROOT_SLOTS];
    __shared__ uint2 wbuf[RS_STREAM_THREADS / 32][32];
    const uint32_t nrec = *nrec_ptr;
    const uint32_t ntiles = (nrec + RS_STREAM_TILE - 1) / RS_STREAM_TILE;
    const uint32_t tid = threadIdx.x, lane = lane_id();
    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (tid == 0) s_nl = 0;
        const uint32_t t0 = tile * RS_STREAM_TILE;
        const uint32_t tend = min(t0 + (uint32_t)RS_STREAM_TILE, nrec);
        // heads of this thread's PER consecutive records, then a block scan
        const uint32_t pb = t0 + tid * PER;
        uint64_t prev = pb > 0 && pb - 1 < nrec ? __ldg(&keys[pb - 1]) : ~0ull;
        uint32_t flags = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            if (pb + i < nrec) {
                const uint64_t k = __ldg(&keys[pb + i]);
                if (pb + i == 0 || tm1_root(prev) != tm1_root(k)) flags |= 1u << i;
                prev = k;
            }
        }
        uint32_t nh;
        uint32_t at = block_scan_excl<uint32_t, OpAddU32>((uint32_t)__popc(flags), nh, scan_sm);
        for (uint32_t f = flags; f; f &= f - 1) heads[at++] = pb + (__ffs(f) - 1);
        if (tid == 0) heads[nh] = tend;
        __syncthreads();
        // long roots first (the hot subscribers' walks are the kernel's critical path)
        for (uint32_t h = tid; h < nh; h += RS_STREAM_THREADS) {
            const uint32_t p = heads[h], e = heads[h + 1];
            if (e - p > RS_LONG || (h + 1 == nh && e < nrec && tm1_root(__ldg(&keys[e])) == tm1_root(__ldg(&keys[p]))))
                longs[atomicAdd(&s_nl, 1u)] = p;
        }
        __syncthreads();
        const uint32_t nl = s_nl;
        int2* ws = wstate[warp_id()];
        for (uint32_t h = warp_id(); h < nl; h += RS_STREAM_THREADS / 32) {
            const uint32_t p = longs[h];
            const uint64_t kp = __ldg(&keys[p]);
            const uint64_t root = tm1_root(kp);
            auto ld = [&](uint32_t q) { return q + lane < nrec ? __ldg(&keys[q + lane]) : ~0ull; };
            uint64_t c0 = ld(p), c1 = ld(p + 32), carry = ~0ull;   // carry: the previous chunk's last key
            uint32_t q = p + 64;
            if (lane < TM1_ROOT_SLOTS) ws[lane] = make_int2(-1, -1);
            __syncwarp();
            bool go = true;
            while (go) {
                const uint64_t c2 = ld(q);
                q += 32;
                // lane-parallel: does this lane's record start a transaction; if so, its
                // <= 3 records (this one and the next two, looking into the next chunk)
                // packed 4 bits each (slot | write << 3) with their count
                uint64_t kprev = __shfl_up_sync(0xffffffffu, c0, 1);
                if (lane == 0) kprev = carry;
                const bool valid = tm1_root(c0) == root;                    // a prefix of the chunk
                const bool start = valid && (lane == 0 && carry == ~0ull ? true : key_idx(c0) != key_idx(kprev));
                const uint64_t a1 = __shfl_down_sync(0xffffffffu, c0, 1), b1 = __shfl_sync(0xffffffffu, c1, (lane + 1) & 31);
                const uint64_t a2 = __shfl_down_sync(0xffffffffu, c0, 2), b2 = __shfl_sync(0xffffffffu, c1, (lane + 2) & 31);
                const uint64_t k1 = lane + 1 < 32 ? a1 : b1, k2 = lane + 2 < 32 ? a2 : b2;
                const uint32_t id = key_idx(c0);
                const bool h1 = tm1_root(k1) == root && key_idx(k1) == id;
                const bool h2 = h1 && tm1_root(k2) == root && key_idx(k2) == id;
                auto enc = [](uint64_t k) { return tm1_slot(k) | (key_mode(k) == 1u ? 8u : 0u); };
                const uint32_t tw = enc(c0) | (h1 ? enc(k1) << 4 | 1u << 12 : 0u) | (h2 ? enc(k2) << 8 | 1u << 13 : 0u);
                const uint32_t vm = __ballot_sync(0xffffffffu, valid);
                go = vm == 0xffffffffu;
                carry = __shfl_sync(0xffffffffu, c0, 31);
                // serial part, one transaction per step (warp-uniform: every lane keeps the
                // same slot state (Wd, Md) in this warp's shared words)
                // the chunk's transactions compacted in order into this warp's buffer, so the
                // serial loop's loads of them are independent of its state chain
                const uint32_t smask = __ballot_sync(0xffffffffu, start);
                if (start) wbuf[warp_id()][__popc(smask & lanemask_lt())] = make_uint2(tw, id);
                __syncwarp();
                const int ns = __popc(smask);
#pragma unroll 8
                for (int j = 0; j < ns; ++j) {
                    const uint2 tj = wbuf[warp_id()][j];
                    const uint32_t t = tj.x, cid = tj.y;
                    const uint32_t e0 = t & 15u, e1 = (t >> 4) & 15u, e2 = (t >> 8) & 15u;
                    const int2 s0 = ws[e0 & 7u], s1 = ws[e1 & 7u], s2 = ws[e2 & 7u];
                    int d = ((e0 & 8u) ? s0.y : s0.x) + 1;
                    if (t & (1u << 12)) d = max(d, ((e1 & 8u) ? s1.y : s1.x) + 1);
                    if (t & (1u << 13)) d = max(d, ((e2 & 8u) ? s2.y : s2.x) + 1);
                    ws[e0 & 7u] = (e0 & 8u) ? make_int2(d, d) : make_int2(s0.x, max(s0.y, d));
                    if (t & (1u << 12)) ws[e1 & 7u] = (e1 & 8u) ? make_int2(d, d) : make_int2(s1.x, max(s1.y, d));
                    if (t & (1u << 13)) ws[e2 & 7u] = (e2 & 8u) ? make_int2(d, d) : make_int2(s2.x, max(s2.y, d));
                    if (lane == 0 && d) D[cid] = (uint32_t)d;
                }
                __syncwarp();
                c0 = c1;
                c1 = c2;
            }
            __syncwarp();
        }
        for (uint32_t h = tid; h < nh; h += RS_STREAM_THREADS) {
            const uint32_t p = heads[h], e = heads[h + 1];
            const uint64_t k0 = __ldg(&keys[p]);
            if (e - p > RS_LONG || (h + 1 == nh && e < nrec && tm1_root(__ldg(&keys[e])) == tm1_root(k0)))
                continue;                                                 // walked by a warp
            if (key_idx(__ldg(&keys[e - 1])) == key_idx(k0)) continue;   // one transaction: depth 0
            Tm1RootState st;
            uint32_t tidx = key_idx(k0);
            for (uint32_t q = p; q < e; ++q) {
                const uint64_t k = __ldg(&keys[q]);            // (L1: this tile)
                const uint32_t id = key_idx(k);
                if (id != tidx) {
                    if (st.d) D[tidx] = (uint32_t)st.d;
                    st.close(true);
                    tidx = id;
                }
                st.access(tm1_slot(k), key_mode(k) == 1u, true);
            }
            if (st.d) D[tidx] = (uint32_t)st.d;
        }
        __syncthreads();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) sc[SC_PASSES] = 1;
}

// =====================================================================================
// group by (depth, type): counting sort.  Each CTA first aggregates its tile's keys in
// a shared-memory table (open addressing) so hot keys (the 0-set of a wide graph) cost
// one global atomic per CTA instead of one per warp; keys that do not fit go global.
// =====================================================================================
// Block-level reductions of grid-stride counters: one global atomic per CTA (a global
// atomic per warp on one address serialises thousands of them at L2).
DEV uint32_t block_sum_u32(uint32_t v) {      // result valid in thread 0 (blockDim.x <= 1024)
    __shared__ uint32_t red_sm[32];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane_id() == 0) red_sm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? red_sm[threadIdx.x] : 0u;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    }
    return v;
}
DEV uint32_t block_max_u32(uint32_t v) {      // result valid in thread 0
    __shared__ uint32_t rmx_sm[32];
#pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane_id() == 0) rmx_sm[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        v = threadIdx.x < (blockDim.x >> 5) ? rmx_sm[threadIdx.x] : 0u;
#pragma unroll
        for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    }
    return v;
}

// (a depth the spine walk left unset -- only after its watchdog tripped, EDEADLOCK -- counts
// as 0 so that nothing downstream sizes work by it)
__global__ void __launch_bounds__(256) depth_reduce_kernel(uint32_t* D, uint32_t n, uint32_t* sc) {
    uint32_t mx = 0, z = 0;
    const uint32_t n4 = n / 4;
    uint4* D4 = reinterpret_cast<uint4*>(D);                     // D is cudaMalloc'ed: 16-B aligned
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
        uint4 d = __ldcg(&D4[i]);
        if ((d.x & d.y & d.z & d.w) == 0xFFFFFFFFu || d.x == 0xFFFFFFFFu || d.y == 0xFFFFFFFFu || d.z == 0xFFFFFFFFu ||
            d.w == 0xFFFFFFFFu) {
            d.x = d.x == 0xFFFFFFFFu ? 0u : d.x; d.y = d.y == 0xFFFFFFFFu ? 0u : d.y;
            d.z = d.z == 0xFFFFFFFFu ? 0u : d.z; d.w = d.w == 0xFFFFFFFFu ? 0u : d.w;
            D4[i] = d;
        }
        mx = max(max(mx, max(d.x, d.y)), max(d.z, d.w));
        z += (d.x == 0) + (d.y == 0) + (d.z == 0) + (d.w == 0);
    }
    for (uint32_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        uint32_t d = __ldcg(&D[i]);
        if (d == 0xFFFFFFFFu) { d = 0; D[i] = 0; }
        mx = max(mx, d);
        z += d == 0;
    }
    mx = block_max_u32(mx);
    z = block_sum_u32(z);
    if (threadIdx.x == 0) {
        atomicMax(&sc[SC_MAXD], mx);
        atomicAdd(&sc[SC_ZERO], z);
    }
}

__global__ void group_nkeys_kernel(uint32_t* sc, uint32_t T) {
    sc[SC_NKEYS] = (sc[SC_MAXD] + 1) * T;
    sc[SC_NKEYS1] = (sc[SC_MAXD] + 1) * T + 1;
}

// group_nkeys_kernel + zero_dev_kernel in one launch: every thread derives the key count
__global__ void __launch_bounds__(256) group_zero_kernel(uint32_t* cnt, uint32_t* sc, uint32_t T) {
    const uint32_t nk = (__ldcg(&sc[SC_MAXD]) + 1) * T;
    if (blockIdx.x == 0 && threadIdx.x == 0) { sc[SC_NKEYS] = nk; sc[SC_NKEYS1] = nk + 1; }
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nk + 1; i += gridDim.x * blockDim.x) cnt[i] = 0;
}

__global__ void pull_sc_kernel(const uint32_t* __restrict__ sc, uint32_t* host_mapped, uint32_t n) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) host_mapped[i] = __ldcg(&sc[i]);
}

// zero `bytes` bytes (16-B vector stores; `a` 16-B aligned).  Used instead of
// cudaMemsetAsync for the per-bulk status / output buffers: a memset can be serviced by a
// copy engine and then queues behind an in-flight D2H of the previous bulk's results
// (gputx_run_bulks measured 1.67 vs 1.05 ms per TM-1 bulk).
__global__ void __launch_bounds__(256) zero_bytes_kernel(uint8_t* a, uint64_t bytes) {
    const uint64_t n16 = bytes / 16;
    uint4* v = reinterpret_cast<uint4*>(a);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
        v[i] = make_uint4(0u, 0u, 0u, 0u);
    for (uint64_t i = n16 * 16 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < bytes;
         i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = 0;
}

__global__ void __launch_bounds__(256) zero_dev_kernel(uint32_t* a, const uint32_t* n_ptr) {
    const uint32_t n = *n_ptr;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = 0;
}

constexpr int GR_ITEMS = 16, GR_TILE = 256 * GR_ITEMS, GR_SLOTS = 1024, GR_PROBE = 8;
constexpr uint32_t GR_EMPTY = 0xFFFFFFFFu;

// insert key into the smem table, returns slot or -1
DEV int gr_slot(uint32_t* skey, uint32_t key) {
    uint32_t h = (key * 0x9E3779B1u) >> 22;            // 10 bits
    for (int p = 0; p < GR_PROBE; ++p) {
        const uint32_t s = (h + p) & (GR_SLOTS - 1);
        const uint32_t old = atomicCAS(&skey[s], GR_EMPTY, key);
        if (old == GR_EMPTY || old == key) return (int)s;
    }
    return -1;
}

// mode 0: histogram into cnt[]; mode 1: scatter perm[] (cnt[] counts down) and, for
// PW > 0, the type and the first PW parameter words of each transaction into execution
// order (ptype[pos], pp[pos*PW..]) so the executor reads them coalesced.
// Owner keys (K-SET owner-local rounds): with OS = the schema, mode 1 also writes
// okeys[pos] = owner(i) << 32 | pos (and own[i]) for the stable owner sort.
struct OwnKeys {
    uint32_t nw;
    uint64_t* keys;
    uint32_t* own;
    uint32_t diag;
    const uint32_t* err;      // pipelined run_bulks: failed bulk -> no parameter reads
};
template <int S>
DEV uint32_t own_of(const uint32_t* p, uint32_t nw, uint32_t idx, uint32_t diag);

template <int MODE, int PW, int OS = 0>
__global__ void __launch_bounds__(256) group_kernel(const uint32_t* __restrict__ D, const uint8_t* __restrict__ type,
                                                    uint32_t n, uint32_t T, uint32_t* cnt, const uint32_t* off,
                                                    uint32_t* perm, const uint32_t* __restrict__ poff,
                                                    const uint32_t* __restrict__ pw, uint8_t* ptype, uint32_t* pp,
                                                    uint32_t P, OwnKeys ok = {}) {
    __shared__ uint32_t skey[GR_SLOTS];
    __shared__ uint32_t scnt[GR_SLOTS];
    __shared__ uint32_t sbase[GR_SLOTS];
    for (uint64_t t0 = (uint64_t)blockIdx.x * GR_TILE; t0 < n; t0 += (uint64_t)gridDim.x * GR_TILE) {
        for (int s = threadIdx.x; s < GR_SLOTS; s += 256) { skey[s] = GR_EMPTY; scnt[s] = 0; }
        __syncthreads();
        uint32_t key[GR_ITEMS];
        int slot[GR_ITEMS];
        uint32_t rank[GR_ITEMS];
#pragma unroll
        for (int k = 0; k < GR_ITEMS; ++k) {
            const uint64_t i = t0 + k * 256 + threadIdx.x;
            // type groups: P partitions of the type ids by their high part (P = T: one
            // group per type; P = 1: depth only) -- PAPER.md:402-404 radix passes on type
            key[k] = i < n ? D[i] * T + (P >= T ? type[i] : type[i] * P / T) : GR_EMPTY;
            const uint32_t peers = __match_any_sync(0xffffffffu, key[k]);
            const int leader = __ffs(peers) - 1;
            int sl = -1;
            uint32_t old = 0;
            if (key[k] != GR_EMPTY && (int)lane_id() == leader) {
                sl = gr_slot(skey, key[k]);
                if (sl >= 0) old = atomicAdd(&scnt[sl], __popc(peers));
                else if (MODE == 0) atomicAdd(&cnt[key[k]], __popc(peers));
                else old = atomicSub(&cnt[key[k]], __popc(peers)) - __popc(peers);   // global slot range
            }
            sl = __shfl_sync(0xffffffffu, sl, leader);
            old = __shfl_sync(0xffffffffu, old, leader);
            slot[k] = sl;
            rank[k] = old + __popc(peers & lanemask_lt());
        }
        __syncthreads();
        for (int s = threadIdx.x; s < GR_SLOTS; s += 256) {
            if (skey[s] != GR_EMPTY) {
                if (MODE == 0) atomicAdd(&cnt[skey[s]], scnt[s]);
                else sbase[s] = atomicSub(&cnt[skey[s]], scnt[s]) - scnt[s];
            }
        }
        __syncthreads();
        if (MODE == 1) {
#pragma unroll
            for (int k = 0; k < GR_ITEMS; ++k) {
                if (key[k] == GR_EMPTY) continue;
                const uint32_t i = (uint32_t)(t0 + k * 256 + threadIdx.x);
                const uint32_t pos = off[key[k]] + (slot[k] >= 0 ? sbase[slot[k]] + rank[k] : rank[k]);
                perm[pos] = i;
                if (OS) {
                    const uint32_t o = ok.err && __ldcg(ok.err) ? 0u : own_of<OS>(pw + poff[i], ok.nw, i, ok.diag);
                    ok.keys[pos] = ((uint64_t)o << 32) | pos;
                    if (ok.own) ok.own[i] = o;
                }
                if (PW > 0) {
                    ptype[pos] = type[i];
                    const uint32_t* src = pw + poff[i];
                    uint32_t v[PW > 0 ? PW : 1];
#pragma unroll
                    for (int w = 0; w < PW; ++w) v[w] = src[w];
#pragma unroll
                    for (int w = 0; w < PW; w += 4)
                        *reinterpret_cast<uint4*>(pp + (uint64_t)pos * PW + w) = make_uint4(v[w], v[w + 1], v[w + 2], v[w + 3]);
                }
            }
        }
        __syncthreads();
    }
}

// =====================================================================================
// K-SET executor.  Round k (k-set k) needs g[k] = ceil(|k-set| / B)
// CTAs (<= grid).  The g[k] participants of round k wait until all g[k-1] participants
// of round k-1 have signalled done[k-1]; no grid-wide barrier.  Consecutive rounds
// that fit one CTA run in CTA 0 separated by __syncthreads only.  Property 1: no
// locks inside a round.  For PW > 0 the next round's transaction ids and parameter
// words are loaded into registers before the current round executes.
// =====================================================================================
__global__ void kset_sched_kernel(const uint32_t* __restrict__ off, uint32_t T, const uint32_t* sc, uint32_t G,
                                  uint32_t per_cta, uint16_t* g, uint32_t* done) {
    const uint32_t nk = __ldcg(&sc[SC_MAXD]) + 1;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nk; k += gridDim.x * blockDim.x) {
        const uint32_t s = off[(k + 1) * T] - off[k * T];
        uint32_t c = (s + per_cta - 1) / per_cta;
        g[k] = (uint16_t)(c < 1 ? 1 : (c > G ? G : c));
        if (done) done[k] = 0;
    }
}

// GPUTX_KSET_DIAG bit 1024 (tests only): a pseudo-random 0..2 us sleep before every
// transaction a thread executes, so that rounds finish in a different order every run
// (timing-perturbation stress test of the round hand-offs, tests/test_gpu_stress.py)
DEV void kx_jitter(uint32_t diag, uint32_t k, uint32_t b, uint32_t tid) {
    if (diag & 1024u) {
        uint32_t h = (k * 0x9E3779B1u) ^ (b * 0x85EBCA77u) ^ (tid * 0xC2B2AE3Du) ^ (uint32_t)clock64();
        h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12;
        __nanosleep(h & 2047u);
    }
}

constexpr int KX_THREADS = 1024;
constexpr uint32_t KX_CH = 2048;      // rounds staged per shared-memory chunk

template <int S, int PW, int KB, bool SH>
__global__ void __launch_bounds__(KB) kset_exec_kernel(DevDb db, const uint32_t* __restrict__ perm,
                                                               const uint32_t* __restrict__ off, uint32_t T,
                                                               const uint16_t* __restrict__ g, uint32_t* done,
                                                               const uint32_t* sc, const uint8_t* __restrict__ ptype,
                                                               const uint32_t* __restrict__ pp, uint64_t* trace,
                                                               uint32_t diag, uint32_t cluster_c) {
    const uint32_t nk = __ldcg(&sc[SC_MAXD]) + 1;
    const uint32_t b = blockIdx.x, tid = threadIdx.x;
    constexpr bool TAILRUN = S != S_TPCC && PW > 0;
    // The cluster hand-offs below are only valid if the launch really formed clusters of
    // cluster_c CTAs.  A launcher that drops the cluster attribute (a profiler replaying
    // the launch does: GPUTEST_r01's ncu-wrapped smoke ran every CTA as its own cluster, so
    // barrier.cluster synchronised nothing and narrow rounds raced) must not break the
    // schedule: read the shape the hardware gave us and fall back to counter hand-offs.
    uint32_t ncta_cluster;
    asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncta_cluster));
    if (cluster_c && ncta_cluster != cluster_c) {
        if (b == 0 && tid == 0) const_cast<uint32_t*>(sc)[SC_NOCLUSTER] = ncta_cluster;
        cluster_c = 0;
    }
    // prefetched first slice of the round this CTA executes next
    uint32_t nidx = 0xFFFFFFFFu, nt = 0;
    uint32_t np[PW > 0 ? PW : 1];
    // CTA b's slice of a round [lo, hi) executed by gk CTAs: contiguous chunk b
    auto slice = [&](uint32_t lo, uint32_t hi, uint32_t gk, uint32_t& slo, uint32_t& shi) {
        const uint32_t chunk = (hi - lo + gk - 1) / gk;
        slo = lo + b * chunk;
        shi = min(hi, slo + chunk);
    };
    // TPC-C: one warp per transaction (tpcc_txn_warp); nothing is staged per thread
    constexpr bool WARPX = S == S_TPCC;
    auto prefetch = [&](uint32_t lo, uint32_t hi) {     // [lo, hi) = this CTA's slice
        const uint32_t j = lo + tid;
        nidx = 0xFFFFFFFFu;
        if (!WARPX && j < hi) {
            nidx = __ldg(&perm[j]);
            if (PW > 0) {
                nt = __ldg(&ptype[j]);
#pragma unroll
                for (int w = 0; w < (PW > 0 ? PW : 1); w += 4) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(pp + (uint64_t)j * PW + w));
                    np[w] = v.x; np[w + 1] = v.y; np[w + 2] = v.z; np[w + 3] = v.w;
                }
            }
        }
    };
    // round metadata (g[k], k-set start off[k*T]) staged in shared memory by chunks:
    // the per-round lookups on the critical path are shared-memory hits
    __shared__ uint16_t sg[KX_CH];
    __shared__ uint32_t soff[KX_CH + 1];
    uint32_t cb = 0xFFFFFFFFu;
    auto load_chunk = [&](uint32_t base) {           // CTA-uniform
        __syncthreads();
        for (uint32_t i = tid; i < KX_CH; i += KB) sg[i] = base + i < nk ? __ldg(&g[base + i]) : (uint16_t)0;
        for (uint32_t i = tid; i <= KX_CH; i += KB) soff[i] = base + i <= nk ? __ldcg(&off[(base + i) * T]) : 0u;
        __syncthreads();
        cb = base;
    };
    auto G = [&](uint32_t kk) -> uint32_t {
        if (kk < cb || kk >= cb + KX_CH) load_chunk(kk - kk % KX_CH);
        return sg[kk - cb];
    };
    auto bounds = [&](uint32_t kk, uint32_t& l, uint32_t& h) {
        G(kk);
        l = soff[kk - cb];
        h = soff[kk - cb + 1];
    };
    if (diag & 128u) {                 // hand-off skeleton only (diagnostics)
        for (uint32_t kk = 0; kk < nk; ++kk) {
            const uint32_t gg = __ldg(&g[kk]);
            if (b >= gg) continue;
            if (kk > 0) {
                if (tid == 0) {
                    const uint32_t need = __ldg(&g[kk - 1]);
                    while (ld_acquire(&done[kk - 1]) < need) { }
                }
                __syncthreads();
            }
            if (trace && b == 0 && tid == 0) trace[8 * kk] = globaltimer_ns();
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                atomicAdd(&done[kk], 1u);
            }
        }
        return;
    }
    // Round classes.  With a cluster launch (C > 0) a round of g <= C CTAs is "narrow":
    // it is run by cluster 0 (CTAs 0..C-1, only the first g hold work) and consecutive
    // narrow rounds are separated by the hardware cluster barrier alone.  A "wide"
    // round (g > C, or any round without clusters) is run by CTAs 0..g-1, which wait for
    // the previous round's signals on done[k-1] and signal done[k] when done.
    const uint32_t C = cluster_c;
    auto narrow = [&](uint32_t kk) -> bool { return C && G(kk) <= C; };
    auto part = [&](uint32_t kk) -> bool { return narrow(kk) ? b < C : b < G(kk); };
    auto nsig = [&](uint32_t kk) -> uint32_t { return narrow(kk) ? C : G(kk); };   // signals of round kk
    // watchdog (GPUTX_WATCHDOG_MS): a wait that times out puts the CTA in drain mode --
    // it still walks the schedule, signals and takes part in cluster barriers so that no
    // other CTA hangs on it, but neither waits nor executes; the host reports EDEADLOCK
    __shared__ uint32_t s_dead;
    __shared__ uint32_t s_run[2];
    if (tid == 0) s_dead = 0;
    bool dead = false;
    uint32_t k = 0;
    while (k < nk && !part(k)) ++k;                      // this CTA's first round
    if (k >= nk) return;
    uint32_t lo, hi;
    bounds(k, lo, hi);
    slice(lo, hi, G(k), lo, hi);
    prefetch(lo, hi);
    uint32_t prev = 0xFFFFFFFFu, gprev = 0;   // last round this CTA executed, its CTA count
    while (k < nk) {
        const uint32_t gk = G(k);
        const bool nar = narrow(k);
        // wait for round k-1 (nothing to wait for after a narrow round: cluster barrier).
        // g[k-1] is read from global memory: round k-1 may lie in the previous staged
        // chunk, and a chunk reload (__syncthreads) must not happen inside tid == 0 code.
        // (from the staged chunk when it holds k-1: a global load here is on the critical path)
        const uint32_t gm1 = k == 0 ? 0u : (k - 1 >= cb && k - 1 < cb + KX_CH) ? (uint32_t)sg[k - 1 - cb]
                                                                               : (uint32_t)__ldg(&g[k - 1]);
        const bool nar_m1 = C && gm1 <= C;
        if (k > 0 && !(nar && nar_m1)) {
            const bool mine = !C && (prev == k - 1) && gprev == 1;
            if (!mine && !dead) {
                if (tid == 0) {
                    // diag 2048 (tests): round 1 waits for one signal too many -> watchdog
                    const uint32_t need = (nar_m1 ? C : gm1) + ((diag & 2048u) && k == 1 ? 1u : 0u);
                    uint32_t spins = 0;
                    SpinWatch wd;
                    while (ld_acquire(&done[k - 1]) < need) {
                        if (++spins > 64) __nanosleep(32);
                        if (wd.expired(const_cast<uint32_t*>(&sc[SC_DEADLOCK]))) { s_dead = 1; break; }
                    }
                    if (trace && b == 0) trace[8 * k + 4] = spins;
                }
                __syncthreads();
                dead = s_dead != 0;
            }
        }
        // Runs of one-CTA rounds: rounds k .. e-1 that are narrow and need one CTA (<= Q
        // transactions each) are executed by the first W warps of CTA 0 alone (W = the
        // run's largest round / 32), thread j taking the round's j-th transaction,
        // separated by __syncwarp() (W = 1) or a named barrier of W warps -- both order the
        // participants' memory accesses -- instead of a 1024-thread __syncthreads; the
        // next round's parameters are loaded before the current one executes.  The run's
        // last round goes through the regular path below (its hand-off to what follows).
        // Other CTAs of the cluster hold no work in these rounds and skip them too.
        if (TAILRUN && nar && gk == 1 && !(diag & 256u) && !dead) {
            // rounds of up to runmax transactions join the run (diag >> 16; 0: one-CTA rounds)
            const uint32_t runmax = min((uint32_t)KB, diag >> 16);
            // the run's end e (first round from k on that is not a one-CTA narrow round, or
            // the staged chunk's end) and its widest round, KB rounds per step in parallel
            // (a serial scan of a ~130-round tail cost ~20 us, profiles/round2_rounds_tm1)
            const uint32_t lim = min(nk, cb + KX_CH - 1);
            if (tid == 0) { s_run[0] = lim; s_run[1] = 0; }
            __syncthreads();
            for (uint32_t base = k; base < lim; base += KB) {
                const uint32_t x = base + tid;
                if (x < lim) {
                    const uint32_t sz = soff[x - cb + 1] - soff[x - cb], gx = sg[x - cb];
                    if (!(C && gx <= C && (gx == 1 || sz <= runmax))) atomicMin(&s_run[0], x);
                }
                __syncthreads();
                if (s_run[0] < base + KB) break;
            }
            const uint32_t e = s_run[0];
            for (uint32_t x = k + tid; x < e; x += KB) atomicMax(&s_run[1], soff[x - cb + 1] - soff[x - cb]);
            __syncthreads();
            const uint32_t wmax = s_run[1];
            __syncthreads();                    // (s_run is rewritten by the next run)
            const uint32_t nthr = min((uint32_t)KB, (wmax + 31) & ~31u);
            if (e >= k + 2) {                   // rounds k .. e-2 in the run, e-1 regular
                if (b == 0 && tid < nthr) {
                    auto ld = [&](uint32_t kk, uint32_t& idx, uint32_t& t, uint32_t* q) {
                        const uint32_t j = soff[kk - cb] + tid;
                        idx = 0xFFFFFFFFu;
                        if (j < soff[kk - cb + 1]) {
                            idx = __ldg(&perm[j]);
                            t = __ldg(&ptype[j]);
#pragma unroll
                            for (int w = 0; w < (PW > 0 ? PW : 1); w += 4) {
                                const uint4 v = __ldg(reinterpret_cast<const uint4*>(pp + (uint64_t)j * PW + w));
                                q[w] = v.x; q[w + 1] = v.y; q[w + 2] = v.z; q[w + 3] = v.w;
                            }
                        }
                    };
                    uint32_t xi, xt = 0, xq[PW > 0 ? PW : 1];
                    ld(k, xi, xt, xq);
                    for (uint32_t kk = k; kk + 1 < e; ++kk) {
                        if (trace && tid == 0) trace[8 * kk] = globaltimer_ns();        // round start
                        uint32_t yi = 0xFFFFFFFFu, yt = 0, yq[PW > 0 ? PW : 1];
                        if (kk + 2 < e) ld(kk + 1, yi, yt, yq);
                        if (xi != 0xFFFFFFFFu) { kx_jitter(diag, kk, b, tid); exec_txn_p<S, SH>(db, xi, xt, xq); }
                        if (yi != 0xFFFFFFFFu) warm_rows<S>(db, yt, yq);      // next round's rows into L2
                        if (nthr == 32) __syncwarp();
                        else asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
                        xi = yi; xt = yt;
#pragma unroll
                        for (int w = 0; w < (PW > 0 ? PW : 1); ++w) xq[w] = yq[w];
                    }
                }
                // the run's writes reach every CTA of the cluster before round e-1 (which
                // may need several of them)
                asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
                k = e - 1;
                bounds(k, lo, hi);
                slice(lo, hi, G(k), lo, hi);
                prefetch(lo, hi);
                prev = k - 1;
                gprev = G(k - 1);
                continue;
            }
        }
        if (trace && tid == 0) {
            const uint64_t now = globaltimer_ns();
            if (b == 0) trace[8 * k] = now;
            atomicMax(reinterpret_cast<unsigned long long*>(&trace[8 * k + 5]), (unsigned long long)now);  // last start
        }
        // take the prefetched slice, then prefetch this CTA's next round
        const uint32_t cidx = nidx, ct = nt;
        uint32_t cp[PW > 0 ? PW : 1];
#pragma unroll
        for (int w = 0; w < (PW > 0 ? PW : 1); ++w) cp[w] = np[w];
        const uint32_t clo = lo, chi = hi;
        // prefetch the next round's slice now only if this CTA takes part in round k+1;
        // a longer scan for its next round happens after it has signalled this one (a
        // CTA must never delay the round others wait for)
        uint32_t k2 = k + 1;
        const bool next_mine = k2 < nk && part(k2);
        if (next_mine) {
            bounds(k2, lo, hi);
            slice(lo, hi, G(k2), lo, hi);
            if (!(diag & 8u)) prefetch(lo, hi);
        }
        if (!WARPX && cidx != 0xFFFFFFFFu && !(diag & 1u) && !dead) {
            const bool tt = trace && (diag & 2u);
            const uint64_t t0 = tt ? globaltimer_ns() : 0;
            kx_jitter(diag, k, b, tid);
            if (PW > 0) exec_txn_p<S, SH>(db, cidx, ct, cp);
            else exec_txn<S, SH>(db, cidx);
            if (tt) {   // slowest transaction of the round: duration << 24 | idx (GPUTX_KSET_DIAG=2)
                const uint64_t d = globaltimer_ns() - t0;
                atomicMax(reinterpret_cast<unsigned long long*>(&trace[8 * k + 3]),
                          (unsigned long long)((d << 24) | cidx));
            }
        }
        if (WARPX && !(diag & 1u) && !dead)
            for (uint32_t j = clo + (tid >> 5); j < chi; j += KB / 32) {
                kx_jitter(diag, k, b, tid & ~31u);
                exec_txn_warp<SH>(db, __ldg(&perm[j]));
            }
        for (uint32_t j = (diag & 1u) || WARPX || dead ? chi : clo + KB + tid; j < chi; j += KB) {
            if (PW > 0) {
                uint32_t q[PW > 0 ? PW : 1];
#pragma unroll
                for (int w = 0; w < (PW > 0 ? PW : 1); w += 4) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(pp + (uint64_t)j * PW + w));
                    q[w] = v.x; q[w + 1] = v.y; q[w + 2] = v.z; q[w + 3] = v.w;
                }
                exec_txn_p<S, SH>(db, __ldg(&perm[j]), __ldg(&ptype[j]), q);
            } else {
                exec_txn<S, SH>(db, __ldg(&perm[j]));
            }
        }
        // the next round's rows into L2 while this round drains (its params have arrived)
        if (PW > 0 && next_mine && nidx != 0xFFFFFFFFu && !(diag & 8u)) warm_rows<S>(db, nt, np);
        if (trace && tid == 0) {
            const uint64_t now = globaltimer_ns();
            if (b == 0) trace[8 * k + 6] = now;                               // CTA 0's work issued
            atomicMax(reinterpret_cast<unsigned long long*>(&trace[8 * k + 7]), (unsigned long long)now);  // last CTA
        }
        if (nar) {
            // Consecutive one-CTA rounds are CTA 0's alone (__syncthreads); otherwise all
            // C CTAs of cluster 0 release their writes to each other and acquire theirs.
            // Every CTA of the cluster takes the same decision from the same schedule.
            const bool solo = gk == 1 && k + 1 < nk && narrow(k + 1) && G(k + 1) == 1;
            if (solo) __syncthreads();
            else asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
            if (k + 1 < nk && !narrow(k + 1) && tid == 0) red_add_release(&done[k], 1u);   // a wide round follows
        } else {
            __syncthreads();
            // without clusters CTA 0 runs every round; for it k2 == k + 1
            const bool next_shared = b > 0 || C || ((k + 1 < nk) && G(k + 1) > 1);
            if (tid == 0 && (gk > 1 || next_shared)) red_add_release(&done[k], 1u);
        }
        if (trace && b == 0 && tid == 0) trace[8 * k + 1] = globaltimer_ns();
        if (!next_mine) {
            while (k2 < nk && !part(k2)) ++k2;
            if (k2 < nk) {
                bounds(k2, lo, hi);
                slice(lo, hi, G(k2), lo, hi);
                if (!(diag & 8u)) prefetch(lo, hi);
            }
        }
        prev = k;
        gprev = gk;
        k = k2;
    }
}

// =====================================================================================
// K-SET with owner-local rounds (DESIGN.md §4 "Owner-local rounds").  Every transaction
// gets an owner warp from its root key (TM-1 subscriber, TPC-B home branch, micro tuple);
// each warp executes ITS transactions k-set by k-set (Property 1 within a k-set, PAPER.md
// :123-125; k-sets in increasing k, §5.3), its rounds separated by __syncwarp().  Nothing
// is global: a transaction whose T-dependency predecessor belongs to
// another warp waits, before it runs, until that warp's progress word says the
// predecessor's k-set is done; every other predecessor is the warp's own, in an earlier
// round.  progress[w] = "all of w's rounds below this value are done" (monotone), written
// only at the end of a round that some other warp waits for.  Waits point to strictly
// smaller k, and all warps are co-resident (cooperative launch), so the warp at the
// smallest pending k can always proceed: no deadlock.
// =====================================================================================
constexpr uint32_t OWN_INF = 0xFFFFFFFFu;
constexpr unsigned long long OWN_GLOBAL = ~0ull;   // wait: every warp's progress >= own k
constexpr int SC_OWNGLOBAL = 39;                    // some transaction waits globally
constexpr uint32_t OWN_WALK = 64;                   // records walked per conflict search

template <int S>
DEV uint32_t own_of(const uint32_t* p, uint32_t nw, uint32_t idx, uint32_t diag) {
    if (diag & 16384u) return (uint32_t)(nbr_hash(idx) % nw);      // tests: arbitrary owners
    if (S == S_TPCB) return p[2] % nw;                               // home branch
    return (uint32_t)(nbr_hash((uint64_t)p[0]) % nw);              // TM-1 subscriber, micro tuple
}

DEV void own_add_wait(unsigned long long* wait, uint32_t idx, uint32_t o, uint32_t need, uint32_t* sc) {
    const unsigned long long v = ((unsigned long long)o << 32) | need;
    const unsigned long long old = atomicCAS(&wait[idx], 0ull, v);
    if (old == 0ull || old == v) return;
    if ((uint32_t)(old >> 32) == o) { atomicMax(&wait[idx], v); return; }   // same warp: the later k
    atomicExch(&wait[idx], OWN_GLOBAL);                                       // two warps: wait for all
    atomicOr(&sc[SC_OWNGLOBAL], 1u);
}

// Cross-owner predecessors from the (item, ts)-sorted records (R/W rule):
// a record conflicts with the earlier records of its item back to (and including) the
// previous write -- a read only with that write.  Predecessors further back are ordered
// before that write, which waited for them itself.  A foreign predecessor p of txn t
// gives t a wait (owner(p), D[p] + 1) and marks p "publish".  More than one foreign warp,
// or a walk longer than OWN_WALK records, makes t wait for every warp (OWN_GLOBAL).
__global__ void __launch_bounds__(256) own_dep_kernel(const uint64_t* __restrict__ keys, const uint32_t* nrec_ptr,
                                                      const uint32_t* __restrict__ own, const uint32_t* __restrict__ D,
                                                      unsigned long long* wait, uint8_t* pub, uint32_t* sc,
                                                      uint32_t diag) {
    const uint32_t nrec = *nrec_ptr;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrec; i += gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        const uint64_t item = key_item(k);
        const uint32_t idx = key_idx(k), m = key_mode(k), o = own[idx];
        uint32_t steps = 0;
        for (uint32_t j = i; j-- > 0;) {
            const uint64_t kj = keys[j];
            if (key_item(kj) != item) break;
            const uint32_t mj = key_mode(kj);
            if (m == 1u || mj == 1u) {
                const uint32_t ij = key_idx(kj), oj = own[ij];
                if (oj != o) {
                    if (diag & 8192u) { atomicExch(&wait[idx], OWN_GLOBAL); atomicOr(&sc[SC_OWNGLOBAL], 1u); }
                    else own_add_wait(wait, idx, oj, D[ij] + 1u, sc);
                    pub[ij] = 1;
                }
            }
            if (mj == 1u) break;
            if (++steps >= OWN_WALK) {
                atomicExch(&wait[idx], OWN_GLOBAL);
                atomicOr(&sc[SC_OWNGLOBAL], 1u);
                break;
            }
        }
    }
}

// Owner-ordered execution arrays: oidx / otype / odep / the first PW parameter words, the
// owner segments oseg[0..nw] and every warp's initial progress (its first k, or INF).
// With the dependency pass, owait[pos] = wait[idx] and bit 31 of odep = pub[idx]: the
// executor's staging is then one level of coalesced loads.
constexpr uint32_t OWN_PUB = 0x80000000u;
template <int PW>
__global__ void __launch_bounds__(256) own_gather_kernel(DevDb db, const uint64_t* __restrict__ skeys, uint32_t n,
                                                         uint32_t nw, const uint32_t* __restrict__ perm,
                                                         const uint32_t* __restrict__ D,
                                                         const unsigned long long* __restrict__ wait,
                                                         const uint8_t* __restrict__ pub, uint32_t* oidx,
                                                         uint8_t* otype, uint32_t* opp, uint32_t* odep,
                                                         unsigned long long* owait, uint32_t* oseg, uint32_t* prog,
                                                         uint32_t* oout) {
    for (uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x; pos < n; pos += gridDim.x * blockDim.x) {
        const uint64_t sk = skeys[pos];
        const uint32_t o = (uint32_t)(sk >> 32), idx = perm[(uint32_t)sk];
        const uint32_t d = D[idx];
        oidx[pos] = idx;
        otype[pos] = db.type[idx];
        odep[pos] = d | (pub && pub[idx] ? OWN_PUB : 0u);
        if (wait) owait[pos] = wait[idx];
        if (oout) oout[pos] = db.out_off[idx];          // packed output offset, staged
        if (PW > 0 && !bulk_failed(db)) {
            const uint32_t* src = db.pw + db.poff[idx];
#pragma unroll
            for (int w = 0; w < PW; w += 4)
                *reinterpret_cast<uint4*>(opp + (uint64_t)pos * PW + w) =
                    make_uint4(src[w], src[w + 1], src[w + 2], src[w + 3]);
        }
        const int64_t prev = pos ? (int64_t)(skeys[pos - 1] >> 32) : -1;
        if ((int64_t)o != prev) {
            for (int64_t q = prev + 1; q < (int64_t)o; ++q) { oseg[q] = pos; prog[q] = OWN_INF; }   // empty owners
            oseg[o] = pos;
            prog[o] = d;
        }
        if (pos == n - 1)
            for (uint32_t q = o + 1; q <= nw; ++q) { oseg[q] = n; if (q < nw) prog[q] = OWN_INF; }
    }
}

// The warp's segment is staged 32 entries at a time in registers, three chunks deep: A
// (being executed), B (landed; its rows warmed into L2 when it became next) and C (in
// flight).  Round d0 = the entries from the cursor on with depth d0 (a prefix: the
// segment is (depth, type)-ordered); lane L takes the round's L-th entry from A or B by
// shuffles, so no load sits between two rounds -- only the round's own memory accesses
// and the __syncwarp() that orders them before the next round's.
template <int S, int PW, bool DEP>
__global__ void __launch_bounds__(256) kset_own_exec_kernel(DevDb db, const uint32_t* __restrict__ oseg,
                                                            const uint32_t* __restrict__ oidx,
                                                            const uint8_t* __restrict__ otype,
                                                            const uint32_t* __restrict__ opp,
                                                            const uint32_t* __restrict__ odep,
                                                            const unsigned long long* __restrict__ owait,
                                                            const uint32_t* __restrict__ oout,
                                                            uint32_t* prog, uint32_t* sc, uint32_t diag) {
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    constexpr int NP = PW > 0 ? PW : 1;
    const uint32_t lane = lane_id();
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    const uint32_t w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t lo = oseg[w], hi = oseg[w + 1];
    if (lo >= hi || bulk_failed(db)) return;
    const bool gmode = DEP && __ldcg(&sc[SC_OWNGLOBAL]) != 0u;
    struct E {
        uint32_t idx, t, d;              // d: depth | OWN_PUB; INF past the segment
        uint32_t oo;                     // packed output offset (OUT_AUTO: fixed stride)
        unsigned long long wt;
        uint32_t q[NP];
    };
    auto load = [&](uint32_t base, E& e) {
        const uint32_t j = base + lane;
        e.idx = OWN_INF; e.t = 0; e.d = OWN_INF; e.wt = 0; e.oo = OUT_AUTO;
#pragma unroll
        for (int x = 0; x < NP; ++x) e.q[x] = 0;
        if (j < hi) {
            e.idx = __ldg(&oidx[j]);
            e.t = __ldg(&otype[j]);
            e.d = __ldg(&odep[j]);
            if (PW > 0) {
#pragma unroll
                for (int x = 0; x < NP; x += 4) {
                    const uint4 v = __ldg(reinterpret_cast<const uint4*>(opp + (uint64_t)j * PW + x));
                    e.q[x] = v.x; e.q[x + 1] = v.y; e.q[x + 2] = v.z; e.q[x + 3] = v.w;
                }
            }
            if (DEP) e.wt = __ldg(&owait[j]);
            if (oout) e.oo = __ldg(&oout[j]);
        }
    };
    // entry (cursor + lane) of the window A|B, by shuffles (every lane takes part)
    auto pick = [&](const E& a, const E& b, uint32_t src, E& x) {
        const uint32_t sl = src & 31u;
        const bool fa = src < 32u;
        uint32_t u, v;
        u = __shfl_sync(FULL, a.idx, sl); v = __shfl_sync(FULL, b.idx, sl); x.idx = fa ? u : v;
        u = __shfl_sync(FULL, a.t, sl);   v = __shfl_sync(FULL, b.t, sl);   x.t = fa ? u : v;
        u = __shfl_sync(FULL, a.d, sl);   v = __shfl_sync(FULL, b.d, sl);   x.d = fa ? u : v;
        u = __shfl_sync(FULL, a.oo, sl);  v = __shfl_sync(FULL, b.oo, sl);  x.oo = fa ? u : v;
        if (DEP) {
            const unsigned long long ua = __shfl_sync(FULL, a.wt, sl), ub = __shfl_sync(FULL, b.wt, sl);
            x.wt = fa ? ua : ub;
        }
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            u = __shfl_sync(FULL, a.q[k], sl); v = __shfl_sync(FULL, b.q[k], sl); x.q[k] = fa ? u : v;
        }
    };
    auto depth_at = [&](const E& a, const E& b, uint32_t p) -> uint32_t {   // uniform p < 64
        const uint32_t u = __shfl_sync(FULL, a.d, p & 31u), v = __shfl_sync(FULL, b.d, p & 31u);
        return (p < 32u ? u : v) & ~OWN_PUB;
    };
    E A, B, C;
    load(lo, A);
    load(lo + 32, B);
    load(lo + 64, C);
    if (B.idx != OWN_INF) warm_rows<S>(db, B.t, B.q);
    uint32_t ca = lo, p = 0;        // window base, cursor offset in it (< 32)
    bool pubr = false;
    uint32_t d0 = depth_at(A, B, 0);
    while (ca + p < hi) {
        E X;
        pick(A, B, p + lane, X);
        const uint32_t xd = X.d & ~OWN_PUB;
        const uint32_t cnt = __popc(__ballot_sync(FULL, xd == d0));       // >= 1; prefix of the window
        if (lane < cnt) {
            if (DEP && X.wt) {
                SpinWatch wd;
                if (X.wt == OWN_GLOBAL) {
                    for (uint32_t q = 0; q < nw; ++q) {
                        if (q == w) continue;
                        while (ld_acquire(&prog[q]) < d0)
                            if (wd.expired(&sc[SC_DEADLOCK])) break;
                    }
                } else {
                    const uint32_t ow = (uint32_t)(X.wt >> 32), need = (uint32_t)X.wt;
                    uint32_t spins = 0;
                    while (ld_acquire(&prog[ow]) < need) {
                        if (++spins > 16) __nanosleep(64);
                        if (wd.expired(&sc[SC_DEADLOCK])) break;
                    }
                }
            }
            kx_jitter(diag, d0, w, lane);
            exec_txn_p<S, false>(db, X.idx, X.t, X.q, X.oo);
        }
        if (DEP) pubr |= __ballot_sync(FULL, lane < cnt && (X.d & OWN_PUB)) != 0u;
        p += cnt;
        if (p >= 32u) {                  // A consumed: slide the window
            A = B;
            B = C;
            ca += 32;
            p -= 32;
            load(ca + 64, C);
            if (B.idx != OWN_INF) warm_rows<S>(db, B.t, B.q);
        }
        const uint32_t dn = ca + p < hi ? depth_at(A, B, p) : OWN_INF;
        if (dn != d0) {                  // round d0 of this warp ends
            const bool publish = DEP && (pubr || gmode);
            if (publish) __threadfence();          // each lane's writes, at gpu scope
            __syncwarp();                          // ... and before the warp's next round
            if (publish && lane == 0) st_release(&prog[w], dn);
            pubr = false;
            d0 = dn;
        }
    }
}

// Owner segments (and every warp's initial progress) straight from the owner-sorted keys
// (owner << 32 | position in the (depth, type) order): for the executor that stages its
// own entries through the perm (kset_own_pipe_kernel), no gather pass.
__global__ void __launch_bounds__(256) own_bounds_kernel(const uint64_t* __restrict__ skeys, uint32_t n,
                                                         uint32_t nw, const uint32_t* __restrict__ perm,
                                                         const uint32_t* __restrict__ D, uint32_t* oseg,
                                                         uint32_t* prog) {
    // one pass over the owner-sorted keys: position i starts the segments of the owners in
    // (owner(i-1), owner(i)] (empty ones included), so every oseg[w] / prog[w] is written once
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += gridDim.x * blockDim.x) {
        const uint32_t prev = i ? (uint32_t)(__ldg(&skeys[i - 1]) >> 32) + 1u : 0u;
        const uint64_t k = i < n ? __ldg(&skeys[i]) : 0ull;
        const uint32_t cur = i < n ? (uint32_t)(k >> 32) : nw;
        for (uint32_t w = prev; w <= cur; ++w) {
            oseg[w] = i;
            if (w < nw) prog[w] = w == cur ? D[perm[(uint32_t)k]] : OWN_INF;
        }
    }
}

// kset_own_exec_kernel without the gather pass: the warp stages its own entries in four
// register stages a chunk of 32 apart -- owner-sorted key -> perm -> (type, offset, depth,
// output offset, wait) -> parameters -- so every stage's loads have a chunk of rounds to land
// (the gather kernel's random reads, 44 us on TM-1, are spread over the rounds instead).
template <int S, int PW, bool DEP>
__global__ void __launch_bounds__(256) kset_own_pipe_kernel(DevDb db, const uint32_t* __restrict__ oseg,
                                                            const uint64_t* __restrict__ skeys,
                                                            const uint32_t* __restrict__ perm,
                                                            const uint32_t* __restrict__ D,
                                                            const unsigned long long* __restrict__ wait,
                                                            const uint8_t* __restrict__ pub,
                                                            uint32_t* prog, uint32_t* sc, uint32_t diag) {
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    constexpr int NP = PW > 0 ? PW : 1;
    const uint32_t lane = lane_id();
    const uint32_t nw = gridDim.x * (blockDim.x >> 5);
    const uint32_t w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t lo = oseg[w], hi = oseg[w + 1];
    if (lo >= hi || bulk_failed(db)) return;
    const bool gmode = DEP && __ldcg(&sc[SC_OWNGLOBAL]) != 0u;
    struct E {
        uint32_t idx, t, d, oo;          // d: depth | OWN_PUB; INF past the segment
        unsigned long long wt;
        uint32_t q[NP];
    };
    struct Meta { uint32_t idx, t, o, d, oo; unsigned long long wt; };
    // stage loads (lane l: entry base + l)
    auto st_key = [&](uint32_t base) -> uint32_t {          // -> position in perm, or INF
        const uint32_t j = base + lane;
        return j < hi ? (uint32_t)__ldg(&skeys[j]) : OWN_INF;
    };
    auto st_idx = [&](uint32_t pos) -> uint32_t { return pos != OWN_INF ? __ldg(&perm[pos]) : OWN_INF; };
    auto st_meta2 = [&](uint32_t idx, const uint32_t* Dd, Meta& m) {
        m.idx = idx; m.t = 0; m.o = 0; m.d = OWN_INF; m.oo = OUT_AUTO; m.wt = 0;
        if (idx == OWN_INF) return;
        m.t = db.type[idx];
        m.o = db.poff[idx];
        m.d = Dd[idx] | (DEP && pub[idx] ? OWN_PUB : 0u);
        m.oo = db.out_off ? db.out_off[idx] : OUT_AUTO;
        if (DEP) m.wt = wait[idx];
    };
    auto st_full = [&](const Meta& m, E& e) {
        e.idx = m.idx; e.t = m.t; e.d = m.d; e.oo = m.oo; e.wt = m.wt;
#pragma unroll
        for (int x = 0; x < NP; ++x) e.q[x] = 0;
        if (m.idx == OWN_INF || PW == 0) return;
        const uint32_t* p = db.pw + m.o;
#pragma unroll
        for (int x = 0; x < NP; ++x) e.q[x] = p[x];
    };
    // prologue: chunks 0, 1 complete; 2 meta; 3 idx; 4 key
    E A, B;
    Meta M2;
    uint32_t I3, K4;
    {
        Meta m0, m1;
        st_meta2(st_idx(st_key(lo)), D, m0);
        st_meta2(st_idx(st_key(lo + 32)), D, m1);
        st_full(m0, A);
        st_full(m1, B);
        st_meta2(st_idx(st_key(lo + 64)), D, M2);
        I3 = st_idx(st_key(lo + 96));
        K4 = st_key(lo + 128);
    }
    E C;
    st_full(M2, C);                              // chunk 2's parameters in flight
    st_meta2(I3, D, M2);                         // chunk 3's metadata in flight
    I3 = st_idx(K4);                             // chunk 4's perm entries in flight
    K4 = st_key(lo + 160);                       // chunk 5's keys in flight
    if (PW > 0 && B.idx != OWN_INF) warm_rows<S>(db, B.t, B.q);
    auto pick = [&](const E& a, const E& b, uint32_t src, E& x) {
        const uint32_t sl = src & 31u;
        const bool fa = src < 32u;
        uint32_t u, v;
        u = __shfl_sync(FULL, a.idx, sl); v = __shfl_sync(FULL, b.idx, sl); x.idx = fa ? u : v;
        u = __shfl_sync(FULL, a.t, sl);   v = __shfl_sync(FULL, b.t, sl);   x.t = fa ? u : v;
        u = __shfl_sync(FULL, a.d, sl);   v = __shfl_sync(FULL, b.d, sl);   x.d = fa ? u : v;
        u = __shfl_sync(FULL, a.oo, sl);  v = __shfl_sync(FULL, b.oo, sl);  x.oo = fa ? u : v;
        if (DEP) {
            const unsigned long long ua = __shfl_sync(FULL, a.wt, sl), ub = __shfl_sync(FULL, b.wt, sl);
            x.wt = fa ? ua : ub;
        }
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            u = __shfl_sync(FULL, a.q[k], sl); v = __shfl_sync(FULL, b.q[k], sl); x.q[k] = fa ? u : v;
        }
    };
    auto depth_at = [&](const E& a, const E& b, uint32_t p) -> uint32_t {
        const uint32_t u = __shfl_sync(FULL, a.d, p & 31u), v = __shfl_sync(FULL, b.d, p & 31u);
        return (p < 32u ? u : v) & ~OWN_PUB;
    };
    uint32_t ca = lo, p = 0;
    bool pubr = false;
    uint32_t d0 = depth_at(A, B, 0);
    while (ca + p < hi) {
        E X;
        pick(A, B, p + lane, X);
        const uint32_t xd = X.d & ~OWN_PUB;
        const uint32_t cnt = __popc(__ballot_sync(FULL, xd == d0));
        if (lane < cnt) {
            if (DEP && X.wt) {
                SpinWatch wd;
                if (X.wt == OWN_GLOBAL) {
                    for (uint32_t q = 0; q < nw; ++q) {
                        if (q == w) continue;
                        while (ld_acquire(&prog[q]) < d0)
                            if (wd.expired(&sc[SC_DEADLOCK])) break;
                    }
                } else {
                    const uint32_t ow = (uint32_t)(X.wt >> 32), need = (uint32_t)X.wt;
                    uint32_t spins = 0;
                    while (ld_acquire(&prog[ow]) < need) {
                        if (++spins > 16) __nanosleep(64);
                        if (wd.expired(&sc[SC_DEADLOCK])) break;
                    }
                }
            }
            kx_jitter(diag, d0, w, lane);
            exec_txn_p<S, false>(db, X.idx, X.t, X.q, X.oo);
        }
        if (DEP) pubr |= __ballot_sync(FULL, lane < cnt && (X.d & OWN_PUB)) != 0u;
        p += cnt;
        if (p >= 32u) {                          // A consumed: advance every stage by a chunk
            A = B;
            B = C;
            ca += 32;
            p -= 32;
            st_full(M2, C);
            st_meta2(I3, D, M2);
            I3 = st_idx(K4);
            K4 = st_key(ca + 160);
            if (PW > 0 && B.idx != OWN_INF) warm_rows<S>(db, B.t, B.q);
        }
        const uint32_t dn = ca + p < hi ? depth_at(A, B, p) : OWN_INF;
        if (dn != d0) {
            const bool publish = DEP && (pubr || gmode);
            if (publish) __threadfence();
            __syncwarp();
            if (publish && lane == 0) st_release(&prog[w], dn);
            pubr = false;
            d0 = dn;
        }
    }
}

// =====================================================================================
// Spine-streaming rank (DESIGN.md §4 "Spine-streaming rank"): every transaction of TPC-B,
// TPC-C and micro writes one *spine* item that only its own kind writes (TPC-B its branch
// balance, TPC-C NewOrder its district's next order id and Payment its warehouse's YTD,
// micro its tuple), so the transactions sharing a spine item form a chain in ts order and
// D[t] = max(D[previous chain member] + 1, max over t's other conflicting predecessors p of
// D[p] + 1) -- the longest-path depth of the T-dependency graph computed
// in one streaming pass per chain.  The other predecessors ("links") come from the
// (item, ts)-sorted records: a read conflicts with the previous write of its item; a
// write with the reads since the previous write (each of which is after that write), or
// with the previous write if there are none.  One warp walks a chain 32 members at a
// time (max-plus scan), writing each member's depth as soon as its links' depths exist.
// =====================================================================================
constexpr uint32_t SP_UNSET = 0xFFFFFFFFu;

template <int S> DEV uint32_t spine_j() { return S == S_TPCB ? 2u : 0u; }   // footprint position

// segmented max of W positions: per record (head of its item group, position of the
// latest write up to it); identity (0, -1)
struct SegMax {
    uint32_t f;
    int32_t v;
};
struct OpSegMax {
    static DEV SegMax identity() { return SegMax{0u, -1}; }
    static DEV SegMax combine(SegMax a, SegMax b) { return SegMax{a.f | b.f, b.f ? b.v : max(a.v, b.v)}; }
};

// lastw[i] encodes what precedes record i in its item group: -1 = i is the group's first
// record; 2w + 1 = the latest write before i is at w; 2g = no write before i, the group
// starts at g (a segmented max-scan of head / write markers).  sp[t] = t's spine item.
template <int S>
__global__ void __launch_bounds__(SC_THREADS) lastw_kernel(const uint64_t* __restrict__ keys, const uint32_t* n_ptr,
                                                           LookBack<SegMax> lb, uint32_t epoch, uint32_t* ticket,
                                                           int32_t* lastw, uint32_t* sp) {
    __shared__ SegMax sm[8];
    __shared__ uint32_t s_tile;
    __shared__ SegMax s_pre;
    const uint32_t n = *n_ptr;
    const uint32_t ntiles = (n + SC_TILE - 1) / SC_TILE;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    if (tile >= ntiles) return;
    const uint64_t b = (uint64_t)tile * SC_TILE + threadIdx.x * SC_ITEMS;
    SegMax e[SC_ITEMS];
    SegMax agg = OpSegMax::identity();
    uint64_t prev_item = b > 0 && b - 1 < n ? key_item(keys[b - 1]) : ~0ull;
    // the thread's 16 keys (128 B, 128-B aligned) as eight 16-B loads when all are in range
    const bool full = b + SC_ITEMS <= n;
    uint64_t kv[SC_ITEMS];
    if (full) {
#pragma unroll
        for (int q = 0; q < SC_ITEMS / 2; ++q) {
            const ulonglong2 x = reinterpret_cast<const ulonglong2*>(keys + b)[q];
            kv[2 * q] = x.x; kv[2 * q + 1] = x.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < SC_ITEMS; ++k) kv[k] = b + k < n ? keys[b + k] : 0ull;
    }
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        e[k] = OpSegMax::identity();
        if (b + k < n) {
            const uint64_t key = kv[k];
            const uint64_t it = key_item(key);
            const bool head = b + k == 0 || it != prev_item;
            e[k] = SegMax{head ? 1u : 0u, key_mode(key) == 1u ? (int32_t)(2 * (b + k) + 1) : head ? (int32_t)(2 * (b + k)) : -1};
            if (key_j(key) == spine_j<S>()) sp[key_idx(key)] = (uint32_t)it;
            prev_item = it;
        }
        agg = OpSegMax::combine(agg, e[k]);
    }
    SegMax tot;
    SegMax ex = block_scan_excl<SegMax, OpSegMax>(agg, tot, sm);
    if (warp_id() == 0) {
        SegMax pre = lookback_warp<SegMax, OpSegMax>(lb, tile, epoch, tot);
        if (lane_id() == 0) s_pre = pre;
    }
    __syncthreads();
    SegMax run = OpSegMax::combine(s_pre, ex);
    int32_t lv[SC_ITEMS];
#pragma unroll
    for (int k = 0; k < SC_ITEMS; ++k) {
        lv[k] = e[k].f ? -1 : run.v;                            // exclusive (a head starts fresh)
        run = OpSegMax::combine(run, e[k]);
    }
    if (full) {
#pragma unroll
        for (int q = 0; q < SC_ITEMS / 4; ++q)
            reinterpret_cast<int4*>(lastw + b)[q] = make_int4(lv[4 * q], lv[4 * q + 1], lv[4 * q + 2], lv[4 * q + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < SC_ITEMS; ++k)
            if (b + k < n) lastw[b + k] = lv[k];
    }
}

// links of record i (not its transaction's spine record): calls f(idx of predecessor)
template <class F>
DEV void sp_links(const uint64_t* __restrict__ keys, const int32_t* __restrict__ lastw, uint32_t i, F f) {
    const uint64_t k = keys[i];
    const int32_t enc = lastw[i];
    if (enc < 0) return;                            // first access of its item
    const bool has_w = enc & 1;
    const int64_t lw = has_w ? (enc - 1) / 2 : -1;  // latest write, or none
    const int64_t lo = has_w ? lw + 1 : enc / 2;    // first read after it (or the group start)
    if (key_mode(k) == 1u) {                        // a write: the reads since the last write, else it
        for (int64_t j = lo; j < (int64_t)i; ++j) f(key_idx(keys[j]));
        if (lo == (int64_t)i && has_w) f(key_idx(keys[lw]));
    } else if (has_w) {                             // a read: the last write
        f(key_idx(keys[lw]));
    }
}

// (a predecessor in t's own chain is implied by the chain order: not a link)
template <int S>
__global__ void __launch_bounds__(256) sp_count_kernel(const uint64_t* __restrict__ keys, const uint32_t* nrec_ptr,
                                                       const int32_t* __restrict__ lastw,
                                                       const uint32_t* __restrict__ sp, uint32_t* lcnt) {
    const uint32_t nrec = *nrec_ptr;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrec; i += gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        if (key_j(k) == spine_j<S>()) continue;     // the chain itself
        const uint32_t me = sp[key_idx(k)];
        uint32_t c = 0;
        sp_links(keys, lastw, i, [&](uint32_t p) { c += sp[p] != me; });
        if (c) atomicAdd(&lcnt[key_idx(k)], c);
    }
}

template <int S>
__global__ void __launch_bounds__(256) sp_fill_kernel(const uint64_t* __restrict__ keys, const uint32_t* nrec_ptr,
                                                      const int32_t* __restrict__ lastw,
                                                      const uint32_t* __restrict__ sp,
                                                      const uint32_t* __restrict__ loff, uint32_t* lfill,
                                                      uint32_t* links, uint32_t* heads, uint32_t* nheads,
                                                      uint8_t* cpub) {
    const uint32_t nrec = *nrec_ptr;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrec; i += gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        const uint32_t t = key_idx(k);
        if (key_j(k) == spine_j<S>()) {             // chain heads (order irrelevant)
            if (i == 0 || key_item(keys[i - 1]) != key_item(k)) heads[atomicAdd(nheads, 1u)] = i;
            continue;
        }
        const uint32_t me = sp[t];
        sp_links(keys, lastw, i, [&](uint32_t p) {
            if (sp[p] != me) {
                links[loff[t] + atomicAdd(&lfill[t], 1u)] = p;
                if (cpub) cpub[p] = 1;                  // (chain executor: p publishes)
            }
        });
    }
}

// One warp per chain (co-resident cooperative grid; a warp owning several chains cycles
// through them, advancing each as far as its links allow: the unprocessed transaction of
// smallest ts always can advance, so the walk terminates).  Chain state in global memory.
template <int S>
__global__ void __launch_bounds__(256) sp_walk_kernel(const uint64_t* __restrict__ keys, const uint32_t* nrec_ptr,
                                                      const uint32_t* __restrict__ heads, const uint32_t* nheads_ptr,
                                                      const uint32_t* __restrict__ loff,
                                                      const uint32_t* __restrict__ links, uint32_t* D,
                                                      uint32_t* cur, int32_t* last, uint32_t* sc) {
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    const uint32_t lane = lane_id();
    const uint32_t nw = gridDim.x * (blockDim.x >> 5), w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t nrec = *nrec_ptr, nh = *nheads_ptr;
    if (w == 0 && lane == 0) sc[SC_PASSES] = 1;          // one streaming pass (stats)
    if (w >= nh) return;
    SpinWatch wd;
    uint32_t left = 0;                                   // chains of this warp not finished
    for (uint32_t c = w; c < nh; c += nw) {
        if (lane == 0) { cur[c] = heads[c]; last[c] = -1; }
        ++left;
    }
    __syncwarp();
    uint32_t idle = 0;
    while (left) {
        bool progress = false;
        for (uint32_t c = w; c < nh; c += nw) {
            uint32_t p = __ldcg(&cur[c]);
            if (p == SP_UNSET) continue;                 // finished
            const uint64_t item = key_item(keys[heads[c]]);
            int32_t ld = __ldcg(&last[c]);
            const bool alone = nh <= nw;                 // this warp's only chain: wait in place
            // software pipeline over the chain's chunks: the keys of chunk i+2 and the link
            // ranges of chunk i+1 are in flight while chunk i is resolved, so a chunk costs its
            // scan (and its links' depth loads), not a keys -> link-range round trip chain
            auto ldk = [&](uint32_t r) -> uint64_t {
                if (r >= nrec) return ~0ull;
                const uint64_t k = keys[r];
                return key_item(k) == item ? k : ~0ull;
            };
            auto ldx = [&](uint64_t k, uint32_t& x, uint32_t& xe) {
                x = xe = 0;
                if (k != ~0ull) { const uint32_t t = key_idx(k); x = loff[t]; xe = loff[t + 1]; }
            };
            uint64_t kc = ldk(p + lane), kn = ldk(p + 32 + lane);
            uint32_t xc, xec;
            ldx(kc, xc, xec);
            while (true) {
                const bool mem = kc != ~0ull;
                const uint32_t t = mem ? key_idx(kc) : 0u;
                const uint32_t memmask = __ballot_sync(FULL, mem);
                const uint32_t clen = memmask == FULL ? 32u : __ffs(~memmask) - 1;   // members in this chunk
                if (clen == 0) {                         // chain done
                    if (lane == 0) cur[c] = SP_UNSET;
                    --left;
                    progress = true;
                    break;
                }
                const uint64_t kn2 = clen == 32 ? ldk(p + 64 + lane) : ~0ull;
                uint32_t xn = 0, xen = 0;
                if (clen == 32) ldx(kn, xn, xen);
                // e = max over links of D[p] + 1 (or -1); a lane is blocked while some link's depth
                // is not there yet.  Lanes [s0, clen) of the chunk are pending; a blocked chunk is
                // re-polled in place (only the unresolved links), not reloaded: a hop between two
                // chains then costs one L2 round trip
                uint32_t x = lane < clen ? xc : 0u, xe = lane < clen ? xec : 0u;
                int32_t e = -1;
                uint32_t s0 = 0, spins = 0;
                while (true) {
                    bool blocked = false;
                    if (lane >= s0 && lane < clen) {
                        for (; x < xe; ++x) {
                            const uint32_t dp = __ldcg(&D[__ldg(&links[x])]);
                            if (dp == SP_UNSET) { blocked = true; break; }
                            e = max(e, (int32_t)dp + 1);
                        }
                    }
                    const uint32_t bm = __ballot_sync(FULL, blocked);
                    const uint32_t k = bm ? __ffs(bm) - 1 : clen;                   // lanes [s0, k) proceed
                    if (k > s0) {
                        // D_l = max(ld + 1 + (l - s0), max_{s0 <= m <= l} (e_m - m) + l)   (max-plus scan)
                        int32_t v = (lane >= s0 && lane < k) ? e - (int32_t)lane : -0x3FFFFFFF;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int32_t y = __shfl_up_sync(FULL, v, o);
                            if ((int)lane >= o) v = max(v, y);
                        }
                        const int32_t dl = max(ld + 1 + (int32_t)lane - (int32_t)s0, v + (int32_t)lane);
                        if (lane >= s0 && lane < k) __stcg(&D[t], (uint32_t)dl);
                        ld = __shfl_sync(FULL, dl, k - 1);
                        s0 = k;
                        progress = true;
                        spins = 0;
                    }
                    if (s0 == clen) break;
                    if (!alone && ++spins > 4) break;    // other chains of this warp may unblock it
                    if (alone && ++spins > 64) {
                        __nanosleep(64);
                        if (wd.expired(&sc[SC_DEADLOCK])) break;
                    }
                }
                p += s0;
                if (s0 < clen) break;                    // blocked: yield (or give up on the watchdog)
                if (clen < 32) {                         // ended inside this chunk: chain done
                    if (lane == 0) cur[c] = SP_UNSET;
                    --left;
                    break;
                }
                kc = kn; xc = xn; xec = xen; kn = kn2;
            }
            if (lane == 0 && __ldcg(&cur[c]) != SP_UNSET) { cur[c] = p; last[c] = ld; }
            __syncwarp();
        }
        if (!progress) {
            if (++idle > 8) __nanosleep(100);
            if (wd.expired(&sc[SC_DEADLOCK])) return;
        } else {
            idle = 0;
        }
    }
}

// =====================================================================================
// K-SET over spine chains (TPC-B; DESIGN.md §4 "Chain owners").  Along a spine chain the
// depth strictly increases (each member conflicts with the previous one), so a chain owns
// exactly one transaction of each of its k-sets: owner-local rounds with the chain as the
// owner are the chain's members in order, one per round, and a round of one transaction
// is ordered after the previous one by the executing thread's program order -- no
// barrier at all.  One warp per chain: lane 0 executes the members; all 32 lanes stage
// them 32 at a time, four chunks ahead, each stage a chunk after the one it depends on
// (keys -> type / offset / links / publish flag -> parameters and output offset -> account
// rows warmed into L2), so lane 0 never waits on metadata.  Before a member runs, lane 0
// waits for the members of OTHER chains it depends on (the spine rank's links: done[p] ==
// epoch, acquire); a member another chain waits for publishes done[t] (release) after it.
// =====================================================================================
constexpr uint32_t CHAIN_NO_RUNS = 1u << 15;      // (engine-set diag bit: GPUTX_CHAIN_RUNS=0)
template <int S>
__global__ void __launch_bounds__(128) kset_chain_exec_kernel(DevDb db, const uint64_t* __restrict__ keys,
                                                              const uint32_t* nrec_ptr,
                                                              const uint32_t* __restrict__ heads,
                                                              const uint32_t* nheads_ptr,
                                                              const uint32_t* __restrict__ loff,
                                                              const uint32_t* __restrict__ links,
                                                              const uint8_t* __restrict__ cpub, uint32_t* done,
                                                              uint32_t epoch, uint32_t* sc, uint32_t diag) {
    constexpr int PW = 4;
    constexpr uint32_t FULL = 0xFFFFFFFFu;
    constexpr uint64_t NONE = ~0ull;
    const uint32_t lane = lane_id();
    const uint32_t c = blockIdx.x * (blockDim.x >> 5) + warp_id();
    const uint32_t nh = *nheads_ptr, nrec = *nrec_ptr;
    if (c >= nh || bulk_failed(db)) return;
    const uint32_t lo = heads[c];
    const uint64_t item = key_item(__ldg(&keys[lo]));
    // stage registers of this lane's member in each chunk
    struct Meta { uint32_t idx, t, o, la, lb, pb, oo; };
    struct Full { uint32_t idx, t, la, lb, pb, oo; uint32_t q[PW]; };
    auto load_key = [&](uint32_t base) -> uint64_t {
        const uint32_t j = base + lane;
        if (j >= nrec) return NONE;
        const uint64_t k = __ldg(&keys[j]);
        return key_item(k) == item ? k : NONE;
    };
    auto load_meta = [&](uint64_t k, Meta& m) {
        m.idx = OWN_INF;
        if (k == NONE) return;
        const uint32_t x = key_idx(k);
        m.idx = x; m.t = db.type[x]; m.o = db.poff[x]; m.la = loff[x]; m.lb = loff[x + 1]; m.pb = cpub[x];
        m.oo = db.out_off ? db.out_off[x] : OUT_AUTO;
    };
    auto load_full = [&](const Meta& m, Full& f) {
        f.idx = m.idx; f.t = m.t; f.la = m.la; f.lb = m.lb; f.pb = m.pb; f.oo = m.oo;
        if (m.idx == OWN_INF) return;
        const uint4 v = *reinterpret_cast<const uint4*>(db.pw + m.o);   // (TPC-B: 4 words, 16-B aligned)
        f.q[0] = v.x; f.q[1] = v.y; f.q[2] = v.z; f.q[3] = v.w;
    };
    // chunk b (relative) = members [lo + 32b, lo + 32b + 32)
    Full E, P1, P2;
    Meta M;
    uint64_t K;
    {
        const uint64_t k0 = load_key(lo), k1 = load_key(lo + 32), k2 = load_key(lo + 64), k3 = load_key(lo + 96);
        Meta m0, m1, m2;
        load_meta(k0, m0); load_meta(k1, m1); load_meta(k2, m2); load_meta(k3, M);
        load_full(m0, E); load_full(m1, P1); load_full(m2, P2);
        K = load_key(lo + 128);
        if (E.idx != OWN_INF && !(diag & 8u)) warm_rows<S>(db, E.t, E.q);
        if (P1.idx != OWN_INF && !(diag & 8u)) warm_rows<S>(db, P1.t, P1.q);
    }
    SpinWatch wd;
    uint32_t len = 0, base = lo;
    while (true) {
        const uint32_t valid = __ballot_sync(FULL, E.idx != OWN_INF);       // a prefix of the chunk
        const uint32_t cnt = __popc(valid);
        // TPC-B deposit runs: a run of deposits (type 0) none of which but the first waits for
        // another chain, on pairwise distinct accounts, executes lane-parallel -- lane l runs
        // member l of the chunk (its staged registers).  No member of a run reads anything
        // another member of the run writes: the accounts differ, teller and branch take
        // reductions (no deposit reads them), history rows are the transactions' own; only
        // the first member waits for other chains (before its own load), and each member
        // publishes (release) after its own account store, which is all its waiter reads.
        // Consecutive runs are ordered by __syncwarp.  Per member the chain was one dependent
        // account load (~0.6 us); a run of up to 32 pays it once.
        const uint32_t okl = __ballot_sync(FULL, S == S_TPCB && E.idx != OWN_INF && E.t == 0u && E.la == E.lb);
        const uint32_t dep0 = __ballot_sync(FULL, S == S_TPCB && E.idx != OWN_INF && E.t == 0u);
        for (uint32_t m = 0; m < cnt;) {
            if (S == S_TPCB && !(diag & (1u | CHAIN_NO_RUNS)) && (dep0 >> m & 1u)) {
                const bool inr = lane >= m && lane < cnt;
                const uint32_t peers = __match_any_sync(FULL, inr ? E.q[0] : 0xFFFFFFFFu - lane);
                const uint32_t dup = __ballot_sync(FULL, inr && (peers & lanemask_lt() & ~((1u << m) - 1u)) != 0u);
                uint32_t stop = ~(okl | (1u << m)) | dup;           // first member that ends the run
                stop &= ~((2u << m) - 1u);                          // (only members after m)
                const uint32_t end = min(cnt, stop ? (uint32_t)(__ffs(stop) - 1) : 32u);
                if (lane >= m && lane < end) {
                    if (lane == m) {
                        for (uint32_t x = E.la; x < E.lb; ++x) {     // the first member's predecessors
                            const uint32_t p = __ldg(&links[x]);
                            uint32_t spins = 0;
                            while (ld_acquire(&done[p]) != epoch) {
                                if (++spins > 8) __nanosleep(64);
                                if (wd.expired(&sc[SC_DEADLOCK])) break;
                            }
                        }
                    }
                    kx_jitter(diag, len + lane, c, 0);
                    int64_t* acc = COL(int64_t, B_ACC);
                    const int64_t nv = ldm(&acc[E.q[0]]) + (int32_t)E.q[3];
                    tpcb_home(db, E.idx, E.q, false);
                    stm(&acc[E.q[0]], nv);
                    *reinterpret_cast<int64_t*>(out_rec<8>(db, E.idx, E.oo)) = nv;
                    if (E.pb) st_release(&done[E.idx], epoch);
                }
                __syncwarp();
                m = end;
                continue;
            }
            const uint32_t idx = __shfl_sync(FULL, E.idx, m), t = __shfl_sync(FULL, E.t, m);
            const uint32_t la = __shfl_sync(FULL, E.la, m), lb = __shfl_sync(FULL, E.lb, m);
            const uint32_t pb = __shfl_sync(FULL, E.pb, m), oo = __shfl_sync(FULL, E.oo, m);
            uint32_t q[PW];
#pragma unroll
            for (int w = 0; w < PW; ++w) q[w] = __shfl_sync(FULL, E.q[w], m);
            if (lane == 0) {
                for (uint32_t x = la; x < lb; ++x) {          // predecessors in other chains
                    const uint32_t p = __ldg(&links[x]);
                    uint32_t spins = 0;
                    while (ld_acquire(&done[p]) != epoch) {
                        if (++spins > 8) __nanosleep(64);
                        if (wd.expired(&sc[SC_DEADLOCK])) break;
                    }
                }
                kx_jitter(diag, len + m, c, 0);
                if (!(diag & 1u)) exec_txn_p<S, false>(db, idx, t, q, oo);   // diag 1: skip bodies (timing)
                if (pb) st_release(&done[idx], epoch);
            }
            __syncwarp();
            ++m;
        }
        len += cnt;
        if (cnt < 32) break;                                  // the chain ended in this chunk
        // rotate the stages: each register set is consumed a chunk after its loads were issued
        base += 32;
        E = P1;
        P1 = P2;
        // the account rows a chunk ahead into L2 (8 members ahead, per member: 2.94 vs 2.60 ms)
        if (P1.idx != OWN_INF && !(diag & 8u)) warm_rows<S>(db, P1.t, P1.q);
        load_full(M, P2);
        load_meta(K, M);
        K = load_key(base + 128);
    }
    if (lane == 0) atomicMax(&sc[SC_MAXCHAIN], len);
}

// =====================================================================================
// PART
// =====================================================================================
template <int S>
__global__ void __launch_bounds__(256) frag_count_kernel(DevDb db, uint32_t* cnt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < db.n; i += gridDim.x * blockDim.x)
        cnt[i] = fragments_local<S>(db, i, nullptr);
}
template <int S>
__global__ void __launch_bounds__(256) frag_emit_kernel(DevDb db, const uint32_t* off, uint64_t* keys) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < db.n; i += gridDim.x * blockDim.x)
        fragments_local<S>(db, i, keys + off[i]);
}
// c of Algorithm 1: transactions whose fragments span > 1 partition
template <int S>
__global__ void __launch_bounds__(256) cross_count_kernel(DevDb db, uint32_t* dst) {
    uint32_t c = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < db.n; i += gridDim.x * blockDim.x)
        c += fragments<S>(db, i, nullptr) > 1;
    c = block_sum_u32(c);
    if (threadIdx.x == 0 && c) atomicAdd(dst, c);
}
__global__ void __launch_bounds__(256) count_gt1_kernel(const uint32_t* cnt, uint32_t n, uint32_t* dst) {
    uint32_t c = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) c += cnt[i] > 1;
    c = block_sum_u32(c);
    if (threadIdx.x == 0 && c) atomicAdd(dst, c);
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
// TPC-C: one warp per partition; a whole-transaction fragment runs as tpcc_txn_warp,
// split fragments (remote lines / customer) on lane 0
// the rows a TPC-C transaction will touch, prefetched into L2 by its warp (lane l: the
// stock and item rows of line l; lane 31: the district; Payment: lane 0, the customer)
DEV void tpcc_warm_warp(const DevDb& db, uint32_t t, const uint32_t* q) {
    const uint32_t lane = lane_id();
    const uint32_t D = db.dims[1], C = db.dims[2], I = db.dims[3];
    const uint32_t w = q[0], dd = q[1];
    if (t == 0) {
        const uint32_t cnt = min(q[3], 15u);
        if (lane < cnt) {
            const uint32_t it = q[4 + 3 * lane], sw = q[5 + 3 * lane];
            if (it < I) {
                l2_warm(&COL(const int32_t, C_S_QTY)[(uint64_t)sw * I + it]);
                l2_warm(&COL(const int32_t, C_I_PRICE)[it]);
            }
        }
        if (lane == 31) l2_warm(&COL(const uint32_t, C_D_NEXT)[(uint64_t)w * D + dd]);
    } else if (lane == 0 && q[4] != 2) {
        l2_warm(&COL(const int64_t, C_C_BAL)[((uint64_t)q[2] * D + q[3]) * C + q[5]]);
    }
}

__global__ void __launch_bounds__(128) part_exec_warp_kernel(DevDb db, const uint64_t* __restrict__ frags,
                                                             const uint32_t* __restrict__ part_off, uint32_t nparts,
                                                             uint32_t* sc) {
    const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (p >= nparts) return;                                   // warp-uniform
    const uint32_t lo = part_off[p], hi = part_off[p + 1];
    const bool sh = db.ts != nullptr;
    const uint32_t lane = lane_id();
    // L2 warming pipeline over the serial chain (cf. part_exec_kernel): while fragment j
    // executes, the parameter words of j+2 and the rows of j+1 (district / stock / item /
    // customer, from its already-warm parameters) are prefetched into L2
    constexpr uint64_t NONE = ~0ull;
    auto key = [&](uint32_t j) -> uint64_t { return j < hi ? __ldg(&frags[j]) : NONE; };
    auto fidx = [](uint64_t fk) -> uint32_t { return (uint32_t)(fk >> 8) & 0xFFFFFFu; };
    uint64_t k1 = key(lo + 1), k2 = key(lo + 2);
    uint32_t o1 = k1 != NONE ? db.poff[fidx(k1)] : 0u, t1 = k1 != NONE ? db.type[fidx(k1)] : 0u;
    for (uint32_t j = lo; j < hi; ++j) {
        const uint64_t fk = __ldg(&frags[j]);
        const uint32_t idx = (uint32_t)(fk >> 8) & 0xFFFFFFu;
        // issue: key of j+3, type/offset of j+2, parameter lines of j+2
        const uint64_t k3 = key(j + 3);
        uint32_t o2 = 0, t2 = 0;
        if (k2 != NONE) {
            o2 = db.poff[fidx(k2)];
            t2 = db.type[fidx(k2)];
            if (lane < 2) l2_warm(db.pw + o2 + 32 * lane);
        }
        // rows of j+1 (its parameters were warmed one iteration ago)
        if (k1 != NONE) tpcc_warm_warp(db, t1, db.pw + o1);
        if ((fk & 0xFFu) == F_WHOLE) {
            tpcc_txn_warp(db, idx, db.type[idx], db.pw + db.poff[idx], sh);
        } else {
            if (lane == 0) exec_frag<S_TPCC>(db, fk);
            __syncwarp();
        }
        k1 = k2; k2 = k3;
        o1 = o2; t1 = t2;
    }
    if (lane == 0 && hi - lo) atomicMax(&sc[SC_MAXCHAIN], hi - lo);
}

// One thread per partition runs its fragments in ts order.  The
// chain is serial, but what each fragment READS before executing (its fragment key, the
// transaction's type and parameter offset, the parameter words) is immutable, so it is
// loaded ahead in a software pipeline: fragment j+3 key, j+2 type/offset, j+1 parameter
// words (and its rows warmed into L2), j executes -- one dependent load per stage per
// iteration instead of a chain of four before every fragment.
template <int S>
__global__ void __launch_bounds__(128) part_exec_kernel(DevDb db, const uint64_t* __restrict__ frags,
                                                        const uint32_t* __restrict__ part_off, uint32_t nparts, uint32_t* sc) {
    constexpr int PW = S == S_TPCB || S == S_MICRO ? 4 : 8;
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= nparts) return;
    const uint32_t lo = part_off[p], hi = part_off[p + 1];
    const bool sh = db.ts != nullptr;
    constexpr uint64_t NONE = ~0ull;
    auto key = [&](uint32_t j) -> uint64_t { return j < hi ? __ldg(&frags[j]) : NONE; };
    auto fidx = [](uint64_t fk) -> uint32_t { return (uint32_t)(fk >> 8) & 0xFFFFFFu; };
    // stage registers: k1..k3 keys of fragments j+1..j+3; t2/o2 type/offset of j+2 (and
    // t1/o1 of j+1); q1 parameter words of j+1; k0/t0/q0 the fragment executing now
    uint64_t k0 = key(lo), k1 = key(lo + 1), k2 = key(lo + 2), k3 = key(lo + 3);
    uint32_t t0 = 0, o0 = 0, t1 = 0, o1 = 0, t2 = 0, o2 = 0;
    if (k0 != NONE) { t0 = db.type[fidx(k0)]; o0 = db.poff[fidx(k0)]; }
    if (k1 != NONE) { t1 = db.type[fidx(k1)]; o1 = db.poff[fidx(k1)]; }
    if (k2 != NONE) { t2 = db.type[fidx(k2)]; o2 = db.poff[fidx(k2)]; }
    uint32_t q0[PW], q1[PW];
#pragma unroll
    for (int w = 0; w < PW; ++w) {
        q0[w] = k0 != NONE ? db.pw[o0 + w] : 0u;
        q1[w] = k1 != NONE ? db.pw[o1 + w] : 0u;
    }
    for (uint32_t j = lo; j < hi; ++j) {
        // issue the next stages' loads (consumed next iteration)
        const uint64_t k4 = key(j + 4);
        uint32_t t3 = 0, o3 = 0;
        if (k3 != NONE) { t3 = db.type[fidx(k3)]; o3 = db.poff[fidx(k3)]; }
        uint32_t q2[PW];
#pragma unroll
        for (int w = 0; w < PW; ++w) q2[w] = k2 != NONE ? db.pw[o2 + w] : 0u;
        if (k1 != NONE) warm_rows<S>(db, t1, q1);
        // execute fragment j
        const uint32_t idx = fidx(k0), kind = (uint32_t)k0 & 0xFFu;
        if (S == S_TPCB) {
            if (t0 == 1) {
                tpcb_withdraw(db, idx, q0);
            } else {
                if (kind != F_REMOTE) tpcb_home(db, idx, q0, sh);
                if (kind != F_HOME) tpcb_account(db, idx, q0);
            }
        } else if (S == S_MICRO) {
            micro_txn(db, idx, t0, q0);
        } else {
            tm1_txn(db, idx, t0, q0);
        }
        // shift the pipeline
        k0 = k1; k1 = k2; k2 = k3; k3 = k4;
        t0 = t1; t1 = t2; t2 = t3;
        o1 = o2; o2 = o3;
#pragma unroll
        for (int w = 0; w < PW; ++w) { q0[w] = q1[w]; q1[w] = q2[w]; }
    }
    (void)o0; (void)o1;
    if (hi - lo) atomicMax(&sc[SC_MAXCHAIN], hi - lo);
}

// aborted transactions of the bulk (status != 0), for gputx_stats without a D2H of status
__global__ void __launch_bounds__(256) count_aborts_kernel(const uint8_t* __restrict__ status, uint32_t n,
                                                           uint32_t* out) {
    uint32_t c = 0;
    const uint32_t n4 = n / 4;
    const uint32_t* s4 = reinterpret_cast<const uint32_t*>(status);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
        const uint32_t v = __ldg(&s4[i]);
        c += ((v & 0xFFu) != 0) + ((v & 0xFF00u) != 0) + ((v & 0xFF0000u) != 0) + ((v & 0xFF000000u) != 0);
    }
    for (uint32_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        c += status[i] != 0;
    c = block_sum_u32(c);
    if (threadIdx.x == 0 && c) atomicAdd(out, c);
}

// =====================================================================================
// shard exchange.  A transaction whose
// fragments live on other shards is sent to each of them as a fixed-stride record
//   [ts, type, len, params[len], 0...]          (shard_stride words)
// and each remote fragment's output comes back to the home shard as
//   [ts, out words]                             (1 + out_stride/4 words)
// Records for one destination are contiguous and in home-bulk (ts) order.
// =====================================================================================
constexpr uint32_t MAX_SHARDS = 8;
constexpr int SC_DEST0 = 24;      // [24, 32): records per destination shard

// destination shards of a home transaction's remote fragments, from its raw (pre-ingest)
// parameters; malformed transactions go nowhere (the home ingest rejects them)
template <int S>
DEV uint32_t dest_mask(const DevDb& db, uint32_t t, const uint32_t* p, uint32_t len) {
    uint32_t m = 0;
    if (S == S_TPCB) {
        if (len == 4 && p[0] < db.dims[0] * db.dims[2]) m |= 1u << shard_of(db, p[0] / db.dims[2]);
    } else if (S == S_TPCC) {
        const uint32_t W = db.dims[0];
        if (t == 0 && len >= 4) {
            const uint32_t cnt = min(p[3], (len - 4) / 3);
            bool abort = false;
            for (uint32_t l = 0; l < cnt; ++l) {
                abort |= p[4 + 3 * l] >= db.dims[3];
                if (p[5 + 3 * l] < W) m |= 1u << shard_of(db, p[5 + 3 * l]);
            }
            if (abort) m = 0;
        } else if (t == 1 && len == 7 && p[2] < W) {
            m |= 1u << shard_of(db, p[2]);
        }
    }
    return m & ~(1u << db.shard);
}

// the caller's home-bulk offsets, checked before anything is read through them:
// param_off[0] == 0, non-decreasing, at most maxlen words per transaction, param_off[nh] ==
// the word count; a violation reports E_OFF at the first bad transaction
__global__ void __launch_bounds__(256) shard_validate_kernel(const uint32_t* poff, uint32_t nh, uint32_t n_words,
                                                             uint32_t maxlen, uint32_t* sc) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x) {
        const uint32_t o0 = poff[i], o1 = poff[i + 1];
        if ((i == 0 && o0 != 0) || o1 < o0 || o1 - o0 > maxlen || o1 > n_words || (i == nh - 1 && o1 != n_words))
            report_err(sc, E_OFF, i);
    }
}
// a transaction's word count as the shard kernels read it: clamped to the record stride
DEV uint32_t shard_len(const uint32_t* poff, uint32_t i, uint32_t maxlen) {
    const uint32_t o0 = poff[i], o1 = poff[i + 1];
    return o1 < o0 ? 0u : min(o1 - o0, maxlen);
}

template <int S>
__global__ void __launch_bounds__(256) shard_count_kernel(DevDb db, const uint8_t* type, const uint32_t* poff,
                                                          const uint32_t* pw, uint32_t nh, uint32_t* cnt) {
    const uint32_t maxlen = S == S_TPCB ? 4u : S == S_TM1 ? 7u : 49u;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x)
        cnt[i] = __popc(dest_mask<S>(db, type[i], pw + poff[i], shard_len(poff, i, maxlen)));
}

template <int S>
__global__ void __launch_bounds__(256) shard_pair_kernel(DevDb db, const uint8_t* type, const uint32_t* poff,
                                                         const uint32_t* pw, uint32_t nh, const uint32_t* off,
                                                         uint64_t* pairs, uint32_t* sc) {
    const uint32_t maxlen = S == S_TPCB ? 4u : S == S_TM1 ? 7u : 49u;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x) {
        uint32_t m = dest_mask<S>(db, type[i], pw + poff[i], shard_len(poff, i, maxlen));
        uint32_t o = off[i];
        while (m) {
            const uint32_t q = __ffs(m) - 1;
            m &= m - 1;
            pairs[o++] = ((uint64_t)q << 32) | i;
            atomicAdd(&sc[SC_DEST0 + q], 1u);
        }
    }
}

__global__ void __launch_bounds__(256) shard_pack_kernel(const uint64_t* pairs, const uint32_t* npairs,
                                                         const uint8_t* type, const uint32_t* poff, const uint32_t* pw,
                                                         const uint32_t* ts, uint32_t stride, uint32_t* send) {
    const uint32_t np = *npairs;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < np; k += gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)pairs[k];
        const uint32_t o0 = poff[i], len = shard_len(poff, i, stride - 3);
        uint32_t* r = send + (uint64_t)k * stride;
        r[0] = ts[i];
        r[1] = type[i];
        r[2] = len;
        for (uint32_t w = 0; w < stride - 3; ++w) r[3 + w] = w < len ? pw[o0 + w] : 0u;
    }
}

// merge: sort keys ts << 32 | source (home i < nh, received nh + j)
__global__ void __launch_bounds__(256) merge_keys_kernel(const uint32_t* hts, uint32_t nh, const uint32_t* recv,
                                                         uint32_t nr, uint32_t stride, uint64_t* keys) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nh + nr; k += gridDim.x * blockDim.x) {
        const uint32_t t = k < nh ? hts[k] : recv[(uint64_t)(k - nh) * stride];
        keys[k] = ((uint64_t)t << 32) | k;
    }
}

__global__ void __launch_bounds__(256) merge_meta_kernel(const uint64_t* keys, uint32_t n, uint32_t nh,
                                                         const uint8_t* htype, const uint32_t* hpoff,
                                                         const uint32_t* hts, const uint32_t* recv, uint32_t stride,
                                                         uint8_t* type, uint32_t* ts, uint32_t* src, uint32_t* home_pos,
                                                         uint32_t* len) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint32_t s = (uint32_t)keys[k];
        if (s < nh) {
            type[k] = htype[s];
            ts[k] = hts[s];
            len[k] = shard_len(hpoff, s, stride - 3);
            src[k] = s;
            home_pos[s] = k;
        } else {
            const uint32_t* r = recv + (uint64_t)(s - nh) * stride;
            type[k] = (uint8_t)min(r[1], 255u);
            ts[k] = r[0];
            len[k] = min(r[2], stride - 3);
            src[k] = NOT_HOME;
        }
    }
}

__global__ void __launch_bounds__(256) merge_params_kernel(const uint64_t* keys, uint32_t n, uint32_t nh,
                                                           const uint32_t* hpoff, const uint32_t* hpw,
                                                           const uint32_t* recv, uint32_t stride, const uint32_t* poff,
                                                           uint32_t* pw, uint32_t max_words) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const uint32_t s = (uint32_t)keys[k];
        const uint32_t o = poff[k], len = poff[k + 1] - o;
        const uint32_t* from = s < nh ? hpw + hpoff[s] : recv + (uint64_t)(s - nh) * stride + 3;
        // writes are bounded by the buffer (the host then rejects n_words > max_words)
        for (uint32_t w = 0; w < len && o + w < max_words; ++w) pw[o + w] = from[w];
    }
}

// results of peers' transactions go back to their home shard
__global__ void __launch_bounds__(256) ret_count_kernel(const uint32_t* src, uint32_t n, uint32_t* cnt) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        cnt[k] = src[k] == NOT_HOME ? 1u : 0u;
}
template <int S>
__global__ void __launch_bounds__(256) ret_pair_kernel(DevDb db, const uint32_t* off, uint64_t* pairs, uint32_t* sc) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < db.n; k += gridDim.x * blockDim.x) {
        if (db.src[k] != NOT_HOME) continue;
        const uint32_t* p = db.pw + db.poff[k];
        const uint32_t q = shard_of(db, S == S_TPCB ? p[2] : p[0]);
        pairs[off[k]] = ((uint64_t)q << 32) | k;
        atomicAdd(&sc[SC_DEST0 + q], 1u);
    }
}

__global__ void __launch_bounds__(256) ret_pack_kernel(const uint64_t* pairs, const uint32_t* npairs, const uint32_t* ts,
                                                       const uint8_t* out, uint32_t ow, uint32_t* send) {
    const uint32_t np = *npairs;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < np; k += gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)pairs[k];
        uint32_t* r = send + (uint64_t)k * (1 + ow);
        r[0] = ts[i];
        const uint32_t* o = reinterpret_cast<const uint32_t*>(out + (uint64_t)i * ow * 4);
        for (uint32_t w = 0; w < ow; ++w) r[1 + w] = o[w];
    }
}

// the fragments write disjoint output fields (zero elsewhere): OR them into the home record
__global__ void __launch_bounds__(256) ret_merge_kernel(const uint32_t* recv, uint32_t nr, uint32_t ow, const uint32_t* ts,
                                                        const uint32_t* src, uint32_t n, uint8_t* out, uint32_t* sc) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < nr; j += gridDim.x * blockDim.x) {
        const uint32_t* r = recv + (uint64_t)j * (1 + ow);
        const uint32_t t = r[0];
        uint32_t lo = 0, hi = n;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (ts[mid] < t) lo = mid + 1; else hi = mid;
        }
        if (lo >= n || ts[lo] != t || src[lo] == NOT_HOME) { report_err(sc, E_OWNER, j); continue; }
        uint32_t* o = reinterpret_cast<uint32_t*>(out + (uint64_t)lo * ow * 4);
        for (uint32_t w = 0; w < ow; ++w)            // several shards may return to one record
            if (r[1 + w]) atomicOr(&o[w], r[1 + w]);
    }
}

// home results in home-bulk order
__global__ void __launch_bounds__(256) home_gather_kernel(const uint32_t* home_pos, uint32_t nh, const uint8_t* status,
                                                          const uint8_t* out, uint32_t stride, uint8_t* hstatus,
                                                          uint8_t* hout) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x) {
        const uint32_t k = home_pos[i];
        hstatus[i] = status[k];
        const uint32_t* a = reinterpret_cast<const uint32_t*>(out + (uint64_t)k * stride);
        uint32_t* b = reinterpret_cast<uint32_t*>(hout + (uint64_t)i * stride);
        for (uint32_t w = 0; w < stride / 4; ++w) b[w] = a[w];
    }
}

// =====================================================================================
// TPL
// =====================================================================================
// index + 1 of the last group head / write / read / add at or before a position
struct Pair { uint32_t h, w, r, a; };
struct OpPair {
    static DEV Pair identity() { return Pair{0u, 0u, 0u, 0u}; }
    static DEV Pair combine(const Pair& x, const Pair& y) {
        return Pair{max(x.h, y.h), max(x.w, y.w), max(x.r, y.r), max(x.a, y.a)};
    }
};
DEV Pair tpl_elem(uint64_t i, bool head, uint32_t mode) {
    const uint32_t p = (uint32_t)i + 1;
    return Pair{head ? p : 0u, mode == 1 ? p : 0u, mode == 0 ? p : 0u, mode == 2 ? p : 0u};
}

// Counter-lock keys (DESIGN.md R-S5): in group order, a write's key is its position in
// the group; a read's (an add's) key is the position of the first record of its run of
// reads (adds), i.e. one past the last record it conflicts with.  A record may enter
// when lock >= key; it releases +1 after its transaction.
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
            agg = OpPair::combine(agg, tpl_elem(i, head, key_mode(kk[k])));
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
            const uint32_t mode = key_mode(kk[k]);
            // index+1 of the last earlier record this one conflicts with (reads: writes and
            // adds; adds: writes and reads)
            const uint32_t lc_ex = mode == 0 ? max(cur.w, cur.a) : max(cur.w, cur.r);
            cur = OpPair::combine(cur, tpl_elem(i, head, mode));
            const uint32_t H = cur.h - 1;                  // group head index
            uint32_t key;
            if (mode == 1) key = (uint32_t)i - H;
            else key = (lc_ex > H) ? lc_ex - H : 0u;
            lkey[rec_off[key_idx(kk[k])] + key_j(kk[k])] = key;
            if (head) lock[key_item(kk[k])] = 0;
        }
    }
}

constexpr uint32_t SPIN_LIMIT = 1u << 24;   // polls before the watchdog trips (EDEADLOCK)

// Enter a counter lock: wait until *lw >= key.  Warp-aggregated acquisition: the lanes
// of a warp currently waiting on the same lock word share one poll (one leader load,
// broadcast).  A waiter sleeps in proportion to the releases it still needs
// (key - value), so a deep queue behind a hot lock does not flood L2 with polls.
// Only lanes already in the loop take part in the collectives (__activemask), and
// no lane waits inside a collective for another lane's release: ITS lets a lane whose
// lock is free leave, execute and release while its siblings keep polling.
__device__ uint32_t g_tpl_sleep_cap = 2048;    // ns; GPUTX_TPL_SLEEP overrides (experiments)

// K-SET dataflow look-ahead throttle: a transaction of depth k does not start polling its
// locks before the k-set (k - ahead - 1) is complete, so the resident lanes poll the locks
// of a few k-sets only (300 k lanes spinning on the next 300 levels of TPC-B's 1,000 branch
// locks saturated L2 with polls: 14 -> 192 ms).  Pure pacing: correctness comes from the
// lock keys alone.  level sizes from the group offsets (goff[k*T]), completions in done[k].
struct DfThrottle {
    const uint32_t* D;         // depth per transaction (null: TPL, no throttle)
    const uint32_t* goff;      // group offsets: k-set k = perm[goff[k*T] .. goff[(k+1)*T])
    uint32_t T, ahead;
    uint32_t* done;            // completed transactions per k-set
    DEV bool on() const { return D != nullptr; }
    DEV void wait(uint32_t idx) const {
        const uint32_t k = __ldg(&D[idx]);
        if (k <= ahead) return;
        const uint32_t lv = k - ahead - 1;
        const uint32_t need = __ldg(&goff[(lv + 1) * T]) - __ldg(&goff[lv * T]);
        uint32_t polls = 0;
        while (ld_relaxed(&done[lv]) < need)
            if (++polls > 4) __nanosleep(256);
    }
    DEV void finish(uint32_t idx) const {
        const uint32_t k = __ldg(&D[idx]);
        const uint32_t am = __activemask();
        const uint32_t peers = __match_any_sync(am, k);
        if ((int)lane_id() == __ffs(peers) - 1) atomicAdd(&done[k], (uint32_t)__popc(peers));
    }
};
DEV bool tpl_acquire(uint32_t* lw, uint32_t key) {
    if (ld_acquire(lw) >= key) return true;          // uncontended: no collective
    uint32_t polls = 0;
    for (;;) {
        const uint32_t am = __activemask();
        const uint32_t peers = __match_any_sync(am, (unsigned long long)lw);
        const int leader = __ffs(peers) - 1;
        uint32_t v = 0;
        if ((int)lane_id() == leader) v = ld_acquire(lw);
        v = __shfl_sync(peers, v, leader);
        if (v >= key) return true;
        if (++polls > SPIN_LIMIT) return false;
        const uint32_t gap = key - v;
        const uint32_t cap = g_tpl_sleep_cap;
        if (cap) {
            if (gap > 1) __nanosleep(min(gap * 32u, cap));
            else if (polls > 8) __nanosleep(32);
        }
    }
}

// Release +1 on a lock word; lanes releasing the same word combine into one atomic.
// The leader's increment is a release (red.release.gpu); __syncwarp(peers) first makes
// every peer's writes happen before it (release is cumulative) -- no fence.sc per lane
// (fence.sc + atomicAdd cost ~0.3 us more per hand-off, tools/handoff.cu).
DEV void tpl_release(uint32_t* lw) {
    const uint32_t am = __activemask();
    const uint32_t peers = __match_any_sync(am, (unsigned long long)lw);
    __syncwarp(peers);
    if ((int)lane_id() == __ffs(peers) - 1) red_add_release(lw, (uint32_t)__popc(peers));
}

template <int S, bool SH>
__global__ void __launch_bounds__(128) tpl_exec_kernel(DevDb db, const uint32_t* __restrict__ rec_off,
                                                       const uint32_t* __restrict__ lkey, uint32_t* lock, uint32_t* sc) {
    __shared__ uint32_t s_base;
    if (threadIdx.x == 0) s_base = atomicAdd(&sc[SC_TICKET], blockDim.x);   // ts-ordered dispatch
    __syncthreads();
    const uint32_t idx = s_base + threadIdx.x;
    // The warp stays converged: every iteration, each unfinished lane advances through
    // the locks it can enter (growing phase, keys order conflicting records by ts); lanes
    // holding all their locks execute and release (shrinking phase) in the same
    // iteration.  A lane whose locks are free therefore never waits behind siblings that
    // keep polling (with per-lane spin loops the polling path starved the ready lanes:
    // TPC-B 4M, 1,000 branches, 130 ms).  Lanes wait only for smaller tickets.
    bool done = idx >= db.n;
    Rec r[MAX_REC];
    int k = 0, j = 0;
    uint32_t ro = 0, key = 0;
    if (!done) {
        k = footprint_local<S>(db, db.type[idx], db.pw + db.poff[idx], r);
        ro = rec_off[idx];
        if (k) key = __ldg(&lkey[ro]);
    }
    uint32_t polls = 0;
    while (__any_sync(0xffffffffu, !done)) {
        bool progressed = false;
        uint32_t gap = 0xFFFFFFFFu;      // releases this lane still needs on its blocking lock
        if (!done) {
            while (j < k) {
                const uint32_t v = ld_acquire(&lock[r[j].item]);
                if (v < key) { gap = key - v; break; }
                ++j;
                progressed = true;
                if (j < k) key = __ldg(&lkey[ro + j]);
            }
            if (j == k) {
                exec_txn<S, SH>(db, idx);
                for (int q = 0; q < k; ++q) tpl_release(&lock[r[q].item]);
                done = true;
                progressed = true;
            }
        }
        if (!__any_sync(0xffffffffu, progressed)) {
            if (++polls > SPIN_LIMIT) {
                if (!done) atomicExch(&sc[SC_DEADLOCK], 1u);
                break;
            }
            // the warp's nearest lock is `g` releases away: sleep in proportion (a deep
            // queue behind a hot lock must not flood L2 with polls)
            const uint32_t g = __reduce_min_sync(0xffffffffu, gap);
            __nanosleep(g == 1 ? (polls > 8 ? 32u : 0u) : min(g * 32u, g_tpl_sleep_cap));
        }
    }
}

// TPL for TPC-C: one warp per transaction.  Lane j waits for the lock of record j (all
// of a transaction's locks are requested at once: keys order every lock's queue by ts,
// so a transaction only ever waits for earlier ones and the order of requests cannot
// deadlock), then the warp runs tpcc_txn_warp and every lane releases its lock.
template <bool SH>
__global__ void __launch_bounds__(128) tpl_exec_warp_kernel(DevDb db, const uint32_t* __restrict__ rec_off,
                                                            const uint32_t* __restrict__ lkey, uint32_t* lock,
                                                            uint32_t* sc, const uint32_t* __restrict__ order,
                                                            DfThrottle thr) {
    __shared__ uint32_t s_base;
    if (threadIdx.x == 0) s_base = atomicAdd(&sc[SC_TICKET], blockDim.x / 32);   // ordered dispatch
    __syncthreads();
    const uint32_t tk = s_base + (threadIdx.x >> 5);
    if (tk >= db.n) return;                                    // warp-uniform
    // tickets follow ts (TPL) or the k-set order (K-SET dataflow: order = perm)
    const uint32_t idx = order ? __ldg(&order[tk]) : tk;
    const uint32_t lane = lane_id();
    Rec r[MAX_REC];
    const int k = footprint_local<S_TPCC>(db, db.type[idx], db.pw + db.poff[idx], r);
    uint64_t item = 0;
#pragma unroll
    for (int j = 0; j < MAX_REC; ++j)
        if (j < k && (uint32_t)j == lane) item = r[j].item;
    const bool mine = (int)lane < k;
    const uint32_t key = mine ? __ldg(&lkey[rec_off[idx] + lane]) : 0u;
    if (thr.on()) thr.wait(idx);
    // the rows come into L2 while the locks are awaited (on the W_YTD / district chains
    // the post-acquire execution is the critical path)
    const uint32_t t = db.type[idx];
    tpcc_warm_warp(db, t, db.pw + db.poff[idx]);
    // Payment: its warehouse's W_YTD lock (record 0, lane 0) is taken LAST -- the rest of
    // the transaction runs and releases D_YTD / CUST first, then W_YTD is updated in its
    // turn and released at once -- so a hop of the ~6.7 k-Payment W_YTD chain of a
    // warehouse costs one lock hand-off and one red.add instead of a whole Payment.
    // Every item is still accessed in its ts-ordered turn (the lock keys), which alone
    // makes the execution equivalent to the serial ts order; a transaction waits only for
    // earlier ones (no lock held while waiting for W_YTD).
    const bool late = t != 0 && !(SH && db.xflag && db.xflag[idx]);
    bool got = !mine || (late && lane == 0);
    uint32_t polls = 0;
    while (!__all_sync(0xffffffffu, got)) {
        uint32_t gap = 0xFFFFFFFFu;
        if (!got) {
            const uint32_t v = ld_acquire(&lock[item]);
            got = v >= key;
            if (!got) gap = key - v;
        }
        if (__all_sync(0xffffffffu, got)) break;
        if (++polls > SPIN_LIMIT) { if (lane == 0) atomicExch(&sc[SC_DEADLOCK], 1u); break; }
        const uint32_t g = __reduce_min_sync(0xffffffffu, gap);
        __nanosleep(g == 1 ? (polls > 8 ? 32u : 0u) : min(g * 32u, g_tpl_sleep_cap));
    }
    if (late) {
        const uint64_t i1 = __shfl_sync(0xffffffffu, item, 1), i2 = __shfl_sync(0xffffffffu, item, 2);
        if (lane == 0) {
            const uint32_t* p = db.pw + db.poff[idx];
            const bool ok = tpcc_payment(db, idx, p, SH, false);
            if (k > 1) red_add_release(&lock[i1], 1u);
            if (k > 2) red_add_release(&lock[i2], 1u);
            uint32_t v, n = 0;
            while ((v = ld_acquire(&lock[item])) < key) {
                if (++n > SPIN_LIMIT) { atomicExch(&sc[SC_DEADLOCK], 1u); break; }
                __nanosleep(key - v == 1 ? (n > 8 ? 32u : 0u) : min((key - v) * 32u, g_tpl_sleep_cap));
            }
            if (ok) red_add(&COL(int64_t, C_W_YTD)[p[0]], (int64_t)p[6]);
            // the W_YTD turn passes without a release fence: the access it orders is a blind
            // atomic add (no transaction reads W_YTD), so the next holder needs the turn, not the
            // visibility of this add -- the hand-off of the ~6,700-Payment W_YTD chains loses the
            // fence's wait for the add's acknowledgement
            atomicAdd(&lock[item], 1u);
            if (thr.on()) atomicAdd(&thr.done[__ldg(&thr.D[idx])], 1u);
        }
        return;
    }
    exec_txn_warp<SH>(db, idx);
    __syncwarp();                              // every lane's writes before any lane's release
    if (mine) red_add_release(&lock[item], 1u);
    if (thr.on() && lane == 0) atomicAdd(&thr.done[__ldg(&thr.D[idx])], 1u);
}

// Persistent TPL: every lane takes its next transaction as soon as it has released the
// previous one (warp-aggregated ticket grab, tickets in ts order).  A lane holding
// ticket t waits only for transactions with smaller tickets, all of which were taken
// by running lanes, so the grid (sized to what is co-resident) always progresses, and
// no slot idles behind a slow sibling of its CTA.
template <int S, bool SH>
__global__ void __launch_bounds__(256) tpl_exec_persistent_kernel(DevDb db, const uint32_t* __restrict__ rec_off,
                                                                  const uint32_t* __restrict__ lkey, uint32_t* lock,
                                                                  uint32_t* sc, const uint32_t* __restrict__ order,
                                                                  DfThrottle thr) {
    for (;;) {
        const uint32_t am = __activemask();
        const int leader = __ffs(am) - 1;
        uint32_t base = 0;
        if ((int)lane_id() == leader) base = atomicAdd(&sc[SC_TICKET], (uint32_t)__popc(am));
        base = __shfl_sync(am, base, leader);
        const uint32_t tk = base + __popc(am & lanemask_lt());
        if (tk >= db.n) break;
        // K-SET dataflow (order = perm): tickets in k-set order, so a transaction only
        // waits for transactions of smaller depth, all already taken by running lanes
        const uint32_t idx = order ? __ldg(&order[tk]) : tk;
        if (thr.on()) thr.wait(idx);
        Rec r[MAX_REC];
        const int k = footprint_local<S>(db, db.type[idx], db.pw + db.poff[idx], r);
        const uint32_t ro = rec_off[idx];
        for (int j = 0; j < k; ++j) {
            const uint32_t key = __ldg(&lkey[ro + j]);
            if (!tpl_acquire(&lock[r[j].item], key)) atomicExch(&sc[SC_DEADLOCK], 1u);
        }
        exec_txn<S, SH>(db, idx);
        for (int j = 0; j < k; ++j) tpl_release(&lock[r[j].item]);
        if (thr.on()) thr.finish(idx);
    }
}

}  // namespace gputx

namespace gputx {
// =====================================================================================
// Streaming K-SET over a live transaction pool (SURVEY.md §8(f)
// NEXT-2).  The pool = transactions not executed yet, in ts order, already ingested, with
// their access records kept SORTED by (item, ts).  Arrivals are ingested in a staging
// area, their records radix-sorted on their own and MERGED into the pool's sorted array
// ("their basic operations are merged into the sorted array").  A step
// executes the pool's 0-set -- found in one pass over the records, no rank fixpoint ("the
// incremental algorithm is able to find the 0-set without computing the k-set from
// scratch"): a transaction is in the 0-set iff no earlier pool transaction conflicts with
// it, i.e. each of its records is a write at the head of its item group, or a read (add)
// with only reads (adds) before it -- then removes them and their records from the pool.
// =====================================================================================
constexpr uint32_t POOL_INF = 0xFFFFFFFFu;

// append the ingested arrivals (staging) to the pool: types, rebased offsets, words,
// timestamps ts0 + i, per-table insert counts (stride cap + 1; TPC-B: one history row each)
__global__ void __launch_bounds__(256) pool_append_kernel(const uint8_t* __restrict__ st_type,
        const uint32_t* __restrict__ st_poff, const uint32_t* __restrict__ st_pw, const uint32_t* __restrict__ st_ins,
        uint32_t m, uint32_t n0, uint32_t w0, uint32_t ts0, uint32_t ntab, uint32_t ins_all_one, uint8_t* p_type,
        uint32_t* p_poff, uint32_t* p_pw, uint32_t* p_ts, uint32_t* p_ins, uint32_t cap) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    for (uint32_t i = tid; i < m; i += nt) {
        p_type[n0 + i] = st_type[i];
        p_poff[n0 + i] = w0 + st_poff[i];
        p_ts[n0 + i] = ts0 + i;
        for (uint32_t t = 0; t < ntab; ++t)
            p_ins[t * (cap + 1) + n0 + i] = ins_all_one ? 1u : st_ins[t * (m + 1) + i];
    }
    const uint32_t nw = st_poff[m];
    for (uint32_t j = tid; j < nw; j += nt) p_pw[w0 + j] = st_pw[j];
    if (tid == 0) p_poff[n0 + m] = w0 + nw;
}

// merge two sorted runs of unique keys: A (the pool's records) and B (the arrivals')
__global__ void __launch_bounds__(256) pool_merge_kernel(const uint64_t* __restrict__ A, uint32_t na,
                                                         const uint64_t* __restrict__ B, const uint32_t* nb_ptr,
                                                         uint64_t* __restrict__ out) {
    const uint32_t nb = *nb_ptr;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    for (uint32_t i = tid; i < na + nb; i += nt) {
        const bool fromA = i < na;
        const uint64_t k = fromA ? __ldg(&A[i]) : __ldg(&B[i - na]);
        const uint64_t* other = fromA ? B : A;
        uint32_t lo = 0, hi = fromA ? nb : na;          // #keys of the other run below k
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(&other[mid]) < k) lo = mid + 1; else hi = mid;
        }
        out[(fromA ? i : i - na) + lo] = k;
    }
}

// 0-set, pass 1: per item group of the pool, reset the first non-read / non-add positions
__global__ void __launch_bounds__(256) pool_zs_init_kernel(const uint64_t* __restrict__ keys, uint32_t nrec,
                                                           uint32_t* fnr, uint32_t* fna, uint32_t* zflag, uint32_t n) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    for (uint32_t r = tid; r < nrec; r += nt) {
        const uint64_t it = key_item(__ldg(&keys[r]));
        fnr[it] = POOL_INF;
        fna[it] = POOL_INF;
    }
    for (uint32_t t = tid; t < n; t += nt) zflag[t] = 1u;
}
// pass 2: first position of a record that is not a read (resp. not an add) in each group
__global__ void __launch_bounds__(256) pool_zs_mark_kernel(const uint64_t* __restrict__ keys, uint32_t nrec,
                                                           uint32_t* fnr, uint32_t* fna) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrec; r += gridDim.x * blockDim.x) {
        const uint64_t k = __ldg(&keys[r]);
        const uint32_t mode = key_mode(k);
        if (mode != 0) atomicMin(&fnr[key_item(k)], r);
        if (mode != 2) atomicMin(&fna[key_item(k)], r);
    }
}
// pass 3: a record with a conflicting earlier record in its group takes its transaction
// out of the 0-set (write: not the group head; read: a non-read before it; add: a non-add)
__global__ void __launch_bounds__(256) pool_zs_check_kernel(const uint64_t* __restrict__ keys, uint32_t nrec,
                                                            const uint32_t* fnr, const uint32_t* fna, uint32_t* zflag) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrec; r += gridDim.x * blockDim.x) {
        const uint64_t k = __ldg(&keys[r]);
        const uint64_t it = key_item(k);
        const uint32_t mode = key_mode(k);
        bool ok;
        if (mode == 1) ok = r == 0 || key_item(__ldg(&keys[r - 1])) != it;
        else if (mode == 0) ok = fnr[it] > r;
        else ok = fna[it] > r;
        if (!ok) zflag[key_idx(k)] = 0u;
    }
}

// the step's insert counts: rows of executed (0-set) transactions only
__global__ void __launch_bounds__(256) pool_ins_mask_kernel(const uint32_t* __restrict__ zflag,
                                                            const uint32_t* __restrict__ p_ins, uint32_t n, uint32_t cap,
                                                            uint32_t ntab, uint32_t* cnt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        for (uint32_t t = 0; t < ntab; ++t) cnt[t * (n + 1) + i] = zflag[i] ? p_ins[t * (cap + 1) + i] : 0u;
}

// execution list of the 0-set (ts order) from the scanned flags
__global__ void __launch_bounds__(256) pool_list_kernel(const uint32_t* __restrict__ zflag,
                                                        const uint32_t* __restrict__ pos, uint32_t n, uint32_t* list) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (zflag[i]) list[pos[i]] = i;
}

// one lock-free round over the 0-set (Property 1): no two listed
// transactions conflict; one thread per transaction (TPC-C: one warp)
template <int S>
__global__ void __launch_bounds__(256) pool_exec_kernel(DevDb db, const uint32_t* __restrict__ list,
                                                        const uint32_t* cnt_ptr) {
    const uint32_t cnt = *cnt_ptr;
    if (S == S_TPCC) {
        const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
        for (uint32_t k = w; k < cnt; k += nw) exec_txn_warp<true>(db, __ldg(&list[k]));
    } else {
        for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x)
            exec_txn<S, true>(db, __ldg(&list[k]));
    }
}

// results of the step, in ts order: ts, status, output record
__global__ void __launch_bounds__(256) pool_results_kernel(const uint32_t* __restrict__ list, const uint32_t* cnt_ptr,
                                                           const uint32_t* __restrict__ p_ts,
                                                           const uint8_t* __restrict__ status,
                                                           const uint8_t* __restrict__ out, uint32_t ow,
                                                           uint32_t* r_ts, uint8_t* r_status, uint8_t* r_out) {
    const uint32_t cnt = *cnt_ptr;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x) {
        const uint32_t i = __ldg(&list[k]);
        r_ts[k] = p_ts[i];
        r_status[k] = status[i];
        for (uint32_t b = 0; b < ow; ++b) r_out[(uint64_t)k * ow + b] = out[(uint64_t)i * ow + b];
    }
}

// keep flags (1 - zflag) and kept parameter lengths, for the compaction scans
__global__ void __launch_bounds__(256) pool_keep_kernel(const uint32_t* __restrict__ zflag,
                                                        const uint32_t* __restrict__ p_poff, uint32_t n,
                                                        uint32_t* keep, uint32_t* klen) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        keep[i] = zflag[i] ? 0u : 1u;
        klen[i] = zflag[i] ? 0u : p_poff[i + 1] - p_poff[i];
    }
}
// move the kept transactions to their new (dense, still ts-ordered) positions
__global__ void __launch_bounds__(256) pool_compact_kernel(const uint32_t* __restrict__ zflag,
        const uint32_t* __restrict__ npos, const uint32_t* __restrict__ noff, uint32_t n, uint32_t ntab, uint32_t cap,
        const uint8_t* __restrict__ p_type, const uint32_t* __restrict__ p_poff, const uint32_t* __restrict__ p_pw,
        const uint32_t* __restrict__ p_ts, const uint32_t* __restrict__ p_ins, uint8_t* q_type, uint32_t* q_poff,
        uint32_t* q_pw, uint32_t* q_ts, uint32_t* q_ins, const uint32_t* nkept_ptr, const uint32_t* nwords_ptr) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
    for (uint32_t i = tid; i < n; i += nt) {
        if (zflag[i]) continue;
        const uint32_t j = npos[i];
        q_type[j] = p_type[i];
        q_ts[j] = p_ts[i];
        q_poff[j] = noff[i];
        for (uint32_t t = 0; t < ntab; ++t) q_ins[t * (cap + 1) + j] = p_ins[t * (cap + 1) + i];
        const uint32_t a = p_poff[i], len = p_poff[i + 1] - a;
        for (uint32_t w = 0; w < len; ++w) q_pw[noff[i] + w] = p_pw[a + w];
    }
    if (tid == 0) q_poff[*nkept_ptr] = *nwords_ptr;
}
// records of kept transactions, idx renumbered (the (item, ts) order is unchanged)
__global__ void __launch_bounds__(256) pool_rec_keep_kernel(const uint64_t* __restrict__ keys, uint32_t nrec,
                                                            const uint32_t* __restrict__ zflag, uint32_t* keep) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrec; r += gridDim.x * blockDim.x)
        keep[r] = zflag[key_idx(__ldg(&keys[r]))] ? 0u : 1u;
}
__global__ void __launch_bounds__(256) pool_rec_compact_kernel(const uint64_t* __restrict__ keys, uint32_t nrec,
                                                               const uint32_t* __restrict__ keep,
                                                               const uint32_t* __restrict__ rpos,
                                                               const uint32_t* __restrict__ npos, uint64_t* out) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrec; r += gridDim.x * blockDim.x) {
        if (!keep[r]) continue;
        const uint64_t k = __ldg(&keys[r]);
        const uint64_t idx_mask = (uint64_t)0xFFFFFFu << 6;
        out[rpos[r]] = (k & ~idx_mask) | ((uint64_t)npos[key_idx(k)] << 6);
    }
}
}  // namespace gputx

namespace gputx {
// =====================================================================================
// Relaxed-timestamp strategies (Appendix G):
// serializability without the timestamp constraint -- the result equals serial execution
// in SOME order, which the executor records (d_order, gputx_read_serial_order).
//   TPL_RELAXED : the basic spin lock of Figure 10 (atomicCAS 0 -> 1, release 0), locks
//                 acquired in increasing item order (no deadlock), strict 2PL; a
//                 transaction takes its serialization number at its lock point (every
//                 lock held), and 2PL serializes transactions in lock-point order.
//   PART_RELAXED: no sort: "each transaction needs to acquire the lock for its partition,
//                 get the counter value as its key value, and increases the counter value
//                 by one ... A prefix sum is used to calculate the start position of each
//                 group"; cross-partition transactions then run under
//                 TPL_RELAXED ("we use TPL"), after every partition.
// =====================================================================================
constexpr uint32_t RX_CROSS = 0xFFFFFFFFu;

DEV void rx_sort_items(Rec* r, int k) {        // insertion sort by item (k <= MAX_REC)
    for (int a = 1; a < k; ++a) {
        const Rec x = r[a];
        int b = a - 1;
        while (b >= 0 && r[b].item > x.item) { r[b + 1] = r[b]; --b; }
        r[b + 1] = x;
    }
}

// list: the transactions to run (nullptr: all of the bulk); order[base + seq] = idx
template <int S>
__global__ void __launch_bounds__(128) tpl_relaxed_kernel(DevDb db, const uint32_t* __restrict__ list,
                                                          const uint32_t* cnt_ptr, uint32_t* lock, uint32_t* order,
                                                          uint32_t base, uint32_t* sc) {
    const uint32_t cnt = list ? *cnt_ptr : db.n;
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    bool done = t >= cnt;
    const uint32_t idx = done ? 0u : (list ? __ldg(&list[t]) : t);
    Rec r[MAX_REC];
    int k = 0, j = 0;
    if (!done) {
        k = footprint<S>(db, db.type[idx], db.pw + db.poff[idx], r);
        rx_sort_items(r, k);
    }
    uint32_t polls = 0;
    // warp-converged acquisition (as tpl_exec_kernel): lanes that can take their next lock
    // advance, lanes holding every lock execute and release in the same iteration
    while (__any_sync(0xffffffffu, !done)) {
        bool progressed = false;
        if (!done) {
            while (j < k) {
                uint32_t old;
                asm volatile("atom.acquire.gpu.global.cas.b32 %0, [%1], 0, 1;" : "=r"(old) : "l"(&lock[r[j].item]) : "memory");
                if (old != 0u) break;
                ++j;
                progressed = true;
            }
            if (j == k) {
                const uint32_t seq = atomicAdd(&sc[SC_TICKET], 1u);       // lock point
                order[base + seq] = idx;
                exec_txn<S, false>(db, idx);
                for (int q = 0; q < k; ++q) st_release(&lock[r[q].item], 0u);
                done = true;
                progressed = true;
            }
        }
        if (!__any_sync(0xffffffffu, progressed)) {
            if (++polls > SPIN_LIMIT) {
                if (!done) atomicExch(&sc[SC_DEADLOCK], 1u);
                break;
            }
            __nanosleep(polls > 8 ? 64u : 0u);
        }
    }
}

// PART_RELAXED step 1: partition key by counter (single-partition transactions) or the
// cross list; step 2 (after a scan of cnt): the partition-major list
template <int S>
__global__ void __launch_bounds__(256) rpart_key_kernel(DevDb db, uint32_t* pcnt, uint32_t* pkey, uint32_t* ppid,
                                                        uint32_t* clist, uint32_t* sc) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < db.n; i += gridDim.x * blockDim.x) {
        uint64_t fk[MAX_REC];
        const int nf = fragments<S>(db, i, fk);
        if (nf == 1) {
            const uint32_t pid = (uint32_t)(fk[0] >> 32);
            ppid[i] = pid;
            pkey[i] = atomicAdd(&pcnt[pid], 1u);
        } else {
            ppid[i] = RX_CROSS;
            clist[atomicAdd(&sc[SC_XTOTAL], 1u)] = i;
        }
    }
}
__global__ void __launch_bounds__(256) rpart_scatter_kernel(const uint32_t* __restrict__ pkey,
                                                            const uint32_t* __restrict__ ppid,
                                                            const uint32_t* __restrict__ pstart, uint32_t n,
                                                            uint32_t* plist) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (ppid[i] != RX_CROSS) plist[pstart[ppid[i]] + pkey[i]] = i;
}
// one thread (TPC-C: one warp) per partition runs its transactions in key order; the
// partition-major list is also the serialization order of this phase
template <int S>
__global__ void __launch_bounds__(128) rpart_exec_kernel(DevDb db, const uint32_t* __restrict__ plist,
                                                         const uint32_t* __restrict__ pstart, uint32_t nparts,
                                                         uint32_t* order, uint32_t* sc) {
    if (S == S_TPCC) {
        const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        if (p >= nparts) return;
        const uint32_t lo = pstart[p], hi = pstart[p + 1];
        for (uint32_t k = lo; k < hi; ++k) {
            const uint32_t idx = __ldg(&plist[k]);
            if (lane_id() == 0) order[k] = idx;
            exec_txn_warp<false>(db, idx);
        }
        if (lane_id() == 0 && hi > lo) atomicMax(&sc[SC_MAXCHAIN], hi - lo);
    } else {
        const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
        if (p >= nparts) return;
        const uint32_t lo = pstart[p], hi = pstart[p + 1];
        for (uint32_t k = lo; k < hi; ++k) {
            const uint32_t idx = __ldg(&plist[k]);
            order[k] = idx;
            exec_txn<S, false>(db, idx);
        }
        if (hi > lo) atomicMax(&sc[SC_MAXCHAIN], hi - lo);
    }
}
}  // namespace gputx

namespace gputx {
// =====================================================================================
// Peer-memory exchange (fused): every shard owns an ARENA in its
// HBM -- per-source arrival flags, a record counter and a record area for the cross-shard
// transactions it receives, the same for returned fragment outputs.  The producing kernel
// writes each record straight into the destination shard's arena (P2P stores over NVLink /
// NVSwitch; same-device stores when the shards share a GPU), reserving its slot with a
// system-scope atomic on the destination's counter; the kernel's last CTA then publishes
// the epoch to every peer (release at system scope).  No host staging, no all-to-all call.
// =====================================================================================
constexpr uint32_t AR_FWD_FLAGS = 0;      // [MAX_SHARDS] x 32 words (own 128-B lines)
constexpr uint32_t AR_RET_FLAGS = 256;
constexpr uint32_t AR_FWD_CNT = 512;
constexpr uint32_t AR_RET_CNT = 544;
constexpr uint32_t AR_OVF = 576;          // overflow: a sender found the record area full
constexpr uint32_t AR_HDR = 640;          // record areas start here (words)
struct PeerTable {
    uint32_t* arena[MAX_SHARDS];           // every shard's arena as seen from this process
    uint64_t ret_base[MAX_SHARDS];         // its geometry (arenas are sized by each shard's max_bulk)
    uint32_t fwd_cap[MAX_SHARDS], ret_cap[MAX_SHARDS];
};
DEV void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
DEV uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// last-CTA publication: every CTA fences its P2P stores at system scope and counts itself;
// the last one (after the acquire fence) stores the epoch into flag[self] of every peer
DEV void p2p_publish(const PeerTable& pt, uint32_t off_flags, uint32_t self, uint32_t G, uint32_t epoch,
                     uint32_t* done_ctas) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const uint32_t prev = atomicAdd(done_ctas, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence_system();
            *done_ctas = 0;                                   // reusable by the next exchange
            for (uint32_t q = 0; q < G; ++q)
                if (q != self) st_release_sys(&pt.arena[q][off_flags + self * 32], epoch);
        }
    }
}

// C1+C2 fused with the pack: [ts, type, len, params] of every (home transaction, remote
// shard owning one of its fragments) into that shard's arena.  Thread 0 of CTA 0 also
// clears this shard's return counter for the coming return exchange (all peers' returns of
// the previous epoch were merged before this dispatch).
template <int S>
__global__ void __launch_bounds__(256) p2p_dispatch_kernel(DevDb db, const uint8_t* __restrict__ type,
        const uint32_t* __restrict__ poff, const uint32_t* __restrict__ pw, const uint32_t* __restrict__ ts,
        uint32_t nh, PeerTable pt, uint32_t self, uint32_t G, uint32_t stride, uint32_t epoch, uint32_t* done_ctas) {
    if (blockIdx.x == 0 && threadIdx.x == 0) pt.arena[self][AR_RET_CNT] = 0;
    const uint32_t maxlen = stride - 3;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nh; i += gridDim.x * blockDim.x) {
        const uint32_t len = shard_len(poff, i, maxlen);
        uint32_t m = dest_mask<S>(db, type[i], pw + poff[i], len) & ~(1u << self);
        while (m) {
            const uint32_t q = __ffs(m) - 1;
            m &= m - 1;
            uint32_t* ar = pt.arena[q];
            const uint32_t slot = atomicAdd_system(&ar[AR_FWD_CNT], 1u);
            if (slot >= pt.fwd_cap[q]) { atomicOr_system(&ar[AR_OVF], 1u); continue; }
            uint32_t* r = ar + AR_HDR + (uint64_t)slot * stride;
            r[0] = ts[i];
            r[1] = type[i];
            r[2] = len;
            const uint32_t* src = pw + poff[i];
            for (uint32_t w = 0; w < len; ++w) r[3 + w] = src[w];
        }
    }
    p2p_publish(pt, AR_FWD_FLAGS, self, G, epoch, done_ctas);
}

// C3 fused: the output record of every peer's transaction executed here goes straight into
// its home shard's arena; thread 0 of CTA 0 clears this shard's forward counter (the
// records it received for this epoch were merged before the execution).
template <int S>
__global__ void __launch_bounds__(256) p2p_return_kernel(DevDb db, PeerTable pt, uint32_t self, uint32_t G,
                                                         uint32_t ow, uint32_t epoch, uint32_t* done_ctas) {
    if (blockIdx.x == 0 && threadIdx.x == 0) pt.arena[self][AR_FWD_CNT] = 0;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < db.n; k += gridDim.x * blockDim.x) {
        if (db.src[k] != NOT_HOME) continue;
        const uint32_t* p = db.pw + db.poff[k];
        const uint32_t q = shard_of(db, S == S_TPCB ? p[2] : p[0]);
        uint32_t* ar = pt.arena[q];
        const uint32_t slot = atomicAdd_system(&ar[AR_RET_CNT], 1u);
        if (slot >= pt.ret_cap[q]) { atomicOr_system(&ar[AR_OVF], 2u); continue; }
        uint32_t* r = ar + pt.ret_base[q] + (uint64_t)slot * (1 + ow);
        r[0] = db.ts[k];
        const uint32_t* o = reinterpret_cast<const uint32_t*>(db.out + (uint64_t)k * ow * 4);
        for (uint32_t w = 0; w < ow; ++w) r[1 + w] = o[w];
    }
    p2p_publish(pt, AR_RET_FLAGS, self, G, epoch, done_ctas);
}

// wait until every peer published `epoch` (watchdog -> SC_DEADLOCK), then copy the count
__global__ void p2p_wait_kernel(uint32_t* arena, uint32_t off_flags, uint32_t off_cnt, uint32_t self, uint32_t G,
                                uint32_t epoch, uint32_t* sc, uint32_t* cnt_out) {
    const uint32_t q = threadIdx.x;
    if (q < G && q != self) {
        SpinWatch wd;
        while (ld_acquire_sys(&arena[off_flags + q * 32]) < epoch)
            if (wd.expired(&sc[SC_DEADLOCK])) break;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        *cnt_out = ld_acquire_sys(&arena[off_cnt]);
        cnt_out[1] = ld_acquire_sys(&arena[AR_OVF]);
    }
}
}  // namespace gputx

namespace gputx {
// TM-1 row groups <-> columns (schema.cuh "TM-1 rows"): pack all fields at seal / reset,
// unpack the mutable ones (vlr, bits, sf.data_a, cf live / end / numberx) before a read
__global__ void __launch_bounds__(256) tm1_pack_kernel(DevDb db) {
    const uint32_t P = db.dims[0];
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < P; s += gridDim.x * blockDim.x) {
        uint8_t* r = db.tm1_sub + (uint64_t)s * TM1_SUBROW;
        *reinterpret_cast<uint64_t*>(r) = COL(const uint64_t, M_NBR)[s];
        *reinterpret_cast<uint64_t*>(r + 8) = COL(const uint64_t, M_HEX)[s];
        *reinterpret_cast<uint32_t*>(r + 16) = COL(const uint32_t, M_MSC)[s];
        *reinterpret_cast<uint32_t*>(r + 20) = COL(const uint32_t, M_VLR)[s];
        *reinterpret_cast<uint16_t*>(r + 24) = COL(const uint16_t, M_BITS)[s];
        for (int k = 0; k < 10; ++k) r[26 + k] = COL(const uint8_t, M_BYTE2)[(uint64_t)s * 10 + k];
        for (int k = 36; k < (int)TM1_SUBROW; ++k) r[k] = 0;
        for (uint32_t j = 0; j < 4; ++j) {
            const uint64_t f = (uint64_t)s * 4 + j;
            uint8_t* a = db.tm1_ai + f * TM1_AIROW;
            a[0] = COL(const uint8_t, M_AI_VALID)[f]; a[1] = COL(const uint8_t, M_AI_D1)[f];
            a[2] = COL(const uint8_t, M_AI_D2)[f]; a[3] = 0;
            *reinterpret_cast<uint32_t*>(a + 4) = COL(const uint32_t, M_AI_D3)[f];
            *reinterpret_cast<uint64_t*>(a + 8) = COL(const uint64_t, M_AI_D4)[f];
            uint8_t* g = db.tm1_sf + f * TM1_SFROW;
            g[0] = COL(const uint8_t, M_SF_VALID)[f]; g[1] = COL(const uint8_t, M_SF_ACTIVE)[f];
            g[2] = COL(const uint8_t, M_SF_ERR)[f]; g[3] = COL(const uint8_t, M_SF_DA)[f];
            *reinterpret_cast<uint32_t*>(g + 4) = 0;
            *reinterpret_cast<uint64_t*>(g + 8) = COL(const uint64_t, M_SF_DB)[f];
            uint8_t* c = db.tm1_cf + f * TM1_CFROW;
            for (int k = 0; k < 16; ++k) c[k] = 0;
            for (int k = 0; k < 3; ++k) {
                c[k] = COL(const uint8_t, M_CF_LIVE)[f * 3 + k];
                c[4 + k] = COL(const uint8_t, M_CF_END)[f * 3 + k];
                *reinterpret_cast<uint64_t*>(c + 16 + 8 * k) = COL(const uint64_t, M_CF_NUM)[f * 3 + k];
            }
            *reinterpret_cast<uint64_t*>(c + 40) = 0;
            *reinterpret_cast<uint64_t*>(c + 48) = 0;
            *reinterpret_cast<uint64_t*>(c + 56) = 0;
        }
    }
}
__global__ void __launch_bounds__(256) tm1_unpack_kernel(DevDb db) {
    const uint32_t P = db.dims[0];
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < P; s += gridDim.x * blockDim.x) {
        const uint8_t* r = db.tm1_sub + (uint64_t)s * TM1_SUBROW;
        COL(uint32_t, M_VLR)[s] = *reinterpret_cast<const uint32_t*>(r + 20);
        COL(uint16_t, M_BITS)[s] = *reinterpret_cast<const uint16_t*>(r + 24);
        for (uint32_t j = 0; j < 4; ++j) {
            const uint64_t f = (uint64_t)s * 4 + j;
            COL(uint8_t, M_SF_DA)[f] = db.tm1_sf[f * TM1_SFROW + 3];
            const uint8_t* c = db.tm1_cf + f * TM1_CFROW;
            for (int k = 0; k < 3; ++k) {
                COL(uint8_t, M_CF_LIVE)[f * 3 + k] = c[k];
                COL(uint8_t, M_CF_END)[f * 3 + k] = c[4 + k];
                COL(uint64_t, M_CF_NUM)[f * 3 + k] = *reinterpret_cast<const uint64_t*>(c + 16 + 8 * k);
            }
        }
    }
}
}  // namespace gputx
