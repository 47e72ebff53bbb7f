// schema.cuh — the registered stored procedures of the three benchmarks as device
// functions, combined per schema into one switch(type) (§3.2),
// their conflict footprints (basic operations, §4.1; Fekete-style
// static analysis PAPER.md:457 -> only columns some type writes produce an
// operation, DESIGN.md R-S18) and their fragment split for PART (DESIGN.md R-S9).
//
// Column store: one HBM array per fixed-length column, row
// index = primary key position.  All procedures are two-phase:
// every abort decision is taken before the first write.
#pragma once
#include <cstdint>
#include "common.cuh"

namespace gputx {

enum Schema { S_TPCB = 1, S_TM1 = 2, S_TPCC = 3, S_MICRO = 4 };
constexpr uint32_t MICRO_MAX_TYPES = 32;     // T: branches of the micro benchmark's switch

// ---- column indices (must match the catalog in engine.cu) -----------------------
enum { B_BR = 0, B_TEL, B_ACC, B_NCOL };
enum { U_TUPLE = 0, U_NCOL };
enum { M_NBR = 0, M_BITS, M_HEX, M_BYTE2, M_MSC, M_VLR, M_AI_VALID, M_AI_D1, M_AI_D2, M_AI_D3, M_AI_D4,
       M_SF_VALID, M_SF_ACTIVE, M_SF_ERR, M_SF_DA, M_SF_DB, M_CF_LIVE, M_CF_END, M_CF_NUM, M_NCOL };
enum { C_W_YTD = 0, C_W_TAX, C_D_YTD, C_D_TAX, C_D_NEXT, C_C_BAL, C_C_YTD, C_C_CNT, C_C_DISC, C_C_CREDIT,
       C_C_LAST, C_C_FIRST, C_I_PRICE, C_I_ORIG, C_S_QTY, C_S_YTD, C_S_OCNT, C_S_RCNT, C_S_ORIG, C_NCOL };
// insert columns: TPC-B history 0..4; TPC-C order 0..6, new_order 7..9, order_line 10..17, history 18..24
enum { IB_TID = 0, IB_BID, IB_AID, IB_DELTA, IB_TS };
enum { IO_ID = 0, IO_D, IO_W, IO_C, IO_ENTRY, IO_OLCNT, IO_ALLLOCAL,
       IN_OID = 7, IN_D, IN_W,
       IL_OID = 10, IL_D, IL_W, IL_NUM, IL_I, IL_SW, IL_QTY, IL_AMT,
       IH_C = 18, IH_CD, IH_CW, IH_D, IH_W, IH_DATE, IH_AMT };
enum { T_ORDER = 0, T_NEWORDER = 1, T_OLINE = 2, T_HIST = 3 };

constexpr int MAX_COLS = 32;
constexpr int MAX_INS = 32;
constexpr int MAX_REC = 16;            // access records per transaction (TPC-C NO: 1 + 15)

struct DevDb {
    int schema;
    uint32_t dims[4];
    uint32_t ntypes;
    uint32_t n;                        // transactions in the bulk
    uint32_t first_ts;
    const uint8_t* type;
    const uint32_t* poff;
    const uint32_t* pw;
    uint8_t* status;
    uint8_t* out;
    uint32_t out_stride;
    const uint32_t* out_off;           // GPUTX_FLAG_PACKED_OUT: record offsets (else nullptr: idx * stride)
    void* col[MAX_COLS];
    void* ins[MAX_INS];
    uint64_t ins_base[4];              // merged-table row count before this bulk
    const uint32_t* ins_off;           // [table][ins_stride] exclusive row offsets within this bulk
    uint32_t ins_stride;
    const uint64_t* hkeys;             // TM-1 sub_nbr hash (open addressing)
    const uint32_t* hvals;
    uint64_t hmask;
    const uint32_t* name_sorted;       // TPC-C customers of (w,d) sorted by (c_last, c_first, c)
    const uint32_t* name_off;          // [(w*D+d)*1000 + last] -> range start, +1 -> end
    uint32_t part_size;
    // shards: this shard owns root keys [root_lo, root_hi) of nroot
    // (root = TPC-B branch, TPC-C warehouse, TM-1 subscriber - 1), shard_of(r) = r*G/nroot
    uint32_t nshards, shard, nroot, root_lo, root_hi;
    uint32_t add_rule;                 // GPUTX_FLAG_ADD_RULE: increments-only items in mode "add"
    const uint32_t* ts;                // global timestamps (NULL: first_ts + idx)
    const uint32_t* src;               // sharded: home-bulk index, or NOT_HOME (a peer's transaction)
    const uint8_t* xflag;              // sharded: 1 = some fragment lives on another shard
    uint32_t idx_base;                 // emit: record idx = idx_base + i (pool arrivals; 0 otherwise)
    // pipelined gputx_run_bulks (no host round trip between ingest and execute): the
    // kernels that read parameters treat the bulk as empty once ingest flagged an error
    // (*err = sc[SC_ERR]); *poison makes every later bulk of the run fail at ingest
    const uint32_t* err;
    uint32_t* poison;
    struct UndoRec* undo;              // per-transaction undo-log slots (non-two-phase types)
    uint32_t ins_dense;                // TPC-B: every transaction is a home deposit -> history row = idx
    uint8_t *tm1_sub, *tm1_ai, *tm1_sf, *tm1_cf;   // TM-1 row groups (tm1_txn)
};

// Undo log: written in GPU memory before each update of a NON-two-phase
// transaction and discarded at commit; on abort the transaction replays it backwards.
// RESTORE puts back the value it overwrote (exclusively held items); ADD compensates an
// increment (items other transactions may increment concurrently under the ADD rule).
enum { UNDO_RESTORE = 0, UNDO_ADD = 1 };
struct UndoRec {
    uint32_t col, kind;
    uint64_t row;
    int64_t val;
};
constexpr int UNDO_SLOTS = 3;          // records per transaction (TPC-B WITHDRAW: account, teller, branch)
constexpr uint32_t NOT_HOME = 0xFFFFFFFFu;

// sh (compile-time in the fused kernels): the bulk carries explicit timestamps (sharded or
// caller-given), insert rows of TPC-B come from ins_off, and cross-shard transactions
// run their local fragments only
DEV uint32_t txn_ts(const DevDb& db, uint32_t idx, bool sh) { return sh ? db.ts[idx] : db.first_ts + idx; }
DEV bool root_local(const DevDb& db, uint64_t root) { return root >= db.root_lo && root < db.root_hi; }
DEV uint32_t shard_of(const DevDb& db, uint64_t root) { return (uint32_t)(root * db.nshards / db.nroot); }

#define COL(T, k) (reinterpret_cast<T*>(db.col[(k)]))
#define INS(T, k) (reinterpret_cast<T*>(db.ins[(k)]))

// Mutable column access.  Plain (weak) loads/stores: every strategy orders conflicting
// accesses with acquire/release synchronisation (k-set round hand-off, cluster
// barrier, counter-lock acquire), whose acquire side invalidates L1, so a weak load
// after it sees the earlier writer.  (ld.global.cg compiles to LDG.E.STRONG.GPU on
// sm_100a, and those serialise the lanes of a warp: 8 NewOrders in one warp took 10x
// the time of 8 in 8 warps.)
template <class T> DEV T ldm(const T* p) { return *p; }
template <class T> DEV void stm(T* p, T v) { *p = v; }
DEV void put32(uint8_t* o, uint32_t v) { *reinterpret_cast<uint32_t*>(o) = v; }
// GPUTX_FLAG_PACKED_OUT record size of a transaction (include/gputx.h): the bytes its
// procedure can write, rounded to the record's alignment
template <int S>
DEV uint32_t out_bytes(uint32_t t, const uint32_t* p) {
    if (S == S_TPCB) return 8;
    if (S == S_MICRO) return 4;
    if (S == S_TM1) return t == 0 ? 40u : t == 1 ? 32u : t == 2 ? 16u : 0u;
    return t == 0 ? (16u + 12u * p[3] + 7u) & ~7u : 16u;
}
// pipelined run_bulks: a bulk whose ingest failed is executed as empty
DEV bool bulk_failed(const DevDb& db) { return db.err && __ldcg(db.err) != 0u; }
// transaction idx's output record: fixed stride, or packed at its submit-time offset --
// `oo` when the caller staged it (OUT_AUTO: loaded here, a dependent load before the store)
constexpr uint32_t OUT_AUTO = 0xFFFFFFFFu;
template <uint32_t STRIDE>
DEV uint8_t* out_rec(const DevDb& db, uint32_t idx, uint32_t oo = OUT_AUTO) {
    if (oo != OUT_AUTO) return db.out + oo;
    return db.out + (db.out_off ? (uint64_t)__ldg(&db.out_off[idx]) : (uint64_t)idx * STRIDE);
}
DEV void put64(uint8_t* o, uint64_t v) {
    reinterpret_cast<uint32_t*>(o)[0] = (uint32_t)v;
    reinterpret_cast<uint32_t*>(o)[1] = (uint32_t)(v >> 32);
}

// =================================================================================
// Item space (dense, per schema) and access records
//   record key = item << 30 | idx << 6 | j << 2 | mode     (0 read, 1 write, 2 add)
// =================================================================================
constexpr int KEY_ITEM_SHIFT = 30;
DEV uint64_t make_key(uint64_t item, uint32_t idx, uint32_t j, uint32_t w) {
    return (item << KEY_ITEM_SHIFT) | ((uint64_t)idx << 6) | ((uint64_t)j << 2) | w;
}
DEV uint64_t key_item(uint64_t k) { return k >> KEY_ITEM_SHIFT; }
DEV uint32_t key_idx(uint64_t k) { return (uint32_t)(k >> 6) & 0xFFFFFFu; }
DEV uint32_t key_j(uint64_t k) { return (uint32_t)(k >> 2) & 0xFu; }
DEV uint32_t key_w(uint64_t k) { return (uint32_t)k & 1u; }
DEV uint32_t key_mode(uint64_t k) { return (uint32_t)k & 3u; }    // 0 read, 1 write, 2 add

struct Rec {
    uint64_t item;
    uint32_t w;        // mode: 0 read, 1 write, 2 add
};

DEV int add_rec(Rec* r, int k, uint64_t item, uint32_t w) {
    for (int j = 0; j < k; ++j)
        if (r[j].item == item) { if (r[j].w != w) r[j].w = 1u; return k; }   // one record; modes differ -> W
    r[k].item = item;
    r[k].w = w;
    return k + 1;
}

// Item ids are partition-major (subscriber / branch / warehouse): all items of one
// root key are adjacent, so the conflict groups a transaction touches sit in the same
// sorted tile and the rank kernel's in-tile iteration resolves their chains on chip.
//   TM-1 : s*32 + {0 BIT1, 1 VLR, 2+sf-1 SFDA, 8+(sf-1)*4+st/8 CF}   (18 of 32 slots: the
//          subscriber is the item id's high bits, so a sort on them alone gives (root, ts))
//   TPC-B: b*(1+T+A) + {0 BR, 1+t TEL, 1+T+a ACC}
//   TPC-C: w*(2D+1+DC+I) + {d DNEXT, D WYTD, D+1+d DYTD, 2D+1+d*C+c CUST, 2D+1+DC+i STOCK}
constexpr uint32_t TM1_SLOT_BITS = 5;
constexpr uint64_t TM1_STRIDE = 1u << TM1_SLOT_BITS;
// A TM-1 transaction touches one of a subscriber's independent item components: {BIT1,
// VLR, SFDA*} (GSD, USD, UL; slots 0-7) or the CF slots of one sf (GND, ICF, DCF; slots
// 8 + 4(sf-1) + st/8).  Slot >> 3 separates {A}, {CF sf 1, 2}, {CF sf 3, 4}: components
// share no transaction, so their depths are independent (streaming rank walks each alone).
constexpr uint32_t TM1_COMP_BITS = 3;
// Basic operations of one (ingested) transaction.  Returns the count (<= MAX_REC).
template <int S>
DEV int footprint(const DevDb& db, uint32_t t, const uint32_t* p, Rec* r) {
    int k = 0;
    // ADD rule: balances / YTDs only incremented by their type and never read by an output
    const uint32_t inc = db.add_rule ? 2u : 1u;
    if (S == S_TPCB) {
        const uint32_t T = db.dims[1], A = db.dims[2];
        const uint64_t sb = 1ull + T + A;
        r[0] = {(uint64_t)(p[0] / A) * sb + 1 + T + p[0] % A, 1u};
        r[1] = {(uint64_t)(p[1] / T) * sb + 1 + p[1] % T, inc};
        r[2] = {(uint64_t)p[2] * sb, inc};
        return 3;
    } else if (S == S_MICRO) {
        r[0] = {(uint64_t)p[0], 1u};                    // read, compute, write back the tuple
        return 1;
    } else if (S == S_TM1) {
        switch (t) {
        case 0: { uint64_t s = (uint64_t)(p[0] - 1) * TM1_STRIDE; r[0] = {s, 0u}; r[1] = {s + 1, 0u}; return 2; }
        case 1: {
            uint64_t c = (uint64_t)(p[0] - 1) * TM1_STRIDE + 8 + (p[1] - 1) * 4;
            r[0] = {c, 0u}; r[1] = {c + 1, 0u}; r[2] = {c + 2, 0u};
            return 3;
        }
        case 2: return 0;
        case 3: { uint64_t s = (uint64_t)(p[0] - 1) * TM1_STRIDE; r[0] = {s, 1u}; r[1] = {s + 2 + (p[1] - 1), 1u}; return 2; }
        case 4: if (p[0] == 0) return 0; r[0] = {(uint64_t)(p[0] - 1) * TM1_STRIDE + 1, 1u}; return 1;
        case 5: case 6:
            if (p[0] == 0) return 0;
            r[0] = {(uint64_t)(p[0] - 1) * TM1_STRIDE + 8 + (p[2] - 1) * 4 + p[3] / 8, 1u};
            return 1;
        }
        return 0;
    } else {
        const uint64_t D = db.dims[1], C = db.dims[2], I = db.dims[3];
        const uint64_t sw_ = 2 * D + 1 + D * C + I;
        if (t == 0) {
            k = add_rec(r, k, (uint64_t)p[0] * sw_ + p[1], 1u);
            const uint32_t cnt = p[3];
            for (uint32_t l = 0; l < cnt; ++l) {
                uint32_t i = p[4 + 3 * l], sw = p[5 + 3 * l];
                if (i >= I) continue;
                k = add_rec(r, k, (uint64_t)sw * sw_ + 2 * D + 1 + D * C + i, 1u);
            }
            return k;
        }
        r[0] = {(uint64_t)p[0] * sw_ + D, inc};
        r[1] = {(uint64_t)p[0] * sw_ + D + 1 + p[1], inc};
        if (p[4] == 2) return 2;                           // by-name lookup found nobody
        r[2] = {(uint64_t)p[2] * sw_ + 2 * D + 1 + (uint64_t)p[3] * C + p[5], 1u};
        return 3;
    }
}

// root key of an item (see the item layout above)
template <int S>
DEV uint64_t item_root(const DevDb& db, uint64_t item) {
    if (S == S_TPCB) return item / (1ull + db.dims[1] + db.dims[2]);
    if (S == S_TM1) return item >> TM1_SLOT_BITS;
    if (S == S_MICRO) return item;
    const uint64_t D = db.dims[1];
    return item / (2 * D + 1 + D * db.dims[2] + db.dims[3]);
}

// the records of the transaction's items on this shard (all of them when unsharded)
template <int S>
DEV int footprint_local(const DevDb& db, uint32_t t, const uint32_t* p, Rec* r) {
    const int k = footprint<S>(db, t, p, r);
    if (db.nshards <= 1) return k;
    int m = 0;
    for (int j = 0; j < k; ++j)
        if (root_local(db, item_root<S>(db, r[j].item))) r[m++] = r[j];
    return m;
}

// =================================================================================
// Stored procedures (whole transaction; K-SET and TPL)
// =================================================================================
// Every procedure issues all of its reads first (static columns speculatively), then
// takes its abort decision, then writes: the loads of one transaction overlap in
// flight instead of serialising behind stores.  Increments whose old value no output
// needs are fire-and-forget reductions (red.global.add) — the transaction holds the
// item exclusively (k-set round, TPL lock, PART partition), so this is plain RMW
// without a round trip.
DEV void red_add(int64_t* p, int64_t v) { atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v); }
DEV void red_add(uint32_t* p, uint32_t v) { atomicAdd(p, v); }

DEV void tpcb_home(const DevDb& db, uint32_t idx, const uint32_t* p, bool sh) {
    const int32_t delta = (int32_t)p[3];
    red_add(&COL(int64_t, B_TEL)[p[1]], (int64_t)delta);
    red_add(&COL(int64_t, B_BR)[p[2]], (int64_t)delta);
    // history row: deposits always commit; the row is the deposit's position among the bulk's
    // (home) deposits -- WITHDRAWs insert nothing (ingest counts, exclusive scan)
    (void)sh;
    const uint64_t r = db.ins_base[0] + (db.ins_dense ? idx : db.ins_off[idx]);
    INS(uint32_t, IB_TID)[r] = p[1];
    INS(uint32_t, IB_BID)[r] = p[2];
    INS(uint32_t, IB_AID)[r] = p[0];
    INS(int32_t, IB_DELTA)[r] = delta;
    INS(uint32_t, IB_TS)[r] = txn_ts(db, idx, sh);
}
DEV void tpcb_account(const DevDb& db, uint32_t idx, const uint32_t* p, uint32_t oo = OUT_AUTO) {
    int64_t* acc = COL(int64_t, B_ACC);
    const int64_t v = ldm(&acc[p[0]]) + (int32_t)p[3];
    stm(&acc[p[0]], v);
    *reinterpret_cast<int64_t*>(out_rec<8>(db, idx, oo)) = v;
}

// WITHDRAW (TPC-B type 1): NON-two-phase on purpose --
// it debits account, teller and branch and only then checks that the account did not go
// negative; an abort rolls its own updates back from the undo log.  Every strategy runs
// it with the items held exclusively (k-set round, PART partition, TPL locks held through
// the rollback), so no other transaction saw the dirty values and the recovery affects
// the transaction alone (DESIGN.md R-U1).
DEV void undo_apply(const DevDb& db, const UndoRec* log, int nl) {
    for (int j = nl - 1; j >= 0; --j) {
        int64_t* c = reinterpret_cast<int64_t*>(db.col[log[j].col]);
        if (log[j].kind == UNDO_RESTORE) stm(&c[log[j].row], log[j].val);
        else red_add(&c[log[j].row], log[j].val);
    }
}
DEV void tpcb_withdraw(const DevDb& db, uint32_t idx, const uint32_t* p, uint32_t oo = OUT_AUTO) {
    UndoRec* log = db.undo + (uint64_t)idx * UNDO_SLOTS;
    const int64_t amt = (int32_t)p[3];
    int64_t* acc = COL(int64_t, B_ACC);
    const int64_t a0 = ldm(&acc[p[0]]);
    log[0] = {B_ACC, UNDO_RESTORE, p[0], a0};          // log first, then update
    stm(&acc[p[0]], a0 - amt);
    log[1] = {B_TEL, UNDO_ADD, p[1], amt};
    red_add(&COL(int64_t, B_TEL)[p[1]], -amt);
    log[2] = {B_BR, UNDO_ADD, p[2], amt};
    red_add(&COL(int64_t, B_BR)[p[2]], -amt);
    const int64_t a1 = ldm(&acc[p[0]]);                // the check reads the updated row
    if (a1 < 0) {
        undo_apply(db, log, UNDO_SLOTS);
        db.status[idx] = 1;
        *reinterpret_cast<int64_t*>(out_rec<8>(db, idx, oo)) = 0;   // (TPC-B output records are not pre-zeroed)
        return;
    }
    *reinterpret_cast<int64_t*>(out_rec<8>(db, idx, oo)) = a1;
}

// ---- TM-1 --------------------------------------------------------------------------
// TM-1 rows (DESIGN.md §5 "TM-1 row groups"): the fields one TATP procedure reads lie in
// one aligned row, so a transaction moves 1-3 sectors with 16-byte vector loads instead of
// ~10 scattered column accesses (the wide 0-set round was bound by L1 wavefronts: 23
// sectors per warp request).  The column store stays the interface (load / read / reset);
// rows are built at seal and after a reset, and unpacked into the mutable columns before
// they are read.
//   SUB (64 B)  [0] nbr u64 [8] hex u64 [16] msc u32 [20] vlr u32 [24] bits u16 [26] byte2[10]
//               -- bytes [0, 36) are exactly GSD's output record
//   AI  (16 B)  [0] valid [1] data1 [2] data2 [4] data3 u32 [8] data4 u64
//   SF  (16 B)  [0] valid [1] active [2] error [3] data_a [8] data_b u64
//   CF  (64 B per (s, sf)) [0..3) live, [4..7) end_time, [16 + 8k] numberx of start 8k
constexpr uint32_t TM1_SUBROW = 64, TM1_AIROW = 16, TM1_SFROW = 16, TM1_CFROW = 64;

DEV void tm1_txn(const DevDb& db, uint32_t idx, uint32_t t, const uint32_t* p, uint32_t oo = OUT_AUTO) {
    uint8_t* o = out_rec<40>(db, idx, oo);
    switch (t) {
    case 0: {   // GET_SUBSCRIBER_DATA: the row's first 36 bytes are the output record
        const uint32_t s = p[0] - 1;
        const uint4* row = reinterpret_cast<const uint4*>(db.tm1_sub + (uint64_t)s * TM1_SUBROW);
        const uint4 a = row[0], b = row[1], c = row[2];        // (vlr, bits live in b: weak loads)
        uint2* q = reinterpret_cast<uint2*>(o);                // out + idx*40 is 8-byte aligned
        q[0] = make_uint2(a.x, a.y);
        q[1] = make_uint2(a.z, a.w);
        q[2] = make_uint2(b.x, b.y);
        q[3] = make_uint2(b.z, b.w);
        q[4] = make_uint2(c.x, 0u);
        return;
    }
    case 1: {   // GET_NEW_DESTINATION
        const uint64_t f = (uint64_t)(p[0] - 1) * 4 + (p[1] - 1);
        const uint4 sf = *reinterpret_cast<const uint4*>(db.tm1_sf + f * TM1_SFROW);
        const uint4* cf = reinterpret_cast<const uint4*>(db.tm1_cf + f * TM1_CFROW);
        const uint4 h = cf[0], n01 = cf[1], n2 = cf[2];
        const uint32_t valid = sf.x & 0xFFu, active = (sf.x >> 8) & 0xFFu;
        if (!valid || !active) { db.status[idx] = 1; return; }
        const uint64_t num[3] = {(uint64_t)n01.x | ((uint64_t)n01.y << 32), (uint64_t)n01.z | ((uint64_t)n01.w << 32),
                                 (uint64_t)n2.x | ((uint64_t)n2.y << 32)};
        uint32_t cnt = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const uint32_t live = (h.x >> (8 * k)) & 0xFFu, endt = (h.y >> (8 * k)) & 0xFFu;
            if (live && (uint32_t)k * 8 <= p[2] && p[3] < endt) {
                put64(o + 8 + 8 * cnt, num[k]);
                ++cnt;
            }
        }
        if (cnt == 0) { db.status[idx] = 1; return; }
        put32(o, cnt);
        return;
    }
    case 2: {   // GET_ACCESS_DATA
        const uint64_t a = (uint64_t)(p[0] - 1) * 4 + (p[1] - 1);
        const uint4 r = *reinterpret_cast<const uint4*>(db.tm1_ai + a * TM1_AIROW);
        if (!(r.x & 0xFFu)) { db.status[idx] = 1; return; }
        uint2* q = reinterpret_cast<uint2*>(o);
        q[0] = make_uint2((r.x >> 8) & 0xFFFFu, r.y);          // data1, data2 | data3
        q[1] = make_uint2(r.z, r.w);                            // data4
        return;
    }
    case 3: {   // UPDATE_SUBSCRIBER_DATA (two-phase: SF existence first)
        const uint32_t s = p[0] - 1;
        const uint64_t f = (uint64_t)s * 4 + (p[1] - 1);
        uint16_t* bits = reinterpret_cast<uint16_t*>(db.tm1_sub + (uint64_t)s * TM1_SUBROW + 24);
        const uint8_t valid = db.tm1_sf[f * TM1_SFROW];
        const uint16_t b = ldm(bits);
        if (!valid) { db.status[idx] = 1; return; }
        stm(bits, (uint16_t)((b & 0xFFFEu) | (p[2] & 1u)));
        stm(db.tm1_sf + f * TM1_SFROW + 3, (uint8_t)p[3]);
        return;
    }
    case 4: {   // UPDATE_LOCATION (sub_nbr resolved at submit)
        if (p[0] == 0) { db.status[idx] = 1; return; }
        stm(reinterpret_cast<uint32_t*>(db.tm1_sub + (uint64_t)(p[0] - 1) * TM1_SUBROW + 20), p[2]);
        return;
    }
    case 5: {   // INSERT_CALL_FORWARDING
        if (p[0] == 0) { db.status[idx] = 1; return; }
        const uint64_t f = (uint64_t)(p[0] - 1) * 4 + (p[2] - 1);
        const uint32_t k = p[3] / 8;
        uint8_t* cf = db.tm1_cf + f * TM1_CFROW;
        const uint8_t valid = db.tm1_sf[f * TM1_SFROW];
        const uint8_t lv = ldm(cf + k);
        if (!valid || lv) { db.status[idx] = 1; return; }
        stm(cf + k, (uint8_t)1);
        stm(cf + 4 + k, (uint8_t)p[4]);
        stm(reinterpret_cast<uint64_t*>(cf + 16 + 8 * k), (uint64_t)p[5] | ((uint64_t)p[6] << 32));
        return;
    }
    case 6: {   // DELETE_CALL_FORWARDING
        if (p[0] == 0) { db.status[idx] = 1; return; }
        uint8_t* cf = db.tm1_cf + ((uint64_t)(p[0] - 1) * 4 + (p[2] - 1)) * TM1_CFROW;
        const uint32_t k = p[3] / 8;
        if (!ldm(cf + k)) { db.status[idx] = 1; return; }
        stm(cf + k, (uint8_t)0);
        return;
    }
    }
}

// ---- Micro benchmark (§6.1) -------------------------------------------
// "Each transaction reads a tuple, and performs computation, and then writes the result
// back to the tuple.  The amount of computation is simulated with calling the _sinf
// function (100 * x) times."  One call of type t (DESIGN.md R-M1): u = fma(v, A_t, B_t),
// then sin(u) ~ u * (1 + s (C3 + s C5)), s = u^2 -- every operation IEEE round-to-nearest
// (__fmaf_rn / __fmul_rn: no contraction), so the result is bit-exact against the C
// oracle.  Each type is its own instantiation with its constants as immediates, so the
// T cases of the combined switch are T distinct code paths (the paper makes sure "the
// branches are not eliminated by code optimization"): lanes of one warp with different
// types serialise, which is what type grouping removes.
template <uint32_t TT>
__device__ __noinline__ float micro_body(float v, uint32_t calls) {
    constexpr float A = 0.9375f - (float)TT * 0.0078125f;
    constexpr float B = ((float)TT - 15.5f) * 0.0009765625f;
    constexpr float C3 = -0x1.555556p-3f, C5 = 0x1.111112p-7f;
#pragma unroll 1
    for (uint32_t j = 0; j < calls; ++j) {
        const float u = __fmaf_rn(v, A, B);
        const float s2 = __fmul_rn(u, u);
        float q = __fmaf_rn(s2, C5, C3);
        q = __fmaf_rn(s2, q, 1.0f);
        v = __fmul_rn(u, q);
    }
    return v;
}

DEV void micro_txn(const DevDb& db, uint32_t idx, uint32_t t, const uint32_t* p, uint32_t oo = OUT_AUTO) {
    uint32_t* tup = COL(uint32_t, U_TUPLE);
    const uint32_t calls = 100u * db.dims[2];
    float v = __uint_as_float(ldm(&tup[p[0]]));
    switch (t) {
#define MICRO_CASE(k) case k: v = micro_body<k>(v, calls); break;
        MICRO_CASE(0) MICRO_CASE(1) MICRO_CASE(2) MICRO_CASE(3) MICRO_CASE(4) MICRO_CASE(5) MICRO_CASE(6)
        MICRO_CASE(7) MICRO_CASE(8) MICRO_CASE(9) MICRO_CASE(10) MICRO_CASE(11) MICRO_CASE(12) MICRO_CASE(13)
        MICRO_CASE(14) MICRO_CASE(15) MICRO_CASE(16) MICRO_CASE(17) MICRO_CASE(18) MICRO_CASE(19)
        MICRO_CASE(20) MICRO_CASE(21) MICRO_CASE(22) MICRO_CASE(23) MICRO_CASE(24) MICRO_CASE(25)
        MICRO_CASE(26) MICRO_CASE(27) MICRO_CASE(28) MICRO_CASE(29) MICRO_CASE(30) MICRO_CASE(31)
#undef MICRO_CASE
    default: break;
    }
    const uint32_t bits = __float_as_uint(v);
    stm(&tup[p[0]], bits);
    put32(out_rec<4>(db, idx, oo), bits);
}

// ---- TPC-C -------------------------------------------------------------------------
// NewOrder home part: district counter, ORDER / NEW_ORDER / ORDER_LINE rows, o_id,
// total, per-line amount + brand; stock lines whose supply warehouse == sw_sel
// (all lines when sw_sel == ALL).
constexpr uint32_t ALL_LINES = 0xFFFFFFFFu;

DEV bool tpcc_no_aborts(const DevDb& db, const uint32_t* p) {
    const uint32_t cnt = p[3];
    for (uint32_t l = 0; l < cnt; ++l)
        if (p[4 + 3 * l] >= db.dims[3]) return true;       // unused item: roll back (static)
    return false;
}

// Stock lines: read every selected line's S_QUANTITY first, then apply the lines in
// order (a repeated (sw, i) sees its earlier line's update), then write.
DEV void tpcc_no_stock(const DevDb& db, uint32_t idx, const uint32_t* p, uint32_t sw_sel) {
    const uint32_t I = db.dims[3], w = p[0], cnt = p[3];
    int32_t* sq = COL(int32_t, C_S_QTY);
    uint64_t sidx[15];
    int32_t q0[15];
#pragma unroll
    for (int l = 0; l < 15; ++l) {
        if ((uint32_t)l < cnt) {
            sidx[l] = (uint64_t)p[5 + 3 * l] * I + p[4 + 3 * l];
            q0[l] = ldm(&sq[sidx[l]]);
        }
    }
    uint8_t* o = out_rec<200>(db, idx);
    int32_t cur[15];
#pragma unroll
    for (int l = 0; l < 15; ++l) {
        if ((uint32_t)l >= cnt) continue;
        const uint32_t sw = p[5 + 3 * l];
        if (sw_sel != ALL_LINES && sw != sw_sel) continue;
        const int32_t q = (int32_t)p[6 + 3 * l];
        int32_t before = q0[l];
#pragma unroll
        for (int m = 0; m < l; ++m)
            if (sidx[m] == sidx[l]) before = cur[m];       // latest earlier update of the same stock row
        cur[l] = before >= q + 10 ? before - q : before - q + 91;
        put32(o + 16 + 12 * l, (uint32_t)before);
        red_add(&COL(int64_t, C_S_YTD)[sidx[l]], (int64_t)q);
        red_add(&COL(uint32_t, C_S_OCNT)[sidx[l]], 1u);
        if (sw != w) red_add(&COL(uint32_t, C_S_RCNT)[sidx[l]], 1u);
    }
#pragma unroll
    for (int l = 0; l < 15; ++l) {
        if ((uint32_t)l >= cnt) continue;
        const uint32_t sw = p[5 + 3 * l];
        if (sw_sel != ALL_LINES && sw != sw_sel) continue;
        stm(&sq[sidx[l]], cur[l]);
    }
}

DEV void tpcc_no_home(const DevDb& db, uint32_t idx, const uint32_t* p, bool sh) {
    const uint32_t D = db.dims[1], C = db.dims[2], I = db.dims[3], w = p[0], d = p[1], c = p[2], cnt = p[3];
    const uint64_t wd = (uint64_t)w * D + d;
    uint32_t* dn = COL(uint32_t, C_D_NEXT);
    const int32_t* price = COL(const int32_t, C_I_PRICE);
    const uint8_t* iorig = COL(const uint8_t, C_I_ORIG);
    const uint8_t* sorig = COL(const uint8_t, C_S_ORIG);
    const uint32_t oid = ldm(&dn[wd]);
    const int64_t disc = __ldg(&COL(const int32_t, C_C_DISC)[wd * C + c]);
    const int64_t tax = (int64_t)__ldg(&COL(const int32_t, C_W_TAX)[w]) + __ldg(&COL(const int32_t, C_D_TAX)[wd]);
    int32_t pr[15];
    uint8_t br[15];
#pragma unroll
    for (int l = 0; l < 15; ++l) {
        if ((uint32_t)l < cnt) {
            const uint32_t i = p[4 + 3 * l], sw = p[5 + 3 * l];
            pr[l] = __ldg(&price[i]);
            br[l] = __ldg(&iorig[i]) & __ldg(&sorig[(uint64_t)sw * I + i]);
        }
    }
    stm(&dn[wd], oid + 1);
    uint32_t all_local = 1;
    for (uint32_t l = 0; l < cnt; ++l) all_local &= (p[5 + 3 * l] == w);
    const uint64_t ro = db.ins_base[T_ORDER] + db.ins_off[T_ORDER * (uint64_t)db.ins_stride + idx];
    INS(uint32_t, IO_ID)[ro] = oid; INS(uint32_t, IO_D)[ro] = d; INS(uint32_t, IO_W)[ro] = w;
    INS(uint32_t, IO_C)[ro] = c; INS(uint32_t, IO_ENTRY)[ro] = txn_ts(db, idx, sh);
    INS(uint32_t, IO_OLCNT)[ro] = cnt; INS(uint32_t, IO_ALLLOCAL)[ro] = all_local;
    const uint64_t rn = db.ins_base[T_NEWORDER] + db.ins_off[T_NEWORDER * (uint64_t)db.ins_stride + idx];
    INS(uint32_t, IN_OID)[rn] = oid; INS(uint32_t, IN_D)[rn] = d; INS(uint32_t, IN_W)[rn] = w;
    const uint64_t rl0 = db.ins_base[T_OLINE] + db.ins_off[T_OLINE * (uint64_t)db.ins_stride + idx];
    uint8_t* o = out_rec<200>(db, idx);
    int64_t sum = 0;
#pragma unroll
    for (int l = 0; l < 15; ++l) {
        if ((uint32_t)l >= cnt) continue;
        const uint32_t i = p[4 + 3 * l], sw = p[5 + 3 * l], q = p[6 + 3 * l];
        const int32_t amount = (int32_t)q * pr[l];
        sum += amount;
        const uint64_t rl = rl0 + l;
        INS(uint32_t, IL_OID)[rl] = oid; INS(uint32_t, IL_D)[rl] = d; INS(uint32_t, IL_W)[rl] = w;
        INS(uint32_t, IL_NUM)[rl] = l; INS(uint32_t, IL_I)[rl] = i; INS(uint32_t, IL_SW)[rl] = sw;
        INS(uint32_t, IL_QTY)[rl] = q; INS(int32_t, IL_AMT)[rl] = amount;
        put32(o + 16 + 12 * l + 4, (uint32_t)amount);
        o[16 + 12 * l + 8] = br[l];
    }
    const int64_t x = sum * (10000 - disc) * (10000 + tax);
    put32(o, oid);
    put32(o + 4, cnt);
    put64(o + 8, (uint64_t)((x + 50000000) / 100000000));
}

DEV void tpcc_pay_home(const DevDb& db, uint32_t idx, const uint32_t* p, bool sh) {
    const uint32_t D = db.dims[1], w = p[0], d = p[1], h = p[6];
    red_add(&COL(int64_t, C_W_YTD)[w], (int64_t)h);
    red_add(&COL(int64_t, C_D_YTD)[(uint64_t)w * D + d], (int64_t)h);
    const uint64_t r = db.ins_base[T_HIST] + db.ins_off[T_HIST * (uint64_t)db.ins_stride + idx];
    INS(uint32_t, IH_C)[r] = p[5]; INS(uint32_t, IH_CD)[r] = p[3]; INS(uint32_t, IH_CW)[r] = p[2];
    INS(uint32_t, IH_D)[r] = d; INS(uint32_t, IH_W)[r] = w; INS(uint32_t, IH_DATE)[r] = txn_ts(db, idx, sh);
    INS(int32_t, IH_AMT)[r] = (int32_t)h;
}
DEV void tpcc_pay_customer(const DevDb& db, uint32_t idx, const uint32_t* p) {
    const uint32_t D = db.dims[1], C = db.dims[2], h = p[6];
    const uint64_t cx = ((uint64_t)p[2] * D + p[3]) * C + p[5];
    int64_t* bal = COL(int64_t, C_C_BAL);
    const int64_t nb = ldm(&bal[cx]) - (int64_t)h;
    const uint8_t credit = __ldg(&COL(const uint8_t, C_C_CREDIT)[cx]);
    stm(&bal[cx], nb);
    red_add(&COL(int64_t, C_C_YTD)[cx], (int64_t)h);
    red_add(&COL(uint32_t, C_C_CNT)[cx], 1u);
    uint8_t* o = out_rec<200>(db, idx);
    put32(o, p[5]);
    put32(o + 4, credit);
    put64(o + 8, (uint64_t)nb);
}

// Whole TPC-C transaction (K-SET, TPL) written for warp convergence: one load phase
// with no early exit or data-dependent loop (the 15 line slots are predicated), so
// the lanes of a warp issue all their loads together; the abort decision and the
// writes come after.  (Lanes that diverged in the line loops with their loads
// outstanding ran one after another: 8 NewOrders in one warp took 10x one.)
DEV void tpcc_txn(const DevDb& db, uint32_t idx, uint32_t t, const uint32_t* p, bool sh) {
    const uint32_t D = db.dims[1], C = db.dims[2], I = db.dims[3];
    const bool no = t == 0;
    const uint32_t w = p[0], d = p[1];
    const uint32_t cnt = no ? min(p[3], 15u) : 0u;
    uint32_t li[15], lsw[15], lq[15];
    bool abort = !no && p[4] == 2;
#pragma unroll
    for (int l = 0; l < 15; ++l) {
        li[l] = 0; lsw[l] = 0; lq[l] = 0;
        if ((uint32_t)l < cnt) { li[l] = p[4 + 3 * l]; lsw[l] = p[5 + 3 * l]; lq[l] = p[6 + 3 * l]; }
    }
#pragma unroll
    for (int l = 0; l < 15; ++l) abort |= ((uint32_t)l < cnt) && li[l] >= I;   // unused item: roll back
    const bool go = !abort;
    const uint64_t wd = (uint64_t)w * D + d;
    // ---- load phase
    uint32_t oid = 0;
    int64_t disc = 0, tax = 0, cbal = 0;
    uint8_t credit = 0;
    uint64_t ro = 0, rn = 0, rl0 = 0, rh = 0, cx = 0;
    uint64_t sidx[15];
    int32_t pr[15], q0[15];
    uint8_t br[15];
    if (no && go) {
        oid = ldm(&COL(uint32_t, C_D_NEXT)[wd]);
        disc = __ldg(&COL(const int32_t, C_C_DISC)[wd * C + p[2]]);
        tax = (int64_t)__ldg(&COL(const int32_t, C_W_TAX)[w]) + __ldg(&COL(const int32_t, C_D_TAX)[wd]);
        ro = db.ins_base[T_ORDER] + db.ins_off[T_ORDER * (uint64_t)db.ins_stride + idx];
        rn = db.ins_base[T_NEWORDER] + db.ins_off[T_NEWORDER * (uint64_t)db.ins_stride + idx];
        rl0 = db.ins_base[T_OLINE] + db.ins_off[T_OLINE * (uint64_t)db.ins_stride + idx];
    }
#pragma unroll
    for (int l = 0; l < 15; ++l) {
        sidx[l] = (uint64_t)lsw[l] * I + li[l];
        pr[l] = 0; q0[l] = 0; br[l] = 0;
        if (no && go && (uint32_t)l < cnt) {
            pr[l] = __ldg(&COL(const int32_t, C_I_PRICE)[li[l]]);
            br[l] = __ldg(&COL(const uint8_t, C_I_ORIG)[li[l]]) & __ldg(&COL(const uint8_t, C_S_ORIG)[sidx[l]]);
            q0[l] = ldm(&COL(int32_t, C_S_QTY)[sidx[l]]);
        }
    }
    if (!no && go) {
        cx = ((uint64_t)p[2] * D + p[3]) * C + p[5];
        cbal = ldm(&COL(int64_t, C_C_BAL)[cx]);
        credit = __ldg(&COL(const uint8_t, C_C_CREDIT)[cx]);
        rh = db.ins_base[T_HIST] + db.ins_off[T_HIST * (uint64_t)db.ins_stride + idx];
    }
    // ---- decide, then write
    if (abort) { db.status[idx] = 1; return; }
    uint8_t* o = out_rec<200>(db, idx);
    if (no) {
        stm(&COL(uint32_t, C_D_NEXT)[wd], oid + 1);
        uint32_t all_local = 1;
#pragma unroll
        for (int l = 0; l < 15; ++l) all_local &= ((uint32_t)l >= cnt) || lsw[l] == w;
        INS(uint32_t, IO_ID)[ro] = oid; INS(uint32_t, IO_D)[ro] = d; INS(uint32_t, IO_W)[ro] = w;
        INS(uint32_t, IO_C)[ro] = p[2]; INS(uint32_t, IO_ENTRY)[ro] = txn_ts(db, idx, sh);
        INS(uint32_t, IO_OLCNT)[ro] = cnt; INS(uint32_t, IO_ALLLOCAL)[ro] = all_local;
        INS(uint32_t, IN_OID)[rn] = oid; INS(uint32_t, IN_D)[rn] = d; INS(uint32_t, IN_W)[rn] = w;
        int64_t sum = 0;
        int32_t cur[15];
#pragma unroll
        for (int l = 0; l < 15; ++l) {
            if ((uint32_t)l >= cnt) continue;
            const int32_t q = (int32_t)lq[l];
            const int32_t amount = q * pr[l];
            sum += amount;
            int32_t before = q0[l];
#pragma unroll
            for (int m = 0; m < l; ++m)
                if (sidx[m] == sidx[l]) before = cur[m];      // latest earlier update of the same stock row
            cur[l] = before >= q + 10 ? before - q : before - q + 91;
            const uint64_t rl = rl0 + l;
            INS(uint32_t, IL_OID)[rl] = oid; INS(uint32_t, IL_D)[rl] = d; INS(uint32_t, IL_W)[rl] = w;
            INS(uint32_t, IL_NUM)[rl] = l; INS(uint32_t, IL_I)[rl] = li[l]; INS(uint32_t, IL_SW)[rl] = lsw[l];
            INS(uint32_t, IL_QTY)[rl] = lq[l]; INS(int32_t, IL_AMT)[rl] = amount;
            put32(o + 16 + 12 * l, (uint32_t)before);
            put32(o + 16 + 12 * l + 4, (uint32_t)amount);
            o[16 + 12 * l + 8] = br[l];
            red_add(&COL(int64_t, C_S_YTD)[sidx[l]], (int64_t)q);
            red_add(&COL(uint32_t, C_S_OCNT)[sidx[l]], 1u);
            if (lsw[l] != w) red_add(&COL(uint32_t, C_S_RCNT)[sidx[l]], 1u);
        }
#pragma unroll
        for (int l = 0; l < 15; ++l)
            if ((uint32_t)l < cnt) stm(&COL(int32_t, C_S_QTY)[sidx[l]], cur[l]);
        const int64_t x = sum * (10000 - disc) * (10000 + tax);
        put32(o, oid);
        put32(o + 4, cnt);
        put64(o + 8, (uint64_t)((x + 50000000) / 100000000));
    } else {
        const uint32_t h = p[6];
        red_add(&COL(int64_t, C_W_YTD)[w], (int64_t)h);
        red_add(&COL(int64_t, C_D_YTD)[wd], (int64_t)h);
        INS(uint32_t, IH_C)[rh] = p[5]; INS(uint32_t, IH_CD)[rh] = p[3]; INS(uint32_t, IH_CW)[rh] = p[2];
        INS(uint32_t, IH_D)[rh] = d; INS(uint32_t, IH_W)[rh] = w; INS(uint32_t, IH_DATE)[rh] = txn_ts(db, idx, sh);
        INS(int32_t, IH_AMT)[rh] = (int32_t)h;
        const int64_t nb = cbal - (int64_t)h;
        stm(&COL(int64_t, C_C_BAL)[cx], nb);
        red_add(&COL(int64_t, C_C_YTD)[cx], (int64_t)h);
        red_add(&COL(uint32_t, C_C_CNT)[cx], 1u);
        put32(o, p[5]);
        put32(o + 4, credit);
        put64(o + 8, (uint64_t)nb);
    }
}

// The same TPC-C transaction executed by a whole warp (K-SET, TPL): NewOrder line l is
// lane l's.  One thread issuing a NewOrder's ~270 scattered loads and stores serially
// was the per-round critical path (~5 us); spread over the lanes it is ~20 per lane.
// Same results as tpcc_txn: a repeated stock row sees its earlier line's update (the
// updates are chained through the lanes in line order) and only its last line stores it.
// TPC-C Payment on the calling thread; with_wytd = false leaves out its W_YTD update
// (the caller applies it under the warehouse's lock: tpl_exec_warp_kernel).  Returns
// false if it aborted (by-name lookup found nobody: no writes at all).
DEV bool tpcc_payment(const DevDb& db, uint32_t idx, const uint32_t* p, bool sh, bool with_wytd) {
    const uint32_t D = db.dims[1], C = db.dims[2];
    const uint32_t w = p[0], d = p[1];
    const uint64_t wd = (uint64_t)w * D + d;
    uint8_t* o = out_rec<200>(db, idx);
    if (p[4] == 2) { db.status[idx] = 1; return false; }
    const uint64_t cx = ((uint64_t)p[2] * D + p[3]) * C + p[5];
    const int64_t cbal = ldm(&COL(int64_t, C_C_BAL)[cx]);
    const uint8_t credit = __ldg(&COL(const uint8_t, C_C_CREDIT)[cx]);
    const uint64_t rh = db.ins_base[T_HIST] + db.ins_off[T_HIST * (uint64_t)db.ins_stride + idx];
    const uint32_t h = p[6];
    if (with_wytd) red_add(&COL(int64_t, C_W_YTD)[w], (int64_t)h);
    red_add(&COL(int64_t, C_D_YTD)[wd], (int64_t)h);
    INS(uint32_t, IH_C)[rh] = p[5]; INS(uint32_t, IH_CD)[rh] = p[3]; INS(uint32_t, IH_CW)[rh] = p[2];
    INS(uint32_t, IH_D)[rh] = d; INS(uint32_t, IH_W)[rh] = w; INS(uint32_t, IH_DATE)[rh] = txn_ts(db, idx, sh);
    INS(int32_t, IH_AMT)[rh] = (int32_t)h;
    const int64_t nb = cbal - (int64_t)h;
    stm(&COL(int64_t, C_C_BAL)[cx], nb);
    red_add(&COL(int64_t, C_C_YTD)[cx], (int64_t)h);
    red_add(&COL(uint32_t, C_C_CNT)[cx], 1u);
    put32(o, p[5]);
    put32(o + 4, credit);
    put64(o + 8, (uint64_t)nb);
    return true;
}

DEV void tpcc_txn_warp(const DevDb& db, uint32_t idx, uint32_t t, const uint32_t* p, bool sh) {
    constexpr uint32_t FULL = 0xffffffffu;
    const uint32_t lane = lane_id();
    const uint32_t D = db.dims[1], C = db.dims[2], I = db.dims[3];
    const uint32_t w = p[0], d = p[1];
    const uint64_t wd = (uint64_t)w * D + d;
    uint8_t* o = out_rec<200>(db, idx);
    if (t != 0) {                                 // Payment: small, lane 0
        if (lane == 0) tpcc_payment(db, idx, p, sh, true);
        return;
    }
    const uint32_t cnt = min(p[3], 15u);
    const bool has = lane < cnt;
    uint32_t li = 0, lsw = 0, lq = 0;
    if (has) { li = p[4 + 3 * lane]; lsw = p[5 + 3 * lane]; lq = p[6 + 3 * lane]; }
    if (__any_sync(FULL, has && li >= I)) {       // unused item: roll back (static)
        if (lane == 0) db.status[idx] = 1;
        return;
    }
    // ---- load phase
    uint32_t oid = 0;
    int64_t disc = 0, tax = 0;
    uint64_t ro = 0, rn = 0, rl0 = 0;
    if (lane == 0) {
        oid = ldm(&COL(uint32_t, C_D_NEXT)[wd]);
        disc = __ldg(&COL(const int32_t, C_C_DISC)[wd * C + p[2]]);
        tax = (int64_t)__ldg(&COL(const int32_t, C_W_TAX)[w]) + __ldg(&COL(const int32_t, C_D_TAX)[wd]);
        ro = db.ins_base[T_ORDER] + db.ins_off[T_ORDER * (uint64_t)db.ins_stride + idx];
        rn = db.ins_base[T_NEWORDER] + db.ins_off[T_NEWORDER * (uint64_t)db.ins_stride + idx];
    }
    if (lane == 1 || cnt == 0) rl0 = db.ins_base[T_OLINE] + db.ins_off[T_OLINE * (uint64_t)db.ins_stride + idx];
    const uint64_t sidx = has ? (uint64_t)lsw * I + li : ~0ull - lane;     // unique for idle lanes
    int32_t pr = 0, q0 = 0;
    uint8_t br = 0;
    if (has) {
        pr = __ldg(&COL(const int32_t, C_I_PRICE)[li]);
        br = __ldg(&COL(const uint8_t, C_I_ORIG)[li]) & __ldg(&COL(const uint8_t, C_S_ORIG)[sidx]);
        q0 = ldm(&COL(int32_t, C_S_QTY)[sidx]);
    }
    oid = __shfl_sync(FULL, oid, 0);
    rl0 = __shfl_sync(FULL, rl0, cnt == 0 ? 0 : 1);
    // ---- stock recurrence in line order (duplicates chained through the lanes)
    int32_t before = q0, cur = 0;
    for (uint32_t m = 0; m < cnt; ++m) {
        const int32_t bm = __shfl_sync(FULL, before, m);
        const int32_t qm = (int32_t)__shfl_sync(FULL, lq, m);
        const uint64_t sm = __shfl_sync(FULL, sidx, m);
        const int32_t cm = bm >= qm + 10 ? bm - qm : bm - qm + 91;
        if (lane == m) cur = cm;
        if (lane > m && sidx == sm) before = cm;      // a later line of the same row sees it
    }
    const uint32_t peers = __match_any_sync(FULL, sidx);
    const bool last_of_row = has && (31 - __clz(peers)) == (int)lane;
    // ---- writes
    const int32_t amount = has ? (int32_t)lq * pr : 0;
    int64_t sum = amount;
#pragma unroll
    for (int sh2 = 16; sh2; sh2 >>= 1) sum += __shfl_xor_sync(FULL, sum, sh2);
    const bool all_local = __all_sync(FULL, !has || lsw == w);
    if (has) {
        const uint64_t rl = rl0 + lane;
        INS(uint32_t, IL_OID)[rl] = oid; INS(uint32_t, IL_D)[rl] = d; INS(uint32_t, IL_W)[rl] = w;
        INS(uint32_t, IL_NUM)[rl] = lane; INS(uint32_t, IL_I)[rl] = li; INS(uint32_t, IL_SW)[rl] = lsw;
        INS(uint32_t, IL_QTY)[rl] = lq; INS(int32_t, IL_AMT)[rl] = amount;
        put32(o + 16 + 12 * lane, (uint32_t)before);
        put32(o + 16 + 12 * lane + 4, (uint32_t)amount);
        o[16 + 12 * lane + 8] = br;
        red_add(&COL(int64_t, C_S_YTD)[sidx], (int64_t)lq);
        red_add(&COL(uint32_t, C_S_OCNT)[sidx], 1u);
        if (lsw != w) red_add(&COL(uint32_t, C_S_RCNT)[sidx], 1u);
        if (last_of_row) stm(&COL(int32_t, C_S_QTY)[sidx], cur);
    }
    if (lane == 0) {
        stm(&COL(uint32_t, C_D_NEXT)[wd], oid + 1);
        INS(uint32_t, IO_ID)[ro] = oid; INS(uint32_t, IO_D)[ro] = d; INS(uint32_t, IO_W)[ro] = w;
        INS(uint32_t, IO_C)[ro] = p[2]; INS(uint32_t, IO_ENTRY)[ro] = txn_ts(db, idx, sh);
        INS(uint32_t, IO_OLCNT)[ro] = cnt; INS(uint32_t, IO_ALLLOCAL)[ro] = all_local ? 1u : 0u;
        INS(uint32_t, IN_OID)[rn] = oid; INS(uint32_t, IN_D)[rn] = d; INS(uint32_t, IN_W)[rn] = w;
        const int64_t x = sum * (10000 - disc) * (10000 + tax);
        put32(o, oid);
        put32(o + 4, cnt);
        put64(o + 8, (uint64_t)((x + 50000000) / 100000000));
    }
}

template <int S> __device__ __noinline__ void exec_local(const DevDb& db, uint32_t idx);

// one TPC-C transaction by the calling (whole) warp
template <bool SH>
DEV void exec_txn_warp(const DevDb& db, uint32_t idx) {
    if (SH && db.xflag && db.xflag[idx]) {        // cross-shard: its local fragments, lane 0
        if (lane_id() == 0) exec_local<S_TPCC>(db, idx);
        return;
    }
    tpcc_txn_warp(db, idx, db.type[idx], db.pw + db.poff[idx], SH);
}

// The combined kernel body: one whole transaction (K-SET, TPL).  Sharded: a transaction
// with a fragment on another shard runs only its local fragments.
// Warm L2 with the rows a transaction of a coming k-set round will touch (from its
// staged parameters).  prefetch.global.L2 returns no data, so it is safe while the
// current round may still write those rows: the round's own loads come after the
// round barrier and then hit L2 instead of HBM.
DEV void l2_warm(const void* a) { asm volatile("prefetch.global.L2 [%0];" ::"l"(a)); }
// TPC-B only: its round-to-round critical path is one HBM miss on the account row (1e8
// accounts); TM-1's rows are hot in L2 already and the extra instructions cost more
// (K-SET exec 0.73 -> 0.79 ms measured), TPC-C stages no parameters.
template <int S>
DEV void warm_rows(const DevDb& db, uint32_t t, const uint32_t* p) {
    if (S == S_TPCB) l2_warm(&COL(const int64_t, B_ACC)[p[0]]);
}

template <int S, bool SH = false>
DEV void exec_txn_p(const DevDb& db, uint32_t idx, uint32_t t, const uint32_t* p, uint32_t oo = OUT_AUTO) {
    if (SH && db.xflag && db.xflag[idx]) { exec_local<S>(db, idx); return; }
    if (S == S_TPCB) {
        if (t == 1) { tpcb_withdraw(db, idx, p, oo); return; }
        tpcb_home(db, idx, p, SH);
        tpcb_account(db, idx, p, oo);
    } else if (S == S_TM1) {
        tm1_txn(db, idx, t, p, oo);
    } else if (S == S_MICRO) {
        micro_txn(db, idx, t, p, oo);
    } else {
        tpcc_txn(db, idx, t, p, SH);
    }
}

template <int S, bool SH = false>
DEV void exec_txn(const DevDb& db, uint32_t idx) {
    exec_txn_p<S, SH>(db, idx, db.type[idx], db.pw + db.poff[idx]);
}

// =================================================================================
// PART fragments (DESIGN.md R-S9): a cross-partition transaction whose parts share
// no data flow runs as one fragment per partition; each partition executes its
// fragments in ts order.  frag key = pid << 32 | idx << 8 | kind
// =================================================================================
enum { F_WHOLE = 0, F_HOME = 1, F_REMOTE = 2 };

DEV uint64_t frag_key(uint32_t pid, uint32_t idx, uint32_t kind) {
    return ((uint64_t)pid << 32) | ((uint64_t)idx << 8) | kind;
}

// number of fragments of txn idx and, if out != nullptr, the keys
template <int S>
DEV int fragments(const DevDb& db, uint32_t idx, uint64_t* out) {
    const uint32_t t = db.type[idx];
    const uint32_t* p = db.pw + db.poff[idx];
    if (S == S_TPCB) {
        const uint32_t home = p[2], own = p[0] / db.dims[2];
        if (home == own || t == 1) { if (out) out[0] = frag_key(home, idx, F_WHOLE); return 1; }
        if (out) { out[0] = frag_key(home, idx, F_HOME); out[1] = frag_key(own, idx, F_REMOTE); }
        return 2;
    } else if (S == S_TM1) {
        const uint32_t pid = p[0] ? (p[0] - 1) / db.part_size : 0;
        if (out) out[0] = frag_key(pid, idx, F_WHOLE);
        return 1;
    } else if (S == S_MICRO) {                         // partition = part_size consecutive tuples
        if (out) out[0] = frag_key(p[0] / db.part_size, idx, F_WHOLE);
        return 1;
    } else {
        const uint32_t w = p[0];
        if (t == 0) {
            // an aborting NewOrder, or one whose lines are all home-warehouse, is whole
            // (the PART executors run whole NewOrders with the warp procedure)
            if (tpcc_no_aborts(db, p)) { if (out) out[0] = frag_key(w, idx, F_WHOLE); return 1; }
            bool local = true;
            for (uint32_t l = 0; l < p[3]; ++l) local &= p[5 + 3 * l] == w;
            if (local) { if (out) out[0] = frag_key(w, idx, F_WHOLE); return 1; }
            int k = 0;
            if (out) out[k] = frag_key(w, idx, F_HOME);
            ++k;
            const uint32_t cnt = p[3];
            for (uint32_t l = 0; l < cnt; ++l) {
                const uint32_t sw = p[5 + 3 * l];
                if (sw == w) continue;
                bool seen = false;
                for (uint32_t m = 0; m < l; ++m) seen |= (p[5 + 3 * m] == sw);
                if (seen) continue;
                if (out) out[k] = frag_key(sw, idx, F_REMOTE);
                ++k;
            }
            return k;
        }
        if (p[4] == 2 || p[2] == w) { if (out) out[0] = frag_key(w, idx, F_WHOLE); return 1; }
        if (out) { out[0] = frag_key(w, idx, F_HOME); out[1] = frag_key(p[2], idx, F_REMOTE); }
        return 2;
    }
}

template <int S>
DEV void exec_frag(const DevDb& db, uint64_t fk) {
    const uint32_t pid = (uint32_t)(fk >> 32), idx = (uint32_t)(fk >> 8) & 0xFFFFFFu, kind = (uint32_t)fk & 0xFFu;
    const uint32_t t = db.type[idx];
    const bool sh = db.ts != nullptr;
    const uint32_t* p = db.pw + db.poff[idx];
    if (S == S_TPCB) {
        if (t == 1) { tpcb_withdraw(db, idx, p); return; }
        if (kind != F_REMOTE) tpcb_home(db, idx, p, sh);
        if (kind != F_HOME) tpcb_account(db, idx, p);
    } else if (S == S_TM1) {
        tm1_txn(db, idx, t, p);
    } else if (S == S_MICRO) {
        micro_txn(db, idx, t, p);
    } else {
        if (t == 0) {
            if (tpcc_no_aborts(db, p)) { db.status[idx] = 1; return; }
            if (kind != F_REMOTE) tpcc_no_home(db, idx, p, sh);
            tpcc_no_stock(db, idx, p, pid);
        } else {
            if (p[4] == 2) { if (kind != F_REMOTE) db.status[idx] = 1; return; }
            if (kind != F_REMOTE) tpcc_pay_home(db, idx, p, sh);
            if (kind != F_HOME) tpcc_pay_customer(db, idx, p);
        }
    }
}

// a fragment lives on this shard (TM-1 transactions are single-root: home = local)
template <int S>
DEV bool frag_local(const DevDb& db, uint64_t fk) {
    return S == S_TM1 || S == S_MICRO || db.nshards <= 1 || root_local(db, fk >> 32);
}

// the fragments of txn idx on this shard (all of them when unsharded)
template <int S>
DEV int fragments_local(const DevDb& db, uint32_t idx, uint64_t* out) {
    uint64_t fk[MAX_REC];
    const int k = fragments<S>(db, idx, fk);
    int m = 0;
    for (int j = 0; j < k; ++j)
        if (frag_local<S>(db, fk[j])) { if (out) out[m] = fk[j]; ++m; }
    return m;
}

// (out of line: the cold sharded path must not cost the fused kernels registers)
template <int S>
__device__ __noinline__ void exec_local(const DevDb& db, uint32_t idx) {
    uint64_t fk[MAX_REC];
    const int k = fragments<S>(db, idx, fk);
    for (int j = 0; j < k; ++j)
        if (frag_local<S>(db, fk[j])) exec_frag<S>(db, fk[j]);
}

}  // namespace gputx
