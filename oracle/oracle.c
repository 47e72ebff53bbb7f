/*
 * oracle.c — TEST INFRASTRUCTURE ONLY.  Plain, slow, single-threaded CPU oracle
 * for GPUTx bulk execution (He & Yu, PVLDB 4(5) 2011, arXiv 1103.3105).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  It shares no code, header, table or
 * constant generator with the CUDA path (paper_1103_3105_b200/); the only
 * common input is the seeded data from workloads/.
 *
 * What it computes
 * ----------------
 *  orc_run():     Definition 1 (§3.1) written out: starting from
 *                 the given database image, execute the bulk's transactions
 *                 ONE AT A TIME in increasing timestamp order (ts = first_ts+i,
 *                 PAPER.md:95), each by its stored procedure (
 *                 the procedures are the public benchmark definitions the
 *                 paper names, as read in DESIGN.md §3).
 *                 Inserts are appended immediately (true serial semantics).
 *                 Produces the final image, per-transaction status and output
 *                 record, and the inserted rows.
 *  orc_footprint(): the conflict footprint (basic operations)
 *                 of each transaction: (item, mode) with same-item accesses
 *                 merged (W dominates) and read-only columns omitted
 *                 ("Fekete ... static analysis"; DESIGN.md R-S3, R-S18).
 *  orc_depths():  T-dependency-graph depth of every transaction (PAPER.md:113-115,
 *                 §4.1) by the streaming recurrence over items:
 *                   d(t) = max over t's ops of (W ? Md[x]+1 : Wd[x]+1), 0 if none,
 *                 where Wd = depth of x's last writer, Md = max depth of the
 *                 accesses to x since (and including) that writer.  This is the
 *                 longest path from a source because a writer conflicts with every
 *                 earlier access to x and writers of x form a chain.
 *
 * Pins (tests/test_oracle_*.py): TPC-B closed forms and sum invariants, TPC-C
 * consistency invariants, TM-1 liveness counts, per-item projection replay,
 * every-linear-extension brute force on tiny bulks, the Figure-1 worked depths,
 * O(n^2) brute-force depths and the Appendix-B graph + topological sort.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------- */
/* schemas (values of the public interface; the oracle keeps its own copy)       */
/* ---------------------------------------------------------------------------- */
enum { S_TPCB = 1, S_TM1 = 2, S_TPCC = 3, S_MICRO = 4 };

#define OUT_TPCB 8
#define OUT_TM1 40
#define OUT_TPCC 200
#define OUT_MICRO 4

static void put_u32(uint8_t* p, uint32_t v) { memcpy(p, &v, 4); }
static void put_i32(uint8_t* p, int32_t v) { memcpy(p, &v, 4); }
static void put_u64(uint8_t* p, uint64_t v) { memcpy(p, &v, 8); }
static void put_i64(uint8_t* p, int64_t v) { memcpy(p, &v, 8); }

/* ============================================================================ */
/* TPC-B (Ext TPC-B "deposit")                                      */
/* cols: 0 br_bal i64[B], 1 tel_bal i64[B*T], 2 acc_bal i64[B*A]                  */
/* ins : history h_tid,h_bid,h_aid u32, h_delta i32, h_ts u32                     */
/* ============================================================================ */
/* WITHDRAW (type 1): a NON-two-phase procedure -- it
 * debits account, teller and branch, THEN aborts if the account went negative, which
 * requires undoing its own updates (here: restoring the values it overwrote).  No history
 * row.  Output on commit: the account balance after the debit. */
static void tpcb_withdraw(void** cols, const uint32_t* p, uint8_t* st, uint8_t* out)
{
    int64_t* br = (int64_t*)cols[0];
    int64_t* tel = (int64_t*)cols[1];
    int64_t* acc = (int64_t*)cols[2];
    uint32_t aid = p[0], tid = p[1], bid = p[2];
    int64_t amt = (int64_t)(int32_t)p[3];
    int64_t a0 = acc[aid], t0 = tel[tid], b0 = br[bid];   /* undo log */
    acc[aid] -= amt;
    tel[tid] -= amt;
    br[bid] -= amt;
    if (acc[aid] < 0) {                                  /* abort after the writes: roll back */
        acc[aid] = a0; tel[tid] = t0; br[bid] = b0;
        *st = 1;
        return;
    }
    put_i64(out, acc[aid]);
    *st = 0;
}

static void tpcb_txn(void** cols, const uint32_t* p, uint64_t ts, uint8_t* st, uint8_t* out,
                     void** ins, uint64_t* nrows)
{
    int64_t* br = (int64_t*)cols[0];
    int64_t* tel = (int64_t*)cols[1];
    int64_t* acc = (int64_t*)cols[2];
    uint32_t aid = p[0], tid = p[1], bid = p[2];
    int32_t delta = (int32_t)p[3];
    acc[aid] += delta;                       /* UPDATE accounts SET Abalance += delta */
    put_i64(out, acc[aid]);                  /* SELECT Abalance                     */
    tel[tid] += delta;                       /* UPDATE tellers                      */
    br[bid] += delta;                        /* UPDATE branches                     */
    uint64_t r = nrows[0]++;                 /* INSERT INTO history                 */
    ((uint32_t*)ins[0])[r] = tid;
    ((uint32_t*)ins[1])[r] = bid;
    ((uint32_t*)ins[2])[r] = aid;
    ((int32_t*)ins[3])[r] = delta;
    ((uint32_t*)ins[4])[r] = (uint32_t)ts;
    *st = 0;
}

/* ============================================================================ */
/* TM-1 / TATP (Ext TATP), s = s_id - 1                          */
/* cols: 0 sub_nbr u64[P] 1 sub_bits u16[P] 2 sub_hex u64[P] 3 sub_byte2 u8[P*10]   */
/*       4 sub_msc u32[P] 5 sub_vlr u32[P]                                           */
/*       6 ai_valid u8[4P] 7 ai_data1 u8 8 ai_data2 u8 9 ai_data3 u32 10 ai_data4 u64 */
/*       11 sf_valid u8[4P] 12 sf_active u8 13 sf_error u8 14 sf_data_a u8 15 sf_data_b u64 */
/*       16 cf_live u8[12P] 17 cf_end u8 18 cf_numberx u64                          */
/* ============================================================================ */
typedef struct {
    uint64_t* nbr; uint16_t* bits; uint64_t* hex; uint8_t* byte2; uint32_t* msc; uint32_t* vlr;
    uint8_t* ai_valid; uint8_t* ai_d1; uint8_t* ai_d2; uint32_t* ai_d3; uint64_t* ai_d4;
    uint8_t* sf_valid; uint8_t* sf_active; uint8_t* sf_err; uint8_t* sf_da; uint64_t* sf_db;
    uint8_t* cf_live; uint8_t* cf_end; uint64_t* cf_num;
    uint32_t P;
} tm1_t;

static tm1_t tm1_bind(void** c, const uint32_t* dims)
{
    tm1_t t;
    t.nbr = c[0]; t.bits = c[1]; t.hex = c[2]; t.byte2 = c[3]; t.msc = c[4]; t.vlr = c[5];
    t.ai_valid = c[6]; t.ai_d1 = c[7]; t.ai_d2 = c[8]; t.ai_d3 = c[9]; t.ai_d4 = c[10];
    t.sf_valid = c[11]; t.sf_active = c[12]; t.sf_err = c[13]; t.sf_da = c[14]; t.sf_db = c[15];
    t.cf_live = c[16]; t.cf_end = c[17]; t.cf_num = c[18];
    t.P = dims[0];
    return t;
}

/* sub_nbr is the 15-digit zero-padded decimal string of s_id (Ext TATP), one digit
 * per nibble.  The lookup transaction of the split is this parse,
 * checked against the stored column; -1 when no subscriber carries the string. */
static int64_t tm1_lookup(const tm1_t* t, uint64_t nbr)
{
    uint64_t v = 0;
    for (int k = 14; k >= 0; --k) {
        uint64_t dgt = (nbr >> (4 * k)) & 0xF;
        if (dgt > 9) return -1;
        v = v * 10 + dgt;
    }
    if (v < 1 || v > t->P) return -1;
    if (t->nbr[v - 1] != nbr) return -1;
    return (int64_t)(v - 1);
}

static void tm1_txn(tm1_t* t, int type, const uint32_t* p, uint8_t* st, uint8_t* out)
{
    *st = 0;
    switch (type) {
    case 0: { /* GET_SUBSCRIBER_DATA(s_id): SELECT * FROM subscriber */
        uint32_t s = p[0] - 1;
        put_u64(out + 0, t->nbr[s]);
        put_u64(out + 8, t->hex[s]);
        put_u32(out + 16, t->msc[s]);
        put_u32(out + 20, t->vlr[s]);
        memcpy(out + 24, &t->bits[s], 2);
        memcpy(out + 26, &t->byte2[(uint64_t)s * 10], 10);
        return;
    }
    case 1: { /* GET_NEW_DESTINATION(s_id, sf_type, start_time, end_time) */
        uint32_t s = p[0] - 1, sf = p[1], stt = p[2], et = p[3];
        uint64_t f = (uint64_t)s * 4 + (sf - 1);
        if (!t->sf_valid[f] || !t->sf_active[f]) { *st = 1; return; }
        uint32_t cnt = 0;
        for (uint32_t k = 0; k < 3; ++k) {          /* start_time = 0, 8, 16 */
            uint64_t c = f * 3 + k;
            if (t->cf_live[c] && k * 8 <= stt && et < t->cf_end[c]) {
                put_u64(out + 8 + 8 * cnt, t->cf_num[c]);
                ++cnt;
            }
        }
        if (cnt == 0) { *st = 1; memset(out, 0, OUT_TM1); return; }
        put_u32(out, cnt);
        return;
    }
    case 2: { /* GET_ACCESS_DATA(s_id, ai_type) */
        uint64_t a = (uint64_t)(p[0] - 1) * 4 + (p[1] - 1);
        if (!t->ai_valid[a]) { *st = 1; return; }
        out[0] = t->ai_d1[a];
        out[1] = t->ai_d2[a];
        put_u32(out + 4, t->ai_d3[a]);
        put_u64(out + 8, t->ai_d4[a]);
        return;
    }
    case 3: { /* UPDATE_SUBSCRIBER_DATA(s_id, sf_type, bit_1, data_a) — two-phase */
        uint32_t s = p[0] - 1;
        uint64_t f = (uint64_t)s * 4 + (p[1] - 1);
        if (!t->sf_valid[f]) { *st = 1; return; }
        t->bits[s] = (uint16_t)((t->bits[s] & ~1u) | (p[2] & 1u));
        t->sf_da[f] = (uint8_t)p[3];
        return;
    }
    case 4: { /* UPDATE_LOCATION(sub_nbr, vlr_location) */
        int64_t s = tm1_lookup(t, (uint64_t)p[0] | ((uint64_t)p[1] << 32));
        if (s < 0) { *st = 1; return; }
        t->vlr[s] = p[2];
        return;
    }
    case 5: { /* INSERT_CALL_FORWARDING(sub_nbr, sf_type, start_time, end_time, numberx) */
        int64_t s = tm1_lookup(t, (uint64_t)p[0] | ((uint64_t)p[1] << 32));
        if (s < 0) { *st = 1; return; }
        uint64_t f = (uint64_t)s * 4 + (p[2] - 1);
        uint64_t c = f * 3 + p[3] / 8;
        if (!t->sf_valid[f] || t->cf_live[c]) { *st = 1; return; }
        t->cf_live[c] = 1;
        t->cf_end[c] = (uint8_t)p[4];
        t->cf_num[c] = (uint64_t)p[5] | ((uint64_t)p[6] << 32);
        return;
    }
    case 6: { /* DELETE_CALL_FORWARDING(sub_nbr, sf_type, start_time) */
        int64_t s = tm1_lookup(t, (uint64_t)p[0] | ((uint64_t)p[1] << 32));
        if (s < 0) { *st = 1; return; }
        uint64_t c = ((uint64_t)s * 4 + (p[2] - 1)) * 3 + p[3] / 8;
        if (!t->cf_live[c]) { *st = 1; return; }
        t->cf_live[c] = 0;
        return;
    }
    }
    *st = 1;
}

/* ============================================================================ */
/* TPC-C NewOrder + Payment (Ext TPC-C 2.4.2, 2.5.2)               */
/* cols: 0 w_ytd i64[W] 1 w_tax i32[W] 2 d_ytd i64[WD] 3 d_tax i32[WD]             */
/*       4 d_next_o_id u32[WD] 5 c_balance i64[WDC] 6 c_ytd_payment i64            */
/*       7 c_payment_cnt u32 8 c_discount i32 9 c_credit u8 10 c_last u16          */
/*       11 c_first u64 12 i_price i32[I] 13 i_original u8[I]                      */
/*       14 s_quantity i32[WI] 15 s_ytd i64 16 s_order_cnt u32 17 s_remote_cnt u32 */
/*       18 s_original u8                                                        */
/* ins:  order     0..6  o_id,o_d,o_w,o_c,o_entry_d,o_ol_cnt,o_all_local (u32)     */
/*       new_order 7..9  no_o_id,no_d,no_w                                         */
/*       order_line 10..17 ol_o_id,ol_d,ol_w,ol_number,ol_i_id,ol_supply_w,        */
/*                        ol_quantity (u32), ol_amount (i32)                       */
/*       history   18..24 h_c,h_cd,h_cw,h_d,h_w,h_date (u32), h_amount (i32)       */
/* nrows[0]=order, [1]=new_order, [2]=order_line, [3]=history                      */
/* ============================================================================ */
#define U32(i) ((uint32_t*)ins[i])

/* customer selected by last name (Ext TPC-C 2.5.2.2): the customers of (w, d)
 * with C_LAST = last, sorted by C_FIRST, row ceil(n/2) (1-based).  Linear scan. */
static int64_t tpcc_by_last(void** cols, const uint32_t* dims, uint32_t w, uint32_t d, uint32_t last)
{
    const uint16_t* c_last = cols[10];
    const uint64_t* c_first = cols[11];
    uint64_t C = dims[2], base = ((uint64_t)w * dims[1] + d) * C;
    uint32_t* hit = malloc(sizeof(uint32_t) * C);
    uint32_t nh = 0;
    for (uint32_t c = 0; c < C; ++c)
        if (c_last[base + c] == last) hit[nh++] = c;
    /* insertion sort by (c_first, c) */
    for (uint32_t a = 1; a < nh; ++a) {
        uint32_t x = hit[a];
        int64_t b = (int64_t)a - 1;
        while (b >= 0 && (c_first[base + hit[b]] > c_first[base + x] ||
                          (c_first[base + hit[b]] == c_first[base + x] && hit[b] > x))) {
            hit[b + 1] = hit[b];
            --b;
        }
        hit[b + 1] = x;
    }
    int64_t r = nh ? (int64_t)hit[(nh + 1) / 2 - 1] : -1;
    free(hit);
    return r;
}

static void tpcc_txn(void** cols, const uint32_t* dims, int type, const uint32_t* p, uint64_t ts,
                     uint8_t* st, uint8_t* out, void** ins, uint64_t* nrows)
{
    uint64_t W = dims[0], D = dims[1], C = dims[2], I = dims[3];
    (void)W;
    int64_t* w_ytd = cols[0]; int32_t* w_tax = cols[1];
    int64_t* d_ytd = cols[2]; int32_t* d_tax = cols[3]; uint32_t* d_next = cols[4];
    int64_t* c_bal = cols[5]; int64_t* c_ytd = cols[6]; uint32_t* c_cnt = cols[7];
    int32_t* c_disc = cols[8]; uint8_t* c_credit = cols[9];
    int32_t* i_price = cols[12]; uint8_t* i_orig = cols[13];
    int32_t* s_qty = cols[14]; int64_t* s_ytd = cols[15]; uint32_t* s_ocnt = cols[16];
    uint32_t* s_rcnt = cols[17]; uint8_t* s_orig = cols[18];
    *st = 0;
    if (type == 0) { /* NewOrder(w, d, c, ol_cnt, lines) */
        uint32_t w = p[0], d = p[1], c = p[2], n = p[3];
        const uint32_t* L = p + 4;
        /* phase 1 (read-only): an unused item id rolls the order back (2.4.2.3) */
        for (uint32_t l = 0; l < n; ++l)
            if (L[3 * l] >= I) { *st = 1; return; }
        uint64_t wd = (uint64_t)w * D + d, wdc = wd * C + c;
        uint32_t o_id = d_next[wd];
        d_next[wd] = o_id + 1;
        uint32_t all_local = 1;
        for (uint32_t l = 0; l < n; ++l) all_local &= (L[3 * l + 1] == w);
        uint64_t r = nrows[0]++;
        U32(0)[r] = o_id; U32(1)[r] = d; U32(2)[r] = w; U32(3)[r] = c;
        U32(4)[r] = (uint32_t)ts; U32(5)[r] = n; U32(6)[r] = all_local;
        r = nrows[1]++;
        U32(7)[r] = o_id; U32(8)[r] = d; U32(9)[r] = w;
        int64_t sum = 0;
        for (uint32_t l = 0; l < n; ++l) {
            uint32_t i = L[3 * l], sw = L[3 * l + 1], q = L[3 * l + 2];
            uint64_t s = (uint64_t)sw * I + i;
            int32_t sq = s_qty[s];
            s_qty[s] = (sq >= (int32_t)q + 10) ? sq - (int32_t)q : sq - (int32_t)q + 91;
            s_ytd[s] += q;
            s_ocnt[s] += 1;
            if (sw != w) s_rcnt[s] += 1;
            int32_t amount = (int32_t)q * i_price[i];
            sum += amount;
            r = nrows[2]++;
            U32(10)[r] = o_id; U32(11)[r] = d; U32(12)[r] = w; U32(13)[r] = l;
            U32(14)[r] = i; U32(15)[r] = sw; U32(16)[r] = q; ((int32_t*)ins[17])[r] = amount;
            uint8_t* o = out + 16 + 12 * l;
            put_i32(o, sq);
            put_i32(o + 4, amount);
            o[8] = (uint8_t)(i_orig[i] && s_orig[s]);   /* brand-generic 'B' */
        }
        /* total = sum * (1 - c_discount) * (1 + w_tax + d_tax), rates in 1e-4,
         * rounded half up to a cent (DESIGN.md R-S14) */
        int64_t num = sum * (int64_t)(10000 - c_disc[wdc]) * (int64_t)(10000 + w_tax[w] + d_tax[wd]);
        int64_t total = (num + 50000000) / 100000000;
        put_u32(out, o_id);
        put_u32(out + 4, n);
        put_i64(out + 8, total);
        return;
    }
    if (type == 1) { /* Payment(w, d, cw, cd, by_name, c_or_last, h_amount) */
        uint32_t w = p[0], d = p[1], cw = p[2], cd = p[3], byname = p[4], h = p[6];
        int64_t c = byname ? tpcc_by_last(cols, dims, cw, cd, p[5]) : (int64_t)p[5];
        if (c < 0) { *st = 1; return; }
        uint64_t wd = (uint64_t)w * D + d;
        uint64_t cwdc = ((uint64_t)cw * D + cd) * C + (uint64_t)c;
        w_ytd[w] += h;
        d_ytd[wd] += h;
        c_bal[cwdc] -= h;
        c_ytd[cwdc] += h;
        c_cnt[cwdc] += 1;
        uint64_t r = nrows[3]++;
        U32(18)[r] = (uint32_t)c; U32(19)[r] = cd; U32(20)[r] = cw; U32(21)[r] = d;
        U32(22)[r] = w; U32(23)[r] = (uint32_t)ts; ((int32_t*)ins[24])[r] = (int32_t)h;
        put_u32(out, (uint32_t)c);
        put_u32(out + 4, c_credit[cwdc]);
        put_i64(out + 8, c_bal[cwdc]);
        return;
    }
    *st = 1;
}

/* ============================================================================ */
/* Micro benchmark (§6.1): "Each transaction reads a tuple, and     */
/* performs computation, and then writes the result back to the tuple.  The      */
/* amount of computation is simulated with calling the _sinf function (100 * x)   */
/* times."  dims = (N tuples, T types, x); params [tuple]; col 0 tuple (f32 bits). */
/* One "sin call" of type t (DESIGN.md R-M1): u = fma(v, A_t, B_t) keeps the      */
/* argument in [-1, 1] and makes every type a different function; then the odd   */
/* polynomial sin(u) ~ u * (1 + s*(C3 + s*C5)), s = u*u, with IEEE fma where     */
/* written and single rounding elsewhere, so the GPU evaluates it bit-exactly.     */
/* Output: the written value (u32 bits).  Never aborts.                            */
/* ============================================================================ */
static void micro_txn(void** cols, const uint32_t* dims, int type, const uint32_t* p, uint8_t* st, uint8_t* out)
{
    uint32_t* tup = (uint32_t*)cols[0];
    float v;
    memcpy(&v, &tup[p[0]], 4);
    const float A = 0.9375f - (float)type * 0.0078125f;        /* exact binary fractions */
    const float B = ((float)type - 15.5f) * 0.0009765625f;
    const float C3 = -0x1.555556p-3f, C5 = 0x1.111112p-7f;      /* -1/6, 1/120 rounded */
    const uint64_t calls = 100ull * dims[2];
    for (uint64_t j = 0; j < calls; ++j) {
        float u = fmaf(v, A, B);
        float s2 = u * u;
        float q = fmaf(s2, C5, C3);
        q = fmaf(s2, q, 1.0f);
        v = u * q;
    }
    memcpy(&tup[p[0]], &v, 4);
    memcpy(out, &v, 4);
    *st = 0;
}

/* ============================================================================ */
/* Definition 1: serial execution in increasing timestamp order                  */
/* ============================================================================ */
uint32_t orc_out_stride(int schema)
{
    return schema == S_TPCB ? OUT_TPCB : schema == S_TM1 ? OUT_TM1 : schema == S_TPCC ? OUT_TPCC
         : schema == S_MICRO ? OUT_MICRO : 0;
}

int orc_run(int schema, const uint32_t* dims, void** cols, uint64_t n, const uint8_t* type,
            const uint32_t* param_off, const uint32_t* param_words, uint64_t first_ts,
            uint8_t* status, uint8_t* out, void** ins, uint64_t* nrows)
{
    uint32_t stride = orc_out_stride(schema);
    if (!stride) return -1;
    memset(out, 0, stride * n);
    tm1_t tm1;
    if (schema == S_TM1) tm1 = tm1_bind(cols, dims);
    for (uint64_t i = 0; i < n; ++i) {           /* one at a time, ts = first_ts + i */
        const uint32_t* p = param_words + param_off[i];
        uint64_t ts = first_ts + i;
        uint8_t* o = out + stride * i;
        if (schema == S_TPCB && type[i] == 1) tpcb_withdraw(cols, p, &status[i], o);
        else if (schema == S_TPCB) tpcb_txn(cols, p, ts, &status[i], o, ins, nrows);
        else if (schema == S_TM1) tm1_txn(&tm1, type[i], p, &status[i], o);
        else if (schema == S_MICRO) micro_txn(cols, dims, type[i], p, &status[i], o);
        else tpcc_txn(cols, dims, type[i], p, ts, &status[i], o, ins, nrows);
        if (status[i]) memset(o, 0, stride);      /* an aborted txn returns no record */
    }
    return 0;
}

/* The same executor over an explicit order (a permutation of 0..n-1): transaction
 * order[k] runs k-th and keeps its own timestamp first_ts + order[k].  Serializability
 * without the timestamp constraint (Appendix G) means "equal to this loop
 * for SOME order"; the relaxed GPU strategies report the order they realised. */
int orc_run_order(int schema, const uint32_t* dims, void** cols, uint64_t n, const uint8_t* type,
                  const uint32_t* param_off, const uint32_t* param_words, uint64_t first_ts,
                  const uint32_t* order, uint8_t* status, uint8_t* out, void** ins, uint64_t* nrows)
{
    uint32_t stride = orc_out_stride(schema);
    if (!stride) return -1;
    memset(out, 0, stride * n);
    tm1_t tm1;
    if (schema == S_TM1) tm1 = tm1_bind(cols, dims);
    for (uint64_t k = 0; k < n; ++k) {
        uint64_t i = order[k];
        if (i >= n) return -2;
        const uint32_t* p = param_words + param_off[i];
        uint64_t ts = first_ts + i;
        uint8_t* o = out + stride * i;
        if (schema == S_TPCB && type[i] == 1) tpcb_withdraw(cols, p, &status[i], o);
        else if (schema == S_TPCB) tpcb_txn(cols, p, ts, &status[i], o, ins, nrows);
        else if (schema == S_TM1) tm1_txn(&tm1, type[i], p, &status[i], o);
        else if (schema == S_MICRO) micro_txn(cols, dims, type[i], p, &status[i], o);
        else tpcc_txn(cols, dims, type[i], p, ts, &status[i], o, ins, nrows);
        if (status[i]) memset(o, 0, stride);
    }
    return 0;
}

/* ============================================================================ */
/* Conflict footprint (basic operations) and depths  */
/* item = table tag << 48 | row;  mode 0 = read, 1 = write, 2 = add (commutative    */
/* increment; only with the ADD rule, SURVEY.md NEXT-1 / PAPER.md:475(c): two adds  */
/* of one item do not conflict, an add conflicts with reads and writes)            */
/* ============================================================================ */
enum { T_ACC = 1, T_TEL, T_BR, T_BIT1, T_VLR, T_SFDA, T_CF, T_DNEXT, T_STOCK, T_WYTD, T_DYTD, T_CUST, T_TUPLE };
#define ITEM(tag, row) (((uint64_t)(tag) << 48) | (uint64_t)(row))

static int add_op(uint64_t* it, uint8_t* md, int k, uint64_t item, uint8_t mode)
{
    for (int j = 0; j < k; ++j)
        if (it[j] == item) { if (md[j] != mode) md[j] = 1; return k; }   /* merge; differing modes -> W */
    it[k] = item;
    md[k] = mode;
    return k + 1;
}

/* Footprint of one transaction: only columns some registered type writes
 * produce operations (DESIGN.md R-S18).  Returns #ops (<= 16). */
static int footprint(int schema, const uint32_t* dims, void** cols, int type, const uint32_t* p,
                     uint64_t* it, uint8_t* md, int add_rule)
{
    int k = 0;
    /* balances / YTDs that only deposits / payments increment and no output reads */
    const uint8_t inc = add_rule ? 2 : 1;
    if (schema == S_TPCB) {
        k = add_op(it, md, k, ITEM(T_ACC, p[0]), 1);
        k = add_op(it, md, k, ITEM(T_TEL, p[1]), inc);
        k = add_op(it, md, k, ITEM(T_BR, p[2]), inc);
        return k;
    }
    if (schema == S_TM1) {
        tm1_t t = tm1_bind(cols, dims);
        int64_t s;
        switch (type) {
        case 0: s = p[0] - 1;
            k = add_op(it, md, k, ITEM(T_BIT1, s), 0);
            k = add_op(it, md, k, ITEM(T_VLR, s), 0);
            return k;
        case 1: s = p[0] - 1;
            for (int j = 0; j < 3; ++j)
                k = add_op(it, md, k, ITEM(T_CF, ((uint64_t)s * 4 + p[1] - 1) * 3 + j), 0);
            return k;
        case 2: return 0;
        case 3: s = p[0] - 1;
            k = add_op(it, md, k, ITEM(T_BIT1, s), 1);
            k = add_op(it, md, k, ITEM(T_SFDA, (uint64_t)s * 4 + p[1] - 1), 1);
            return k;
        case 4: s = tm1_lookup(&t, (uint64_t)p[0] | ((uint64_t)p[1] << 32));
            if (s < 0) return 0;
            return add_op(it, md, k, ITEM(T_VLR, s), 1);
        case 5: case 6: s = tm1_lookup(&t, (uint64_t)p[0] | ((uint64_t)p[1] << 32));
            if (s < 0) return 0;
            return add_op(it, md, k, ITEM(T_CF, ((uint64_t)s * 4 + p[2] - 1) * 3 + p[3] / 8), 1);
        }
        return 0;
    }
    if (schema == S_MICRO)          /* read, compute, write back: one write of the tuple */
        return add_op(it, md, k, ITEM(T_TUPLE, p[0]), 1);
    /* TPC-C */
    uint64_t D = dims[1], C = dims[2], I = dims[3];
    if (type == 0) {
        k = add_op(it, md, k, ITEM(T_DNEXT, (uint64_t)p[0] * D + p[1]), 1);
        for (uint32_t l = 0; l < p[3]; ++l) {
            uint32_t i = p[4 + 3 * l], sw = p[5 + 3 * l];
            if (i >= I) continue;
            k = add_op(it, md, k, ITEM(T_STOCK, (uint64_t)sw * I + i), 1);
        }
        return k;
    }
    int64_t c = p[4] ? tpcc_by_last(cols, dims, p[2], p[3], p[5]) : (int64_t)p[5];
    k = add_op(it, md, k, ITEM(T_WYTD, p[0]), inc);
    k = add_op(it, md, k, ITEM(T_DYTD, (uint64_t)p[0] * D + p[1]), inc);
    if (c >= 0) k = add_op(it, md, k, ITEM(T_CUST, ((uint64_t)p[2] * D + p[3]) * C + (uint64_t)c), 1);
    return k;
}

/* ops_off[n+1], items[], modes[] are filled; returns total ops or -1 if cap is short */
int64_t orc_footprint(int schema, const uint32_t* dims, void** cols, uint64_t n, const uint8_t* type,
                      const uint32_t* param_off, const uint32_t* param_words,
                      uint64_t* ops_off, uint64_t* items, uint8_t* modes, uint64_t cap, int add_rule)
{
    uint64_t tot = 0;
    uint64_t it[16];
    uint8_t md[16];
    for (uint64_t i = 0; i < n; ++i) {
        ops_off[i] = tot;
        int k = footprint(schema, dims, cols, type[i], param_words + param_off[i], it, md, add_rule);
        if (tot + k > cap) return -1;
        for (int j = 0; j < k; ++j) { items[tot + j] = it[j]; modes[tot + j] = md[j]; }
        tot += k;
    }
    ops_off[n] = tot;
    return (int64_t)tot;
}

/* Streaming depth recurrence.  Per item, over the accesses so far in ts order:
 *   rd = max depth of the last writer and the reads since it,
 *   ad = max depth of the last writer and the adds since it   (-1 if none).
 * A transaction's depth d = max over its operations of
 *   read: ad + 1,   add: rd + 1,   write: max(rd, ad) + 1     (0 if it has none);
 * then read: rd = max(rd, d); add: ad = max(ad, d); write: rd = ad = d.
 * Without adds ad is the last writer's depth and this is the (Wd, Md) recurrence. */
typedef struct { uint64_t key; int32_t rd, ad; } slot_t;

int orc_depths(uint64_t n, const uint64_t* ops_off, const uint64_t* items, const uint8_t* modes,
               uint32_t* depth)
{
    uint64_t nops = ops_off[n], cap = 16;
    while (cap < 2 * nops + 16) cap <<= 1;
    slot_t* tab = malloc(sizeof(slot_t) * cap);
    if (!tab) return -1;
    for (uint64_t j = 0; j < cap; ++j) tab[j].key = UINT64_MAX;
    for (uint64_t t = 0; t < n; ++t) {
        int32_t d = 0;
        for (uint64_t j = ops_off[t]; j < ops_off[t + 1]; ++j) {
            uint64_t h = (items[j] * 0x9E3779B97F4A7C15ull) & (cap - 1);
            while (tab[h].key != UINT64_MAX && tab[h].key != items[j]) h = (h + 1) & (cap - 1);
            if (tab[h].key == UINT64_MAX) { tab[h].key = items[j]; tab[h].rd = -1; tab[h].ad = -1; }
            const int32_t rd = tab[h].rd, ad = tab[h].ad;
            int32_t c = modes[j] == 0 ? ad + 1 : modes[j] == 2 ? rd + 1 : (rd > ad ? rd : ad) + 1;
            if (c > d) d = c;
        }
        for (uint64_t j = ops_off[t]; j < ops_off[t + 1]; ++j) {
            uint64_t h = (items[j] * 0x9E3779B97F4A7C15ull) & (cap - 1);
            while (tab[h].key != items[j]) h = (h + 1) & (cap - 1);
            if (modes[j] == 1) { tab[h].rd = d; tab[h].ad = d; }
            else if (modes[j] == 0) { if (d > tab[h].rd) tab[h].rd = d; }
            else if (d > tab[h].ad) tab[h].ad = d;
        }
        depth[t] = (uint32_t)d;
    }
    free(tab);
    return 0;
}
