// engine.cu — host runtime of the B200 GPUTx engine and the C ABI of include/gputx.h.
//
// Owns the HBM-resident column store and indexes, the bulk
// buffers, and the per-strategy pipelines:
//   K-SET: emit -> radix sort by item -> rank fixpoint -> group (depth, type) -> rounds
//   PART : fragments -> radix sort by partition -> bounds -> one thread per partition
//   TPL  : emit -> radix sort by item -> lock keys -> ts-ordered 2PL execution
#include <algorithm>
#include <cstdio>
#include <unistd.h>
#include <cstring>
#include <string>
#include <vector>
#include <emmintrin.h>

#include <nvtx3/nvToolsExt.h>         // header-only NVTX ranges: phases visible to nsys / ncu --nvtx

#include "../../include/gputx.h"
#include "common.cuh"
#include "kernels.cuh"
#include "schema.cuh"
#include "sort.cuh"

using namespace gputx;

namespace {

struct ColSpec {
    const char* name;
    uint32_t elem;
    uint64_t count;
};

struct InsSpec {
    const char* table;
    int table_id;
    std::vector<const char*> cols;
    uint32_t per_txn;
};

std::vector<ColSpec> column_specs(int schema, const uint32_t* d) {
    const uint64_t a = d[0], b = d[1], c = d[2], e = d[3];
    if (schema == S_TPCB)
        return {{"br_bal", 8, a}, {"tel_bal", 8, a * b}, {"acc_bal", 8, a * c}};
    if (schema == S_MICRO) return {{"tuple", 4, a}};          // f32 bit patterns
    if (schema == S_TM1) {
        const uint64_t P = a;
        return {{"sub_nbr", 8, P},      {"sub_bits", 2, P},     {"sub_hex", 8, P},       {"sub_byte2", 1, 10 * P},
                {"sub_msc", 4, P},      {"sub_vlr", 4, P},      {"ai_valid", 1, 4 * P},  {"ai_data1", 1, 4 * P},
                {"ai_data2", 1, 4 * P}, {"ai_data3", 4, 4 * P}, {"ai_data4", 8, 4 * P},  {"sf_valid", 1, 4 * P},
                {"sf_active", 1, 4 * P}, {"sf_error", 1, 4 * P}, {"sf_data_a", 1, 4 * P}, {"sf_data_b", 8, 4 * P},
                {"cf_live", 1, 12 * P}, {"cf_end", 1, 12 * P},  {"cf_numberx", 8, 12 * P}};
    }
    const uint64_t W = a, WD = a * b, WDC = a * b * c, I = e, WI = a * e;
    return {{"w_ytd", 8, W},          {"w_tax", 4, W},         {"d_ytd", 8, WD},          {"d_tax", 4, WD},
            {"d_next_o_id", 4, WD},   {"c_balance", 8, WDC},   {"c_ytd_payment", 8, WDC}, {"c_payment_cnt", 4, WDC},
            {"c_discount", 4, WDC},   {"c_credit", 1, WDC},    {"c_last", 2, WDC},        {"c_first", 8, WDC},
            {"i_price", 4, I},        {"i_original", 1, I},    {"s_quantity", 4, WI},     {"s_ytd", 8, WI},
            {"s_order_cnt", 4, WI},   {"s_remote_cnt", 4, WI}, {"s_original", 1, WI}};
}

std::vector<InsSpec> insert_specs(int schema) {
    if (schema == S_TPCB) return {{"history", 0, {"h_tid", "h_bid", "h_aid", "h_delta", "h_ts"}, 1}};
    if (schema == S_TPCC)
        return {{"order", T_ORDER, {"o_id", "o_d", "o_w", "o_c", "o_entry_d", "o_ol_cnt", "o_all_local"}, 1},
                {"new_order", T_NEWORDER, {"no_o_id", "no_d", "no_w"}, 1},
                {"order_line", T_OLINE,
                 {"ol_o_id", "ol_d", "ol_w", "ol_number", "ol_i_id", "ol_supply_w", "ol_quantity", "ol_amount"}, 15},
                {"history", T_HIST, {"h_c", "h_cd", "h_cw", "h_d", "h_w", "h_date", "h_amount"}, 1}};
    return {};
}

uint32_t ntypes_of(int schema, const uint32_t* d) {
    return schema == S_TPCB ? 2 : schema == S_TM1 ? 7 : schema == S_MICRO ? d[1] : 2;   // TPC-B: deposit, withdraw
}
uint32_t bits_for(uint64_t maxval) {   // bits to represent values in [0, maxval]
    uint32_t b = 0;
    while (b < 64 && (maxval >> b)) ++b;
    return b ? b : 1;
}

struct Col {
    ColSpec spec;
    void* d = nullptr;
    void* pristine = nullptr;
    bool loaded = false;
};
struct InsCol {
    std::string name;
    void* d = nullptr;
};
struct InsTable {
    std::string name;
    int table_id;
    uint32_t per_txn;
    uint64_t cap = 0, rows = 0, pending = 0;
    std::vector<InsCol> cols;
};

}  // namespace

struct gputx_db {
    gputx_db_config cfg{};
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    std::string err;
    int schema = 0;
    uint32_t ntypes = 0, type_mask = 0;
    std::vector<Col> cols;
    std::vector<InsTable> ins;
    bool sealed = false, submitted = false, executed = false, poisoned = false;
    bool exec_pending = false;                // gputx_execute_async launched, gputx_wait not yet
    int exec_st = 0;                          // its requested strategy
    int last_strategy = -1;
    int chosen = -1;                          // strategy that ran for the last execute
    // Algorithm 1 thresholds (gputx_set_chooser); w0_bar 0 => 64 x #SMs.  Calibrated on
    // B200 by tools/calibrate_chooser.py (profiles/round1_chooser_calibration.json): d_bar = 0
    // (PART whenever K-SET is not chosen) lifts the mean chosen/best throughput 0.70 -> 0.88
    uint64_t ch_w0 = 0, ch_d = 0, ch_c = 0;
    uint64_t n = 0, first_ts = 0, next_ts = 0, max_bulk = 0, max_words = 0, max_rec = 0, n_items = 0;
    uint32_t item_bits = 0;
    uint32_t nparts = 0, part_bits = 0, part_size = 128;
    // bulk + results
    uint8_t* d_type = nullptr;
    uint32_t* d_poff = nullptr;
    uint32_t* d_pw = nullptr;
    uint8_t* d_status = nullptr;
    uint8_t* d_out = nullptr;
    bool packed = false;               // GPUTX_FLAG_PACKED_OUT
    bool rec_at_ingest = false;        // this submit counted the access records (emit skips its count pass)
    bool deferred = false;             // GPUTX_FLAG_DEFERRED_CHECK: this bulk's validation verdict is pending
    bool guard = false;                // ... and its kernels treat a failed ingest as an empty bulk
    LookBack<uint2> lb_scan2{};        // paired scan (output sizes + record counts)
    uint32_t* d_out_off = nullptr;     // packed record offsets [n + 1]
    uint64_t out_bytes = 0;            // the submitted bulk's output bytes (packed: out_off[n])
    uint32_t out_stride = 0;
    uint32_t* d_ins_off = nullptr;   // 4 * (max_bulk + 1)
    // indexes
    uint64_t* d_hkeys = nullptr;
    uint32_t* d_hvals = nullptr;
    uint64_t hmask = 0;
    uint32_t* d_name_sorted = nullptr;
    uint32_t* d_name_off = nullptr;
    std::vector<uint64_t> h_nbr;
    std::vector<uint16_t> h_last;
    std::vector<uint64_t> h_first;
    // workspaces
    uint64_t* d_rec_a = nullptr;
    uint64_t* d_rec_b = nullptr;
    uint64_t* d_sorted = nullptr;
    uint64_t* d_item_sorted = nullptr;  // records in (item, ts) order after the K-SET sort (or null)
    int kset_df = -1;                   // K-SET executor: 1 dataflow, 0 rounds, -1 schema default
    bool kset_ran_df = false;
    bool ins_dense = false;
    uint32_t* h_sc_dev = nullptr;       // device alias of the mapped host counters
    // pipelined gputx_run_bulks (no host round trip per bulk): per-bulk counter slots in
    // mapped host memory, the failed-bulk guard and the run's poison word
    bool pipe = false;
    uint32_t* pull_target = nullptr;    // device alias where pull_sc writes (nullptr: h_sc_dev)
    uint32_t* h_slots = nullptr;        // [slots_cap][SC_COUNT] mapped
    uint32_t* h_slots_dev = nullptr;
    uint64_t slots_cap = 0;
    uint32_t* d_poison = nullptr;
    uint8_t *tm1_sub = nullptr, *tm1_ai = nullptr, *tm1_sf = nullptr, *tm1_cf = nullptr;   // TM-1 row groups
    bool rows_dirty = false;            // TM-1: rows hold newer mutable fields than the columns
    // gputx_run_bulks: copy streams and double-buffered device slots (lazily created)
    cudaStream_t st_h2d = nullptr, st_d2h = nullptr;
    cudaEvent_t ev_in[2] = {}, ev_in_free[2] = {}, ev_res[2] = {}, ev_res_free[2] = {};
    uint8_t* in_type[2] = {};
    uint32_t *in_poff[2] = {}, *in_pw[2] = {};
    uint8_t *res_status[2] = {}, *res_out[2] = {};
    // peer-memory exchange (gputx_shard_export / connect / dispatch / receive / return / collect)
    uint32_t* arena = nullptr;          // this shard's arena (cudaMalloc: exportable by IPC)
    uint64_t arena_words = 0, ret_base = 0;
    uint32_t fwd_cap = 0, ret_cap = 0, xepoch = 0;
    uint32_t* d_done_ctas = nullptr;
    PeerTable pt{};
    bool p2p = false;
    std::vector<void*> ipc_open;
    uint32_t kset_df_ahead = 0;         // dataflow look-ahead throttle in k-sets, 0 = off (GPUTX_KSET_DF_AHEAD)
    uint32_t kset_df_grid = 0;          // dataflow persistent grid cap (GPUTX_KSET_DF_GRID), 0 = co-resident
    uint32_t* d_cnt = nullptr;       // max(max_bulk, max_rec) + 1
    uint32_t* d_rec_off = nullptr;   // max_bulk + 1
    uint32_t* d_D = nullptr;
    uint32_t* d_perm = nullptr;
    uint32_t* d_gcnt = nullptr;      // max_bulk * ntypes + 2
    uint32_t* d_goff = nullptr;
    uint32_t* d_lock = nullptr;
    uint32_t* d_lkey = nullptr;
    uint32_t* d_part_off = nullptr;
    uint16_t* d_g = nullptr;         // CTAs per k-set round
    uint8_t* d_ptype = nullptr;      // types in k-set execution order
    uint32_t* d_pp = nullptr;        // first 8 parameter words in k-set execution order
    uint64_t* d_trace = nullptr;     // per-round start times (ns), CTA 0, when trace_rounds
    bool trace_rounds = false;
    uint32_t* d_done = nullptr;      // per-round completion counters
    uint32_t* d_sc = nullptr;
    uint32_t* h_sc = nullptr;        // pinned mirror
    GridBar* d_bar = nullptr;
    uint32_t* d_tickets = nullptr;   // [256]
    LookBack<uint32_t> lb_scan{};
    LookBack<Xf> lb_rank{};
    LookBack<Pair> lb_tpl{};
    RkMemo rank_memo{};               // per-tile memo of the rank passes
    uint64_t* d_rtrace = nullptr;     // rank pass phase times (diagnostics)
    SortWs sort_ws{};
    uint32_t epoch = 0;        // look-back epochs of scans / sorts / TPL keys
    uint32_t rank_epoch = 0;   // look-back epochs of rank passes (own array)
    uint32_t ticket_slot = 0;
    int nsm = 0;
    int rank_grid = 0, kset_grid = 0, kset_grid_ts = 0;
    uint32_t rank_local = RK_LOCAL_DEFAULT;   // GPUTX_RANK_LOCAL overrides (experiments)
    uint32_t rank_dirty = 1;                  // dirty-tile worklist (GPUTX_RANK_DIRTY overrides)
    uint32_t rank_root = 0;                   // root-local sweeps (GPUTX_RANK_ROOT overrides)
    uint32_t rank_stream = 1;                 // TM-1 per-subscriber streaming rank (GPUTX_RANK_STREAM overrides)
    uint32_t rank_spine = 1;                  // TPC-B / TPC-C / micro spine-streaming rank (GPUTX_RANK_SPINE)
    int32_t* d_lastw = nullptr;               // spine rank: latest write before each record
    uint32_t *d_sp = nullptr, *d_lcnt = nullptr, *d_loff = nullptr, *d_lfill = nullptr, *d_links = nullptr;
    uint32_t *d_heads = nullptr, *d_ccur = nullptr;
    int32_t* d_clast = nullptr;
    LookBack<SegMax> lb_seg{};
    int sp_grid = 0;
    bool spine_ran = false;                   // this bulk's depths came from the spine rank
    uint8_t* d_cpub = nullptr;                // chain executor: transaction another chain waits for
    uint32_t* d_cdone = nullptr;              // chain executor: done[t] == chain_epoch
    uint32_t chain_epoch = 0;
    int chain_cap = 0;                        // co-resident chain threads
    bool kset_ran_chain = false;
    uint32_t rank_window = 0;                 // TPC-C windowed rank: log2 window (GPUTX_RANK_WINDOW overrides)
    int rank_window_grid = 0;
    uint32_t rank_window_cluster = 0;         // 0: cooperative grid with grid barriers (GPUTX_RANK_WCLUSTER)
    uint32_t* d_wseg = nullptr;               // window -> first sorted record
    int2* d_wst = nullptr;                    // item -> (a, m) at the end of the previous windows
    bool rec_item_sorted = false;             // d_sorted holds records in (item, ts) order
    int rank_root_grid = 0;
    uint32_t kset_q = 128;     // max transactions per CTA per k-set round (GPUTX_KSET_Q overrides)
    uint32_t group_p = 0;      // type groups per k-set (gputx_set_grouping; 0 = one per type)
    bool sync_stages = false;  // GPUTX_SYNC (diagnostics): synchronise and check after each stage
    uint32_t kset_diag = 0;    // GPUTX_KSET_DIAG (diagnostics): 1 skip bodies, 8 skip prefetch, 128 hand-off skeleton
    uint32_t exec_grid_override = 0;
    bool tpl_persistent = false;   // GPUTX_TPL_PERSISTENT=1: persistent per-lane tickets (slower: divergent spinners)
    uint32_t kset_cluster = 8;     // CTAs per thread-block cluster of the K-SET executor
    // owner-local K-SET rounds: GPUTX_KSET_OWN=0 restores the global rounds
    int kset_own = 1;
    int kset_chain = 1;                // TPC-B: K-SET over spine chains (GPUTX_KSET_CHAIN=0: owner warps)
    int chain_runs = 1;                // lane-parallel deposit runs (GPUTX_CHAIN_RUNS=0: lane 0 only)
    int own_pipe = 1;                  // owner-local rounds staged through the perm (GPUTX_OWN_PIPE=0: gather pass)
    bool kset_ran_own = false;
    int own_grid[2] = {0, 0};          // co-resident CTAs of the executor without / with waits
    uint32_t own_g = 0, own_nw = 0;    // this bulk's executor grid and owner warps
    uint32_t* d_oseg = nullptr;        // owner segments [OWN_MAXW + 1] and the sort count word
    uint32_t* d_prog = nullptr;        // per-warp progress [OWN_MAXW]
    uint32_t* d_own = nullptr;         // per-transaction owner (dependency pass)
    uint32_t* d_oout = nullptr;        // packed output offsets in owner order
    unsigned long long* d_wait = nullptr;   // per-transaction cross-owner wait
    unsigned long long* d_owait = nullptr;  // the same in owner order
    uint8_t* d_pub = nullptr;          // per-transaction "another warp waits for me"
    cudaEvent_t ev[8] = {};
    cudaEvent_t ev_sub[2] = {};       // submit start / end (ms_ingest)
    cudaEvent_t ev_x[4] = {};         // sharded exchange: pack start/end, merge start/end (ms_exchange)
    bool have_x = false;
    bool has_depth = false, has_perm = false;
    uint64_t launches = 0;     // kernels launched since the last submit
    // timestamps and shards
    uint32_t* d_ts = nullptr;        // global ts per bulk position (when has_ts)
    bool has_ts = false;
    uint32_t nshards = 1, shard = 0, nroot = 1, root_lo = 0, root_hi = 1;
    uint32_t* d_src = nullptr;       // sharded: home-bulk index or NOT_HOME
    uint32_t* d_home_pos = nullptr;  // sharded: bulk position of home transaction i
    uint8_t* d_xflag = nullptr;      // sharded: has a fragment on another shard
    uint8_t* s_type = nullptr;       // sharded: staged home bulk (gputx_shard_pack)
    uint32_t *s_poff = nullptr, *s_pw = nullptr, *s_ts = nullptr;
    uint8_t *d_hstatus = nullptr, *d_hout = nullptr;   // sharded: home results in home order
    uint32_t* d_order = nullptr;     // relaxed strategies: the serialization order they produced
    UndoRec* d_undo = nullptr;       // undo-log slots (TPC-B WITHDRAW, a non-two-phase type)
    bool has_order = false;
    // streaming K-SET pool (gputx_pool_*): pending transactions live in d_type/d_poff/d_pw/d_ts
    // (positions 0..pool_n-1, ts order); their sorted access records in d_prec
    bool pool_ready = false;
    uint64_t pool_n = 0, pool_words = 0, pool_nrec = 0, pool_exec = 0;
    uint64_t *d_prec = nullptr, *d_prec2 = nullptr;
    uint32_t *d_pins = nullptr, *q_ins = nullptr, *st_ins = nullptr;   // per-table insert counts
    uint8_t* q_type = nullptr;
    uint32_t *q_poff = nullptr, *q_pw = nullptr, *q_ts = nullptr;      // compaction targets
    uint32_t *d_zflag = nullptr, *d_fna = nullptr, *d_list = nullptr, *d_npos = nullptr, *d_noff = nullptr,
             *d_rpos = nullptr, *d_rts = nullptr;
    uint8_t *d_rstatus = nullptr, *d_rout = nullptr;
    uint64_t nh = 0;                 // sharded: home transactions staged / in the bulk
    bool staged = false, returned = false;
};

namespace {

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            db->err = std::string(#x) + ": " + cudaGetErrorString(e_);                          \
            return GPUTX_ECUDA;                                                                 \
        }                                                                                       \
    } while (0)

gputx_status fail(gputx_db* db, gputx_status s, const std::string& m) {
    if (db) db->err = m;
    return s;
}

// device counters -> mapped host counters (kernel stores, no copy engine); read by the host
// after it synchronises the stream
gputx_status pull_sc(gputx_db* db, cudaStream_t s) {
    pull_sc_kernel<<<1, 64, 0, s>>>(db->d_sc, db->pull_target ? db->pull_target : db->h_sc_dev, SC_COUNT);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(db, GPUTX_ECUDA, std::string("pull_sc: ") + cudaGetErrorString(e));
    return GPUTX_OK;
}

// the first bad transaction of the last validating kernel and its error code (report_err)
uint64_t err_packed(const gputx_db* db) {
    return (uint64_t)db->h_sc[SC_ERRPK] | ((uint64_t)db->h_sc[SC_ERRPK + 1] << 32);
}
uint32_t err_code(const gputx_db* db) { return (uint32_t)(err_packed(db) & 0xFFu); }
uint32_t err_idx(const gputx_db* db) { return (uint32_t)(err_packed(db) >> 8); }

template <class T>
gputx_status dalloc(gputx_db* db, T** p, uint64_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    if (db->cfg.alloc) {        // the caller's allocator (e.g. PyTorch's caching allocator)
        *p = (T*)db->cfg.alloc(count * sizeof(T), (void*)db->stream, db->cfg.alloc_ctx);
        if (!*p) {
            db->err = "cfg.alloc(" + std::to_string(count * sizeof(T)) + ") returned NULL";
            return GPUTX_ENOMEM;
        }
        return GPUTX_OK;
    }
    cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
    if (e != cudaSuccess) {
        db->err = std::string("cudaMalloc(") + std::to_string(count * sizeof(T)) + "): " + cudaGetErrorString(e);
        return GPUTX_ENOMEM;
    }
    return GPUTX_OK;
}

void dfree(gputx_db* db, void* p) {
    if (!p) return;
    if (db->cfg.free) db->cfg.free(p, (void*)db->stream, db->cfg.alloc_ctx);
    else cudaFree(p);
}

#define STAGE(name)                                                                             \
    do {                                                                                        \
        if (db->sync_stages) {                                                                  \
            cudaError_t e_ = cudaStreamSynchronize(db->stream);                                 \
            if (e_ != cudaSuccess) return fail(db, GPUTX_ECUDA, std::string(name) + ": " + cudaGetErrorString(e_)); \
        }                                                                                       \
    } while (0)
// NVTX range per pipeline phase (host side; ncu --nvtx --nvtx-include "gputx.rank/" etc.)
struct NvtxRange {
    explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
    ~NvtxRange() { nvtxRangePop(); }
};
#define NVTX_SCOPE(name) NvtxRange nvtx_scope_(name)
#define TRY(x)                              \
    do {                                    \
        gputx_status s_ = (x);              \
        if (s_ != GPUTX_OK) return s_;      \
    } while (0)

uint32_t* next_ticket(gputx_db* db) {
    // 256 ticket counters zeroed together; a slot is used once per memset cycle
    if (db->ticket_slot == 0) dev_fill(db->d_tickets, 0, 256 * sizeof(uint32_t), db->stream);
    uint32_t* t = db->d_tickets + db->ticket_slot;
    db->ticket_slot = (db->ticket_slot + 1) & 255u;
    return t;
}

// exclusive scan of n (device or host count) u32 values; out[n] = total
void scan_u32(gputx_db* db, const uint32_t* in, uint32_t* out, const uint32_t* n_dev, uint64_t n_max, uint32_t* total) {
    const uint32_t grid = (uint32_t)((n_max + SC_TILE) / SC_TILE);
    ++db->epoch;
    scan_kernel<<<grid, SC_THREADS, 0, db->stream>>>(in, out, n_dev, (uint32_t)n_max, db->lb_scan, db->epoch,
                                                     next_ticket(db), total);
                                                     ++db->launches;
}

// exclusive scans of two u32 arrays in one pass; outX[n], outY[n] and the totals set
void scan2_u32(gputx_db* db, const uint32_t* inX, const uint32_t* inY, uint32_t* outX, uint32_t* outY, uint64_t n,
               uint32_t* totX, uint32_t* totY) {
    const uint32_t grid = (uint32_t)((n + SC_TILE) / SC_TILE);
    ++db->epoch;
    scan2_kernel<<<grid, SC_THREADS, 0, db->stream>>>(inX, inY, outX, outY, (uint32_t)n, db->lb_scan2, db->epoch,
                                                      next_ticket(db), totX, totY);
    ++db->launches;
}

DevDb make_devdb(gputx_db* db) {
    DevDb v{};
    v.schema = db->schema;
    for (int k = 0; k < 4; ++k) v.dims[k] = db->cfg.dims[k];
    v.ntypes = db->ntypes;
    v.n = (uint32_t)db->n;
    v.first_ts = (uint32_t)db->first_ts;
    v.type = db->d_type;
    v.poff = db->d_poff;
    v.pw = db->d_pw;
    v.status = db->d_status;
    v.out = db->d_out;
    v.out_stride = db->out_stride;
    v.out_off = db->packed ? db->d_out_off : nullptr;
    for (size_t k = 0; k < db->cols.size() && k < (size_t)MAX_COLS; ++k) v.col[k] = db->cols[k].d;
    int c = 0;
    for (auto& t : db->ins) {
        v.ins_base[t.table_id] = t.rows;
        for (auto& ic : t.cols) v.ins[c++] = ic.d;
    }
    v.ins_off = db->d_ins_off;
    v.ins_stride = (uint32_t)(db->n + 1);
    v.hkeys = db->d_hkeys;
    v.hvals = db->d_hvals;
    v.hmask = db->hmask;
    v.name_sorted = db->d_name_sorted;
    v.name_off = db->d_name_off;
    v.part_size = db->part_size;
    v.add_rule = (db->cfg.flags & GPUTX_FLAG_ADD_RULE) ? 1u : 0u;
    v.nshards = db->nshards;
    v.err = (db->pipe || db->guard) ? db->d_sc + SC_ERR : nullptr;
    v.poison = db->pipe ? db->d_poison : nullptr;
    v.shard = db->shard;
    v.nroot = db->nroot;
    v.root_lo = db->root_lo;
    v.root_hi = db->root_hi;
    v.ts = db->has_ts ? db->d_ts : nullptr;
    v.src = db->nshards > 1 ? db->d_src : nullptr;
    v.xflag = db->nshards > 1 ? db->d_xflag : nullptr;
    v.undo = db->d_undo;
    v.ins_dense = db->ins_dense ? 1u : 0u;
    v.tm1_sub = db->tm1_sub;
    v.tm1_ai = db->tm1_ai;
    v.tm1_sf = db->tm1_sf;
    v.tm1_cf = db->tm1_cf;
    return v;
}

template <class K>
int coop_grid(gputx_db* db, K kernel, int block, size_t smem) {
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, block, smem);
    if (per < 1) per = 1;
    return per * db->nsm;
}

gputx_status launch_coop(gputx_db* db, const void* fn, int grid, int block, void** args) {
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(block), args, 0, db->stream);
    if (e != cudaSuccess) return fail(db, GPUTX_ECUDA, std::string("cooperative launch: ") + cudaGetErrorString(e));
    return GPUTX_OK;
}

uint32_t grid_for(uint64_t n, uint32_t block, uint32_t cap) {
    uint64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (uint32_t)g;
}

// ------------------------------------------------------------------------------- K-SET
// parameter words staged in registers by the K-SET executor (0: read from HBM)
template <int S> constexpr int kset_pw() { return S == S_TPCB || S == S_MICRO ? 4 : S == S_TM1 ? 8 : 0; }
// executor CTA size: 256 for TM-1 / TPC-B (a round's CTA holds <= Q = 128 / 32 transactions;
// smaller CTAs make its barriers cheaper: TM-1 exec 0.428 -> 0.408 ms, TPC-B 12.0 -> 10.0 ms;
// 128 / 64 measured no better, tools/gpu_kb_sweep.sh), TPC-C 256 (one warp per
// transaction), micro 1024 (compute-heavy types)
template <int S> constexpr int kset_block() { return S == S_MICRO ? KX_THREADS : 256; }
template <int S> const void* kset_fn(bool sh) {
    return sh ? (const void*)kset_exec_kernel<S, kset_pw<S>(), kset_block<S>(), true>
              : (const void*)kset_exec_kernel<S, kset_pw<S>(), kset_block<S>(), false>;
}
template <int S>
gputx_status emit_records(gputx_db* db, const DevDb& v) {
    const uint32_t g = grid_for(db->n, 256, 148 * 16);
    if (!db->rec_at_ingest) {                 // (counted and scanned at submit otherwise)
        emit_count_kernel<S><<<g, 256, 0, db->stream>>>(v, db->d_cnt);
        ++db->launches;
        scan_u32(db, db->d_cnt, db->d_rec_off, nullptr, db->n, db->d_sc + SC_NREC);
    }
    emit_write_kernel<S><<<g, 256, 0, db->stream>>>(v, db->d_rec_off, db->d_rec_a);
    ++db->launches;
    return GPUTX_OK;
}

gputx_status sort_records(gputx_db* db, uint32_t lo, uint32_t nbits, const uint32_t* n_dev, uint64_t n_max) {
    db->d_sorted = radix_sort_u64(db->d_rec_a, db->d_rec_b, n_dev, n_max, lo, nbits, db->sort_ws, db->epoch, db->stream);
    db->launches += 2 + (nbits + 7) / 8;
    return GPUTX_OK;
}

// Spine-streaming rank: links from the (item, ts)-sorted records, then one
// warp per chain walks its members in ts order (kernels.cuh "Spine-streaming rank").
template <int S>
gputx_status spine_rank(gputx_db* db) {
    cudaStream_t s = db->stream;
    const uint64_t NB = db->max_bulk, MR = db->max_rec;
    if (!db->d_lastw) {
        gputx_status st;
        const uint64_t tiles = MR / SC_TILE + 4;
        if ((st = dalloc(db, &db->d_lastw, MR)) || (st = dalloc(db, &db->d_sp, NB + 1)) ||
            (st = dalloc(db, &db->d_lcnt, NB + 1)) || (st = dalloc(db, &db->d_loff, NB + 2)) ||
            (st = dalloc(db, &db->d_lfill, NB + 1)) || (st = dalloc(db, &db->d_links, MR)) ||
            (st = dalloc(db, &db->d_heads, NB + 1)) || (st = dalloc(db, &db->d_ccur, NB + 1)) ||
            (st = dalloc(db, &db->d_clast, NB + 1)) || (st = dalloc(db, &db->d_cpub, NB + 1)) ||
            (st = dalloc(db, &db->d_cdone, NB + 1)) || (st = dalloc(db, &db->lb_seg.flag, tiles)) ||
            (st = dalloc(db, &db->lb_seg.agg, tiles)) || (st = dalloc(db, &db->lb_seg.inc, tiles)))
            return st;
        dev_fill(db->lb_seg.flag, 0, tiles * 4, s);
        dev_fill(db->d_cdone, 0, (NB + 1) * 4, s);
        int perc = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&perc, kset_chain_exec_kernel<S_TPCB>, 128, 0);
        db->chain_cap = std::max(1, perc) * db->nsm * 4;              // chains (one per warp)
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, sp_walk_kernel<S>, 256, 0);
        db->sp_grid = std::max(1, per) * db->nsm;
    }
    const uint64_t n = db->n;
    CK(dev_fill_multi(s, {fseg(db->d_D, 0xFF, n * 4), fseg(db->d_lcnt, 0, (n + 1) * 4), fseg(db->d_lfill, 0, n * 4),
                          fseg(db->d_sc + SC_NCHAIN, 0, 4), fseg(db->d_cpub, 0, S != S_MICRO ? n : 0)}));
    ++db->launches;
    ++db->epoch;
    const uint32_t tiles = (uint32_t)((db->max_rec + SC_TILE - 1) / SC_TILE);
    lastw_kernel<S><<<tiles, SC_THREADS, 0, s>>>(db->d_sorted, db->d_sc + SC_NREC, db->lb_seg, db->epoch,
                                                  next_ticket(db), db->d_lastw, db->d_sp);
    const uint32_t g = grid_for(db->max_rec, 256, (uint32_t)db->nsm * 8);
    sp_count_kernel<S><<<g, 256, 0, s>>>(db->d_sorted, db->d_sc + SC_NREC, db->d_lastw, db->d_sp, db->d_lcnt);
    scan_u32(db, db->d_lcnt, db->d_loff, nullptr, n, nullptr);
    sp_fill_kernel<S><<<g, 256, 0, s>>>(db->d_sorted, db->d_sc + SC_NREC, db->d_lastw, db->d_sp, db->d_loff,
                                         db->d_lfill, db->d_links, db->d_heads, db->d_sc + SC_NCHAIN,
                                         S != S_MICRO ? db->d_cpub : nullptr);
    db->launches += 3;
    const uint64_t* keys = db->d_sorted;
    const uint32_t* nrec = db->d_sc + SC_NREC;
    const uint32_t* heads = db->d_heads;
    const uint32_t* nh = db->d_sc + SC_NCHAIN;
    const uint32_t* loff = db->d_loff;
    const uint32_t* links = db->d_links;
    uint32_t* D = db->d_D;
    uint32_t* cur = db->d_ccur;
    int32_t* last = db->d_clast;
    uint32_t* sc = db->d_sc;
    void* args[] = {&keys, &nrec, &heads, &nh, &loff, &links, &D, &cur, &last, &sc};
    TRY(launch_coop(db, (const void*)sp_walk_kernel<S>, db->sp_grid, 256, args));
    ++db->launches;
    return GPUTX_OK;
}

// K-SET part 1 (also the analysis half of GPUTX_AUTO): emit, sort, rank fixpoint, and
// the depth reduction giving d = max depth and w0 = |0-set|
template <int S>
gputx_status kset_rank(gputx_db* db, const DevDb& v) {
    NVTX_SCOPE("gputx.kset.emit_sort_rank");
    cudaStream_t s = db->stream;
    cudaEventRecord(db->ev[1], s);
    TRY(emit_records<S>(db, v));
    STAGE("emit");
    cudaEventRecord(db->ev[2], s);
    // TM-1: single-subscriber transactions -> sort on the subscriber bits only and run
    // the exact streaming recurrence per subscriber (rank_stream_tm1_kernel)
    const bool stream = S == S_TM1 && db->rank_stream;
    // spine-streaming rank (TPC-B / TPC-C / micro under the R/W rule, unsharded)
    const bool spine = S != S_TM1 && db->rank_spine && !db->has_ts && !(db->cfg.flags & GPUTX_FLAG_ADD_RULE) &&
                       db->item_bits <= 32;
    // TPC-C: windowed rank -> (window, item, ts) order: stable sort on the item bits, then
    // on the window bits of the transaction index (key bits [6 + WB, 30))
    const uint32_t wb = db->rank_window;
    const bool windowed = !spine && S == S_TPCC && wb && db->n > (1ull << wb);
    const uint32_t nwin = windowed ? (uint32_t)((db->n - 1) >> wb) + 1 : 1;
    if (stream)
        TRY(sort_records(db, KEY_ITEM_SHIFT + TM1_COMP_BITS, db->item_bits - TM1_COMP_BITS, db->d_sc + SC_NREC,
                         db->max_rec));
    else
        TRY(sort_records(db, KEY_ITEM_SHIFT, db->item_bits, db->d_sc + SC_NREC, db->max_rec));
    db->d_item_sorted = stream ? nullptr : db->d_sorted;   // (item, ts) order (TPL keys / K-SET dataflow)
    if (windowed) {
        uint64_t* other = db->d_sorted == db->d_rec_a ? db->d_rec_b : db->d_rec_a;
        db->d_sorted = radix_sort_u64(db->d_sorted, other, db->d_sc + SC_NREC, db->max_rec, 6 + wb, bits_for(nwin - 1),
                                      db->sort_ws, db->epoch, s);
        db->launches += 2 + (bits_for(nwin - 1) + 7) / 8;
        // one 8-bit pass reads the item-sorted buffer and writes the other: the item order
        // survives for the dataflow executor (more passes would overwrite it)
        if ((bits_for(nwin - 1) + 7) / 8 != 1) db->d_item_sorted = nullptr;
    }
    db->rec_item_sorted = !stream && !windowed;
    STAGE("sort");
    cudaEventRecord(db->ev[3], s);
    // rank fixpoint (persistent, cooperative)
    CK(dev_fill_multi(s, {fseg(db->d_D, 0, db->n * sizeof(uint32_t)), fseg(&db->d_bar->dead, 0, sizeof(uint32_t))}));
    db->spine_ran = spine;
    if (spine) {
        TRY(spine_rank<S>(db));
    } else if (windowed) {
        win_bounds_kernel<<<grid_for(db->max_rec + 1, 256, 148 * 8), 256, 0, s>>>(db->d_sorted, db->d_sc + SC_NREC, wb,
                                                                             nwin, db->d_wseg);
        ++db->launches;
        CK(dev_fill(db->d_wst, 0xFF, db->n_items * sizeof(int2), s));     // (-1, -1): no access yet
        const uint64_t* keys = db->d_sorted;
        const uint32_t* seg = db->d_wseg;
        uint32_t nw = nwin;
        uint32_t* D = db->d_D;
        int2* wst = db->d_wst;
        LookBack<Xf> lb = db->lb_rank;
        GridBar* bar = db->d_bar;
        uint32_t* sc = db->d_sc;
        uint32_t maxp = 1u << 16;
        uint32_t lmax = db->rank_local;
        void* args[] = {&keys, &seg, &nw, &D, &wst, &lb, &bar, &sc, &maxp, &lmax};
        if (db->rank_window_cluster) {           // one cluster; hardware cluster barriers
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(db->rank_window_cluster);
            lc.blockDim = dim3(RK_THREADS);
            lc.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = db->rank_window_cluster;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            cudaError_t e = cudaLaunchKernelExC(&lc, (const void*)rank_window_kernel<true>, args);
            if (e != cudaSuccess) return fail(db, GPUTX_ECUDA, std::string("rank cluster launch: ") + cudaGetErrorString(e));
        } else {
            TRY(launch_coop(db, (const void*)rank_window_kernel<false>, db->rank_window_grid, RK_THREADS, args));
        }
        ++db->launches;
    } else if (stream) {
        const uint32_t gs = grid_for(db->max_rec, RS_STREAM_TILE, (uint32_t)db->nsm * 16);   // (all resident)
        rank_stream_tm1_kernel<<<gs, RS_STREAM_THREADS, 0, s>>>(db->d_sorted, db->d_sc + SC_NREC, db->d_D, db->d_sc);
        ++db->launches;
    } else {
        const uint64_t* keys = db->d_sorted;
        const uint32_t* nrec = db->d_sc + SC_NREC;
        uint32_t* D = db->d_D;
        LookBack<Xf> lb = db->lb_rank;
        uint32_t epoch0 = db->rank_epoch + 1;
        GridBar* bar = db->d_bar;
        uint32_t* sc = db->d_sc;
        uint32_t maxp = 1u << 20;
        uint32_t lmax = db->rank_local;
        uint32_t dirty = db->rank_dirty;
        RkMemo memo = db->rank_memo;
        memo.rec_off = db->d_rec_off;
        uint64_t* rtrace = db->trace_rounds ? db->d_rtrace : nullptr;
        if (rtrace) CK(dev_fill(rtrace, 0, RANK_TRACE_SLOTS * 8, s));
        if (db->rank_root) {             // root-local sweeps (TM-1: single-root transactions)
            DevDb vv = v;
            void* rargs[] = {&vv, &keys, &nrec, &D, &bar, &sc, &maxp, &rtrace, &lb, &epoch0, &lmax, &dirty, &memo};
            TRY(launch_coop(db, (const void*)rank_root_kernel<S>, db->rank_root_grid, RK_THREADS, rargs));
        } else {
            void* args[] = {&keys, &nrec, &D, &lb, &epoch0, &bar, &sc, &maxp, &lmax, &dirty, &memo, &rtrace};
            TRY(launch_coop(db, (const void*)rank_kernel, db->rank_grid, RK_THREADS, args));
        }
        ++db->launches;
    }
    const uint32_t g = grid_for(db->n / 4 + 1, 256, 148 * 4);
    depth_reduce_kernel<<<g, 256, 0, s>>>(db->d_D, (uint32_t)db->n, db->d_sc);
    ++db->launches;
    STAGE("rank");
    cudaEventRecord(db->ev[4], s);
    db->has_depth = true;
    return GPUTX_OK;
}

constexpr uint32_t OWN_MAXW = 16384;    // owner warps (executor CTAs x 8)

template <int S, bool DEP>
const void* own_fn() {
    return (const void*)kset_own_exec_kernel<S, kset_pw<S>(), DEP>;
}

// owner-local rounds: TM-1 / TPC-B / micro under the R/W rule, unsharded; the round
// diagnostics (GPUTX_KSET_DIAG bits other than jitter / own-test bits) and round traces
// belong to the global-round executor
template <int S>
bool kset_use_own(const gputx_db* db) {
    if (S == S_TPCC || !db->kset_own || db->has_ts || db->trace_rounds) return false;
    if (db->cfg.flags & GPUTX_FLAG_ADD_RULE) return false;
    if (db->kset_diag & ~(1024u | 8192u | 16384u | 0xFFFF0000u)) return false;
    const bool dep = S == S_TPCB || (db->kset_diag & 16384u);
    return !dep || db->rec_item_sorted;          // the dependency pass walks (item, ts) records
}

template <int S>
gputx_status own_prepare(gputx_db* db) {
    const bool dep = S == S_TPCB || (db->kset_diag & 16384u);
    if (!db->d_oseg) {
        gputx_status st;
        if ((st = dalloc(db, &db->d_oseg, OWN_MAXW + 2)) || (st = dalloc(db, &db->d_prog, OWN_MAXW))) return st;
        if (db->packed && (st = dalloc(db, &db->d_oout, db->max_bulk))) return st;
    }
    if (dep && !db->d_own) {
        gputx_status st;
        if ((st = dalloc(db, &db->d_own, db->max_bulk)) || (st = dalloc(db, &db->d_wait, db->max_bulk)) ||
            (st = dalloc(db, &db->d_pub, db->max_bulk)) || (st = dalloc(db, &db->d_owait, db->max_bulk)))
            return st;
    }
    int& gridv = db->own_grid[dep ? 1 : 0];
    if (!gridv) {
        int per = 0;
        const void* fn = db->own_pipe ? (dep ? (const void*)kset_own_pipe_kernel<S, kset_pw<S>(), true>
                                             : (const void*)kset_own_pipe_kernel<S, kset_pw<S>(), false>)
                                      : (dep ? own_fn<S, true>() : own_fn<S, false>());
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, 256, 0);
        gridv = std::max(1, per) * db->nsm;
        gridv = std::min<int>(gridv, OWN_MAXW / 8);
    }
    uint32_t G = (uint32_t)gridv;
    if (db->exec_grid_override) G = std::min(G, db->exec_grid_override);
    db->own_g = G;
    db->own_nw = G * 8;
    return GPUTX_OK;
}

// (after group_kernel<1, 0, S> wrote the owner keys)
template <int S>
gputx_status kset_own_exec(gputx_db* db, const DevDb& v) {
    cudaStream_t s = db->stream;
    const bool dep = S == S_TPCB || (db->kset_diag & 16384u);
    const uint32_t n = (uint32_t)db->n;
    const uint32_t G = db->own_g, NW = db->own_nw;
    const uint32_t g = grid_for(n, 256, (uint32_t)db->nsm * 8);
    uint64_t* kb = db->d_sorted == db->d_rec_a ? db->d_rec_b : db->d_rec_a;
    uint32_t diag = db->kset_diag;
    if (dep) {
        CK(dev_fill_multi(s, {fseg(db->d_wait, 0, (uint64_t)n * 8), fseg(db->d_pub, 0, n),
                              fseg(db->d_sc + SC_OWNGLOBAL, 0, 4)}));
        own_dep_kernel<<<grid_for(db->max_rec, 256, (uint32_t)db->nsm * 8), 256, 0, s>>>(
            db->d_sorted, db->d_sc + SC_NREC, db->d_own, db->d_D, db->d_wait, db->d_pub, db->d_sc, diag);
        ++db->launches;
    }
    // stable sort on the owner bits: (owner, depth, type) order
    uint64_t* tmp = db->d_sorted == db->d_rec_a ? db->d_rec_a : db->d_rec_b;
    uint64_t* sk = radix_sort_u64(kb, tmp, db->d_sc + SC_NTXN, n, 32, bits_for(NW - 1), db->sort_ws, db->epoch, s);
    db->launches += 2 + (bits_for(NW - 1) + 7) / 8;
    constexpr int PW = kset_pw<S>();
    if (db->own_pipe) {                          // no gather: the executor stages through the perm
        own_bounds_kernel<<<grid_for(n + 1, 256, 148 * 8), 256, 0, s>>>(sk, n, NW, db->d_perm, db->d_D, db->d_oseg,
                                                                    db->d_prog);
        ++db->launches;
        STAGE("own group");
        cudaEventRecord(db->ev[5], s);
        DevDb vv = v;
        const uint32_t* oseg = db->d_oseg;
        const uint64_t* skp = sk;
        const uint32_t* perm = db->d_perm;
        const uint32_t* Dp = db->d_D;
        const unsigned long long* wt = dep ? db->d_wait : nullptr;
        const uint8_t* pb = dep ? db->d_pub : nullptr;
        uint32_t* prog = db->d_prog;
        uint32_t* sc = db->d_sc;
        void* args[] = {&vv, &oseg, &skp, &perm, &Dp, &wt, &pb, &prog, &sc, &diag};
        const void* fn = dep ? (const void*)kset_own_pipe_kernel<S, kset_pw<S>(), true>
                             : (const void*)kset_own_pipe_kernel<S, kset_pw<S>(), false>;
        TRY(launch_coop(db, fn, (int)G, 256, args));
        ++db->launches;
        return GPUTX_OK;
    }
    own_gather_kernel<PW><<<g, 256, 0, s>>>(v, sk, n, NW, db->d_perm, db->d_D, dep ? db->d_wait : nullptr,
                                            dep ? db->d_pub : nullptr, db->d_done, db->d_ptype, db->d_pp, db->d_cnt,
                                            dep ? db->d_owait : nullptr, db->d_oseg, db->d_prog,
                                            db->packed ? db->d_oout : nullptr);
    ++db->launches;
    STAGE("own group");
    cudaEventRecord(db->ev[5], s);
    DevDb vv = v;
    const uint32_t* oseg = db->d_oseg;
    const uint32_t* oidx = db->d_done;
    const uint8_t* otype = db->d_ptype;
    const uint32_t* opp = db->d_pp;
    const uint32_t* odep = db->d_cnt;
    const unsigned long long* wt = db->d_owait;
    const uint32_t* oout = db->packed ? db->d_oout : nullptr;
    uint32_t* prog = db->d_prog;
    uint32_t* sc = db->d_sc;
    void* args[] = {&vv, &oseg, &oidx, &otype, &opp, &odep, &wt, &oout, &prog, &sc, &diag};
    TRY(launch_coop(db, dep ? own_fn<S, true>() : own_fn<S, false>(), (int)G, 256, args));
    ++db->launches;
    return GPUTX_OK;
}

template <int S>
bool kset_use_dataflow(const gputx_db* db) {
    if (S == S_TM1) return false;       // records sorted by item component, not by item
    if (db->kset_df >= 0) return db->kset_df != 0;
    // measured (profiles/round2_kset_dataflow.txt): TPC-C exec 34.1 -> 23.5 ms (its long
    // W_YTD / D_NEXT_O_ID chains with ~125-transaction k-sets); TPC-B rounds 13.9 vs dataflow
    // >= 33.7 ms (1,000 hot branch chains, 3 locks per hop); micro/TM-1: rounds
    return S == S_TPCC;
}

// K-SET part 2: group by (depth, type), then the k-set rounds
// K-SET over spine chains (TPC-B): one thread per chain, no group step (kernels.cuh)
// an upper bound of the spine chains: TPC-B branches; TPC-C warehouses + districts
template <int S>
uint64_t chain_bound(const gputx_db* db) {
    return S == S_TPCB ? db->cfg.dims[0] : (uint64_t)db->cfg.dims[0] * (1 + db->cfg.dims[1]);
}

template <int S>
bool kset_use_chain(const gputx_db* db) {
    // (TPC-C: a warp per chain running whole Payments one after another was slower than the
    // dataflow executor, 18.3 vs 12.8 ms -- its W_YTD chains serialise whole transactions)
    return S == S_TPCB && db->spine_ran && db->kset_own && db->kset_chain && !db->has_ts &&
           !db->trace_rounds && !(db->kset_diag & ~(1u | 8u | 1024u | 0xFFFF0000u)) &&
           chain_bound<S>(db) <= (uint64_t)db->chain_cap;
}

template <int S>
gputx_status kset_chain_exec(gputx_db* db, const DevDb& v) {
    cudaStream_t s = db->stream;
    cudaEventRecord(db->ev[5], s);
    if (++db->chain_epoch == 0) ++db->chain_epoch;
    DevDb vv = v;
    const uint64_t* keys = db->d_sorted;
    const uint32_t* nrec = db->d_sc + SC_NREC;
    const uint32_t* heads = db->d_heads;
    const uint32_t* nh = db->d_sc + SC_NCHAIN;
    const uint32_t* loff = db->d_loff;
    const uint32_t* links = db->d_links;
    const uint8_t* cpub = db->d_cpub;
    uint32_t* done = db->d_cdone;
    uint32_t ep = db->chain_epoch;
    uint32_t* sc = db->d_sc;
    uint32_t diag = db->kset_diag | (db->chain_runs ? 0u : CHAIN_NO_RUNS);
    void* args[] = {&vv, &keys, &nrec, &heads, &nh, &loff, &links, &cpub, &done, &ep, &sc, &diag};
    const int grid = (int)((chain_bound<S>(db) + 3) / 4);           // one chain per warp, 4 per CTA
    TRY(launch_coop(db, (const void*)kset_chain_exec_kernel<S_TPCB>, std::max(1, grid), 128, args));
    ++db->launches;
    db->kset_ran_chain = true;
    db->kset_ran_own = true;
    db->kset_ran_df = false;
    db->has_perm = false;                     // (gputx_read_perm groups on demand)
    return GPUTX_OK;
}

template <int S>
gputx_status kset_exec(gputx_db* db, const DevDb& v) {
    NVTX_SCOPE("gputx.kset.group_exec");
    cudaStream_t s = db->stream;
    const uint32_t T = db->ntypes;
    db->kset_ran_chain = false;
    if (kset_use_chain<S>(db) && db->n) {
        TRY(kset_chain_exec<S>(db, v));
        STAGE("kset exec");
        cudaEventRecord(db->ev[6], s);
        return GPUTX_OK;
    }
    group_zero_kernel<<<148 * 4, 256, 0, s>>>(db->d_gcnt, db->d_sc, T);     // key count + zeroed counters
    ++db->launches;
    const uint32_t gg = grid_for((db->n + GR_TILE - 1) / GR_TILE, 1, 148 * 4);
    const uint32_t P = db->group_p ? std::min(db->group_p, T) : T;
    group_kernel<0, 0><<<gg, 256, 0, s>>>(db->d_D, db->d_type, (uint32_t)db->n, T, db->d_gcnt, nullptr, nullptr,
                                          nullptr, nullptr, nullptr, nullptr, P);
    ++db->launches;
    scan_u32(db, db->d_gcnt, db->d_goff, db->d_sc + SC_NKEYS, db->n * T + 1, nullptr);
    ++db->launches;
    const bool df = kset_use_dataflow<S>(db) && db->d_item_sorted;
    const bool own = !df && kset_use_own<S>(db) && db->n > 0;
    if (own) {      // + the owner keys; the owner gather stages types / parameters itself
        TRY(own_prepare<S>(db));
        const bool dep = S == S_TPCB || (db->kset_diag & 16384u);
        OwnKeys ok{db->own_nw, db->d_sorted == db->d_rec_a ? db->d_rec_b : db->d_rec_a, dep ? db->d_own : nullptr,
                   db->kset_diag, (db->pipe || db->guard) ? db->d_sc + SC_ERR : nullptr};
        group_kernel<1, 0, S><<<gg, 256, 0, s>>>(db->d_D, db->d_type, (uint32_t)db->n, T, db->d_gcnt, db->d_goff,
                                                 db->d_perm, db->d_poff, db->d_pw, nullptr, nullptr, P, ok);
    } else
        group_kernel<1, kset_pw<S>()><<<gg, 256, 0, s>>>(db->d_D, db->d_type, (uint32_t)db->n, T, db->d_gcnt,
                                                         db->d_goff, db->d_perm, db->d_poff, db->d_pw, db->d_ptype,
                                                         db->d_pp, P);
    ++db->launches;
    STAGE("group");
    db->kset_ran_own = own;
    if (own) {
        TRY(kset_own_exec<S>(db, v));
        STAGE("kset exec");
        cudaEventRecord(db->ev[6], s);
        db->has_perm = true;
        return GPUTX_OK;
    }
    cudaEventRecord(db->ev[5], s);
    // K-SET dataflow executor (deep graphs: TPC-B / TPC-C / micro under the R/W rule): the
    // k-sets are executed in k-set order without round barriers -- every transaction waits
    // only until its own predecessors in the T-dependency graph are done, read from per-item
    // completion counters keyed by position in the item's ts-ordered access list (the same
    // keys as TPL, PAPER.md:370-388 / DESIGN.md R-S5); dispatch in perm order makes every
    // wait point to a transaction of smaller depth, already taken by a running lane.
    db->kset_ran_df = df;
    if (df) {
        ++db->epoch;
        tpl_keys_kernel<<<(uint32_t)((db->max_rec + RK_TILE - 1) / RK_TILE) + 1, RK_THREADS, 0, s>>>(
            db->d_item_sorted, db->d_sc + SC_NREC, db->d_rec_off, db->d_lkey, db->d_lock, db->lb_tpl, db->epoch,
            next_ticket(db));
        const bool sh = db->has_ts;
        // per-k-set completion counters (zeroed by the schedule kernel) for the look-ahead throttle
        kset_sched_kernel<<<grid_for(db->n, 256, 148 * 4), 256, 0, s>>>(db->d_goff, T, db->d_sc, 1, db->kset_q,
                                                                         db->d_g, db->d_done);
        DfThrottle thr = db->kset_df_ahead ? DfThrottle{db->d_D, db->d_goff, T, db->kset_df_ahead, db->d_done}
                                           : DfThrottle{};
        if (S == S_TPCC) {
            const uint32_t grid = (uint32_t)((db->n + 3) / 4);
            if (sh) tpl_exec_warp_kernel<true><<<grid, 128, 0, s>>>(v, db->d_rec_off, db->d_lkey, db->d_lock, db->d_sc, db->d_perm, thr);
            else tpl_exec_warp_kernel<false><<<grid, 128, 0, s>>>(v, db->d_rec_off, db->d_lkey, db->d_lock, db->d_sc, db->d_perm, thr);
        } else {
            int per = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tpl_exec_persistent_kernel<S, true>, 256, 0);
            // resident lanes = the look-ahead of the dispatch (GPUTX_KSET_DF_GRID CTAs of 256)
            uint32_t grid = std::min<uint64_t>((uint32_t)std::max(1, per) * (uint32_t)db->nsm, (db->n + 255) / 256);
            if (db->kset_df_grid) grid = std::min(grid, db->kset_df_grid);
            if (sh) tpl_exec_persistent_kernel<S, true><<<grid, 256, 0, s>>>(v, db->d_rec_off, db->d_lkey, db->d_lock, db->d_sc, db->d_perm, thr);
            else tpl_exec_persistent_kernel<S, false><<<grid, 256, 0, s>>>(v, db->d_rec_off, db->d_lkey, db->d_lock, db->d_sc, db->d_perm, thr);
        }
        db->launches += 2;
    }
    // rounds
    if (!df) {
        const uint32_t Gv = (uint32_t)(db->has_ts ? db->kset_grid_ts : db->kset_grid);   // co-resident grid
        uint32_t G = db->exec_grid_override ? std::min(db->exec_grid_override, Gv) : Gv;
        if (db->kset_cluster) G = std::max(db->kset_cluster, G / db->kset_cluster * db->kset_cluster);
        uint32_t* done = db->d_done;
        if (db->kset_diag & 16u) CK(dev_fill(done, 0, db->n * 4, s));
        kset_sched_kernel<<<grid_for(db->n, 256, 148 * 4), 256, 0, s>>>(db->d_goff, T, db->d_sc, G, db->kset_q,
                                                                         db->d_g, (db->kset_diag & 16u) ? nullptr : done);
        ++db->launches;
        DevDb vv = v;
        const uint32_t* perm = db->d_perm;
        const uint32_t* off = db->d_goff;
        const uint16_t* gk = db->d_g;
        const uint32_t* sc = db->d_sc;
        uint32_t TT = T;
        const uint8_t* pt = db->d_ptype;
        const uint32_t* pp = db->d_pp;
        uint64_t* trace = db->trace_rounds ? db->d_trace : nullptr;
        if (trace) CK(dev_fill(trace, 0, (db->n + 1) * 64, s));
        uint32_t diag = db->kset_diag;
        uint32_t C = db->kset_cluster;
        if (diag & 64u) {                 // diagnostics: run on freshly allocated metadata buffers
            static uint16_t* fg = nullptr;
            static uint32_t *fdone = nullptr, *foff = nullptr;
            static uint64_t fcap = 0;
            if (fcap < db->n * T + 2) {
                cudaFree(fg); cudaFree(fdone); cudaFree(foff);
                fcap = db->n * T + 2;
                cudaMalloc(&fg, fcap * 2); cudaMalloc(&fdone, fcap * 4); cudaMalloc(&foff, fcap * 4);
            }
            cudaMemcpyAsync(fg, db->d_g, db->n * 2, cudaMemcpyDeviceToDevice, s);
            dev_fill(fdone, 0, db->n * 4, s);
            cudaMemcpyAsync(foff, db->d_goff, (db->n * T + 1) * 4, cudaMemcpyDeviceToDevice, s);
            gk = fg; done = fdone; off = foff;
        }
        void* args[] = {&vv, &perm, &off, &TT, &gk, &done, &sc, &pt, &pp, &trace, &diag, &C};
        // diag 512: launch WITHOUT the cluster attribute while still passing C (what a
        // profiler replaying the launch does); the kernel must detect it (SC_NOCLUSTER)
        if (C && !(diag & 512u)) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(G);
            lc.blockDim = dim3(kset_block<S>());
            lc.stream = s;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = C;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            at[1].id = cudaLaunchAttributeCooperative;
            at[1].val.cooperative = 1;
            lc.attrs = at;
            lc.numAttrs = 2;
            cudaError_t e = cudaLaunchKernelExC(&lc, kset_fn<S>(db->has_ts), args);
            if (e != cudaSuccess) return fail(db, GPUTX_ECUDA, std::string("cluster launch: ") + cudaGetErrorString(e));
        } else {
            TRY(launch_coop(db, kset_fn<S>(db->has_ts), (int)G, kset_block<S>(), args));
        }
        ++db->launches;
    }
    STAGE("kset exec");
    cudaEventRecord(db->ev[6], s);
    db->has_perm = true;
    return GPUTX_OK;
}

template <int S>
gputx_status run_kset(gputx_db* db, const DevDb& v) {
    TRY(kset_rank<S>(db, v));
    return kset_exec<S>(db, v);
}

// -------------------------------------------------------------------------------- PART
// count_cross = false: GPUTX_AUTO counted c already
template <int S>
gputx_status run_part(gputx_db* db, const DevDb& v, bool count_cross = true) {
    NVTX_SCOPE("gputx.part");
    cudaStream_t s = db->stream;
    cudaEventRecord(db->ev[1], s);
    const uint32_t g = grid_for(db->n, 256, 148 * 16);
    frag_count_kernel<S><<<g, 256, 0, s>>>(v, db->d_cnt);
    ++db->launches;
    if (count_cross) {
        count_gt1_kernel<<<grid_for(db->n, 256, 148 * 4), 256, 0, s>>>(db->d_cnt, (uint32_t)db->n, db->d_sc + SC_CROSS);
        ++db->launches;
    }
    scan_u32(db, db->d_cnt, db->d_rec_off, nullptr, db->n, db->d_sc + SC_NFRAG);
    frag_emit_kernel<S><<<g, 256, 0, s>>>(v, db->d_rec_off, db->d_rec_a);
    ++db->launches;
    cudaEventRecord(db->ev[2], s);
    TRY(sort_records(db, 32, db->part_bits, db->d_sc + SC_NFRAG, db->max_rec));
    cudaEventRecord(db->ev[3], s);
    part_bounds_kernel<<<grid_for(db->max_rec + 1, 256, 148 * 8), 256, 0, s>>>(db->d_sorted, db->d_sc + SC_NFRAG,
                                                                               db->nparts, db->d_part_off);
                                                                               ++db->launches;
    cudaEventRecord(db->ev[4], s);
    cudaEventRecord(db->ev[5], s);
    const uint32_t pb = 128;
    if (S == S_TPCC)
        part_exec_warp_kernel<<<(db->nparts * 32 + pb - 1) / pb, pb, 0, s>>>(v, db->d_sorted, db->d_part_off, db->nparts,
                                                                             db->d_sc);
    else
        part_exec_kernel<S><<<(db->nparts + pb - 1) / pb, pb, 0, s>>>(v, db->d_sorted, db->d_part_off, db->nparts, db->d_sc);
    ++db->launches;
    cudaEventRecord(db->ev[6], s);
    return GPUTX_OK;
}

// --------------------------------------------------------------------------------- TPL
// sorted = true: the access records are already emitted and sorted (GPUTX_AUTO ran the
// K-SET analysis first; TPL's records are the same)
template <int S>
gputx_status run_tpl(gputx_db* db, const DevDb& v, bool sorted = false) {
    NVTX_SCOPE("gputx.tpl");
    cudaStream_t s = db->stream;
    if (!sorted) {
        cudaEventRecord(db->ev[1], s);
        TRY(emit_records<S>(db, v));
        cudaEventRecord(db->ev[2], s);
        TRY(sort_records(db, KEY_ITEM_SHIFT, db->item_bits, db->d_sc + SC_NREC, db->max_rec));
        cudaEventRecord(db->ev[3], s);
    }
    ++db->epoch;
    tpl_keys_kernel<<<(uint32_t)((db->max_rec + RK_TILE - 1) / RK_TILE) + 1, RK_THREADS, 0, s>>>(
        db->d_sorted, db->d_sc + SC_NREC, db->d_rec_off, db->d_lkey, db->d_lock, db->lb_tpl, db->epoch, next_ticket(db));
        ++db->launches;
    cudaEventRecord(db->ev[4], s);
    cudaEventRecord(db->ev[5], s);
    const bool sh = db->has_ts;
    if (db->tpl_persistent) {
        // grid = what is co-resident (every ticket holder must be running)
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, tpl_exec_persistent_kernel<S, true>, 256, 0);
        const uint32_t grid = std::min<uint64_t>((uint32_t)std::max(1, per) * (uint32_t)db->nsm, (db->n + 255) / 256);
        if (sh) tpl_exec_persistent_kernel<S, true><<<grid, 256, 0, s>>>(v, db->d_rec_off, db->d_lkey, db->d_lock, db->d_sc, nullptr, DfThrottle{});
        else tpl_exec_persistent_kernel<S, false><<<grid, 256, 0, s>>>(v, db->d_rec_off, db->d_lkey, db->d_lock, db->d_sc, nullptr, DfThrottle{});
    } else if (S == S_TPCC) {                 // one warp per transaction
        const uint32_t grid = (uint32_t)((db->n + 3) / 4);
        if (sh) tpl_exec_warp_kernel<true><<<grid, 128, 0, s>>>(v, db->d_rec_off, db->d_lkey, db->d_lock, db->d_sc, nullptr, DfThrottle{});
        else tpl_exec_warp_kernel<false><<<grid, 128, 0, s>>>(v, db->d_rec_off, db->d_lkey, db->d_lock, db->d_sc, nullptr, DfThrottle{});
    } else {
        const uint32_t tb = 128, grid = (uint32_t)((db->n + tb - 1) / tb);
        if (sh) tpl_exec_kernel<S, true><<<grid, tb, 0, s>>>(v, db->d_rec_off, db->d_lkey, db->d_lock, db->d_sc);
        else tpl_exec_kernel<S, false><<<grid, tb, 0, s>>>(v, db->d_rec_off, db->d_lkey, db->d_lock, db->d_sc);
    }
    ++db->launches;
    cudaEventRecord(db->ev[6], s);
    return GPUTX_OK;
}

// ------------------------------------------------------------ relaxed-timestamp strategies
// (Appendix G): serializability only; the executed serialization order
// is recorded in d_order (gputx_read_serial_order)
template <int S>
gputx_status run_tpl_relaxed(gputx_db* db, const DevDb& v) {
    cudaStream_t s = db->stream;
    cudaEventRecord(db->ev[1], s);
    CK(dev_fill(db->d_lock, 0, db->n_items * 4, s));          // spin locks free
    for (int k = 2; k < 6; ++k) cudaEventRecord(db->ev[k], s);
    tpl_relaxed_kernel<S><<<(uint32_t)((db->n + 127) / 128), 128, 0, s>>>(v, nullptr, nullptr, db->d_lock,
                                                                          db->d_order, 0, db->d_sc);
    ++db->launches;
    cudaEventRecord(db->ev[6], s);
    db->has_order = true;
    return GPUTX_OK;
}

template <int S>
gputx_status run_part_relaxed(gputx_db* db, const DevDb& v) {
    cudaStream_t s = db->stream;
    const uint32_t g = grid_for(db->n, 256, 148 * 16);
    cudaEventRecord(db->ev[1], s);
    CK(dev_fill(db->d_part_off, 0, ((uint64_t)db->nparts + 1) * 4, s));
    // bulk generation without sort: per-partition counters -> keys, prefix sum -> starts
    rpart_key_kernel<S><<<g, 256, 0, s>>>(v, db->d_part_off, db->d_D, db->d_perm, db->d_cnt, db->d_sc);
    scan_u32(db, db->d_part_off, db->d_part_off, nullptr, db->nparts, db->d_sc + SC_NFRAG);
    rpart_scatter_kernel<<<g, 256, 0, s>>>(db->d_D, db->d_perm, db->d_part_off, (uint32_t)db->n, db->d_rec_off);
    db->launches += 3;
    for (int k = 2; k < 6; ++k) cudaEventRecord(db->ev[k], s);
    const uint32_t pb = 128, np = db->nparts;
    rpart_exec_kernel<S><<<(uint32_t)(((uint64_t)np * (S == S_TPCC ? 32 : 1) + pb - 1) / pb), pb, 0, s>>>(
        v, db->d_rec_off, db->d_part_off, np, db->d_order, db->d_sc);
    // cross-partition transactions afterwards under the basic spin locks;
    // their serialization numbers follow the single-partition ones (base = #single)
    CK(dev_fill(db->d_lock, 0, db->n_items * 4, s));
    TRY(pull_sc(db, s));
    CK(cudaStreamSynchronize(s));
    const uint32_t ncross = db->h_sc[SC_XTOTAL];
    if (ncross)
        tpl_relaxed_kernel<S><<<(ncross + 127) / 128, 128, 0, s>>>(v, db->d_cnt, db->d_sc + SC_XTOTAL, db->d_lock,
                                                                 db->d_order, (uint32_t)db->n - ncross, db->d_sc);
    db->launches += 2;
    cudaEventRecord(db->ev[6], s);
    db->has_order = true;
    return GPUTX_OK;
}

// Algorithm 1 on the bulk's structural parameters
gputx_strategy choose_strategy(const gputx_db* db, uint64_t w0, uint64_t d, uint64_t c) {
    const uint64_t w0_bar = db->ch_w0 ? db->ch_w0 : 64ull * (uint64_t)db->nsm;
    if (w0 >= w0_bar) return GPUTX_KSET;                   // lines 2-3
    if (c <= db->ch_c || d >= db->ch_d) return GPUTX_PART;  // lines 5-8
    return GPUTX_TPL;                                      // line 10
}

template <int S>
gputx_status run_auto(gputx_db* db, const DevDb& v) {
    cudaStream_t s = db->stream;
    cross_count_kernel<S><<<grid_for(db->n, 256, 148 * 8), 256, 0, s>>>(v, db->d_sc + SC_CROSS);
    ++db->launches;
    TRY(kset_rank<S>(db, v));                               // line 1: w0 (and d)
    TRY(pull_sc(db, s));
    CK(cudaStreamSynchronize(s));
    if (db->h_sc[SC_NOCONV]) return fail(db, GPUTX_ECUDA, "rank did not converge");
    const gputx_strategy ch = choose_strategy(db, db->h_sc[SC_ZERO], db->h_sc[SC_MAXD], db->h_sc[SC_CROSS]);
    db->chosen = (int)ch;
    if (ch == GPUTX_KSET) return kset_exec<S>(db, v);
    if (ch == GPUTX_TPL) return run_tpl<S>(db, v, db->rec_item_sorted);
    return run_part<S>(db, v, false);
}

template <int S>
gputx_status execute_schema(gputx_db* db, gputx_strategy st) {
    DevDb v = make_devdb(db);
    if (st == GPUTX_AUTO) return run_auto<S>(db, v);
    if (st == GPUTX_TPL_RELAXED) return run_tpl_relaxed<S>(db, v);
    if (st == GPUTX_PART_RELAXED) return run_part_relaxed<S>(db, v);
    if (st == GPUTX_KSET) return run_kset<S>(db, v);
    if (st == GPUTX_PART) return run_part<S>(db, v);
    return run_tpl<S>(db, v);
}

template <int S>
void launch_ingest(gputx_db* db, uint32_t n_words, const uint32_t* nw_ptr) {
    DevDb v = make_devdb(db);
    const uint32_t g = grid_for(db->n, 256, 148 * 16);
    ingest_kernel<S><<<g, 256, 0, db->stream>>>(v, db->d_pw, n_words, nw_ptr, db->type_mask, db->d_ins_off,
                                                (uint32_t)(db->n + 1), db->d_sc, db->d_xflag,
                                                db->packed ? db->d_out_off : nullptr,
                                                db->rec_at_ingest ? db->d_cnt : nullptr);
                                                ++db->launches;
}

gputx_status submit_check(gputx_db* db, const gputx_bulk* b) {
    if (!db->sealed) return fail(db, GPUTX_ESTATE, "submit before seal");
    if (db->pool_n) return fail(db, GPUTX_ESTATE, "the transaction pool is not empty (gputx_pool_step until drained)");
    if (db->submitted) return fail(db, GPUTX_ESTATE, "a bulk is already submitted");
    if (db->poisoned) return fail(db, GPUTX_ESTATE, "database poisoned by a deadlock; reset first");
    if (b->n > db->max_bulk) return fail(db, GPUTX_ECAPACITY, "bulk larger than max_bulk");
    if (b->n && (!b->type || !b->param_off || !b->param_words)) return GPUTX_EINVAL;
    return GPUTX_OK;
}

// the bulk is in d_type / d_poff / d_pw (/ d_ts, d_src): validate it, resolve the split
// lookups, count insert rows
// pw_src (device, optional): the caller's parameter words, copied here with their count
// read on the device from d_poff[n] (n_words is then ignored)
gputx_status submit_verdict(gputx_db* db);

gputx_status finish_submit(gputx_db* db, uint64_t n, uint32_t n_words, const uint32_t* pw_src = nullptr) {
    cudaStream_t s = db->stream;
    // GPUTX_FLAG_DEFERRED_CHECK (TM-1 / micro, unsharded): no host round trip here; the
    // verdict is taken at execute (include/gputx.h)
    const bool defer = (db->cfg.flags & GPUTX_FLAG_DEFERRED_CHECK) && db->nshards == 1 && !db->has_ts &&
                       (db->schema == S_TM1 || db->schema == S_MICRO);
    db->deferred = defer;
    db->guard = defer;
    db->n = n;
    db->launches = 0;
    db->has_depth = db->has_perm = false;
    db->executed = false;
    CK(dev_fill_multi(s, {fseg(db->d_sc, 0, SC_ERRPK * 4), fseg(db->d_sc + SC_ERRPK, 0xFF, 8),
                              fseg(db->d_sc + SC_ERRPK + 2, 0, (SC_COUNT - SC_ERRPK - 2) * 4)}));
    const bool ins_scan = db->schema == S_TPCC || db->schema == S_TPCB || db->has_ts;
    const int ntab = db->schema == S_TPCC ? 4 : 1;
    if (n) {
        if (ins_scan) CK(dev_fill(db->d_ins_off, 0, 4 * (n + 1) * ntab, s));
        if (db->nshards > 1) CK(dev_fill(db->d_xflag, 0, n, s));
        const uint32_t* nw_ptr = nullptr;
        if (pw_src) {
            nw_ptr = db->d_poff + n;
            n_words = (uint32_t)db->max_words;
            copy_pw_kernel<<<148 * 4, 256, 0, s>>>(pw_src, nw_ptr, db->d_pw, n_words, db->d_sc);
            ++db->launches;
        }
        db->rec_at_ingest = db->nshards == 1;      // (sharded emits count their local records)
        if (db->schema == S_TPCB) launch_ingest<S_TPCB>(db, n_words, nw_ptr);
        else if (db->schema == S_TM1) launch_ingest<S_TM1>(db, n_words, nw_ptr);
        else if (db->schema == S_MICRO) launch_ingest<S_MICRO>(db, n_words, nw_ptr);
        else launch_ingest<S_TPCC>(db, n_words, nw_ptr);
        if (ins_scan && db->schema != S_TM1)
            for (int t = 0; t < ntab; ++t)
                scan_u32(db, db->d_ins_off + t * (n + 1), db->d_ins_off + t * (n + 1), nullptr, n,
                         db->d_sc + SC_INS0 + t);
        if (db->rec_at_ingest && db->packed)
            scan2_u32(db, db->d_out_off, db->d_cnt, db->d_out_off, db->d_rec_off, n, db->d_sc + SC_OUTBYTES,
                      db->d_sc + SC_NREC);
        else if (db->rec_at_ingest)
            scan_u32(db, db->d_cnt, db->d_rec_off, nullptr, n, db->d_sc + SC_NREC);
        else if (db->packed)
            scan_u32(db, db->d_out_off, db->d_out_off, nullptr, n, db->d_sc + SC_OUTBYTES);
    }
    cudaEventRecord(db->ev_sub[1], s);
    if (defer) {
        db->ins_dense = false;
        db->out_bytes = n * db->out_stride;   // (an upper bound until the verdict: zero-fill size)
        for (auto& t : db->ins) t.pending = 0;
        db->submitted = true;
        return GPUTX_OK;
    }
    TRY(pull_sc(db, s));
    CK(cudaStreamSynchronize(s));
    return submit_verdict(db);
}

// the host half of a submit: validation errors, insert-table capacity (h_sc is current)
gputx_status submit_verdict(gputx_db* db) {
    const uint64_t n = db->n;
    if (db->h_sc[SC_ERR]) {
        static const char* what[] = {"", "type id out of range", "type not registered", "wrong parameter count",
                                     "parameter out of range", "bad param_off", "timestamps not increasing",
                                     "home partition not owned by this shard", "too many parameter words"};
        const uint32_t e = err_code(db);
        db->n = 0;
        if (e == E_WORDS) return fail(db, GPUTX_ECAPACITY, "too many parameter words");
        return fail(db, e <= 2 ? GPUTX_EUNKNOWN_TYPE : e == E_OWNER ? GPUTX_ECROSS : GPUTX_EINVAL,
                    std::string("transaction ") + std::to_string(err_idx(db)) + ": " + what[e < 9 ? e : 0]);
    }
    // TPC-B: when every transaction is a home deposit, its history row is its position (no
    // ins_off load on the executors' critical paths, e.g. PART's serial branch chains)
    db->ins_dense = db->schema == S_TPCB && !db->h_sc[SC_SPARSE];
    db->out_bytes = db->packed ? (uint64_t)db->h_sc[SC_OUTBYTES] : n * db->out_stride;
    // insert rows this bulk will append (decisions are static: two-phase procedures)
    for (auto& t : db->ins) {
        t.pending = db->h_sc[SC_INS0 + t.table_id];
        if (t.rows + t.pending > t.cap) {
            db->n = 0;
            return fail(db, GPUTX_ECAPACITY, "insert table " + t.name + " full; reset or raise insert_capacity");
        }
    }
    db->submitted = true;
    return GPUTX_OK;
}

// ---------------------------------------------------------------- streaming K-SET pool
constexpr int SC_POOL_KEPT = SC_CHG0, SC_POOL_WORDS = SC_CHG1;   // (rank slots, unused in pool steps)

gputx_status pool_alloc(gputx_db* db) {
    if (db->pool_ready) return GPUTX_OK;
    const uint64_t NB = db->max_bulk;
    gputx_status st;
    if (!db->s_type &&
        ((st = dalloc(db, &db->s_type, NB + 1)) || (st = dalloc(db, &db->s_poff, NB + 1)) ||
         (st = dalloc(db, &db->s_pw, db->max_words + 16))))
        return st;
    if ((st = dalloc(db, &db->d_prec, db->max_rec + 1)) || (st = dalloc(db, &db->d_prec2, db->max_rec + 1)) ||
        (st = dalloc(db, &db->d_pins, 4 * (NB + 1))) || (st = dalloc(db, &db->q_ins, 4 * (NB + 1))) ||
        (st = dalloc(db, &db->st_ins, 4 * (NB + 1))) || (st = dalloc(db, &db->q_type, NB + 1)) ||
        (st = dalloc(db, &db->q_poff, NB + 1)) || (st = dalloc(db, &db->q_pw, db->max_words + 16)) ||
        (st = dalloc(db, &db->q_ts, NB + 1)) || (st = dalloc(db, &db->d_zflag, NB + 1)) ||
        (st = dalloc(db, &db->d_fna, db->n_items)) || (st = dalloc(db, &db->d_list, NB + 1)) ||
        (st = dalloc(db, &db->d_npos, NB + 2)) || (st = dalloc(db, &db->d_noff, NB + 2)) ||
        (st = dalloc(db, &db->d_rpos, db->max_rec + 2)) || (st = dalloc(db, &db->d_rts, NB + 1)) ||
        (st = dalloc(db, &db->d_rstatus, NB + 1)) || (st = dalloc(db, &db->d_rout, NB * db->out_stride + 16)))
        return st;
    db->pool_ready = true;
    return GPUTX_OK;
}

template <int S>
gputx_status pool_submit_schema(gputx_db* db, uint64_t m, uint32_t words) {
    cudaStream_t s = db->stream;
    const uint32_t ntab = (uint32_t)db->ins.size();
    // 1. ingest the arrivals in the staging area (validation, split lookups, insert counts)
    CK(dev_fill_multi(s, {fseg(db->d_sc, 0, SC_ERRPK * 4), fseg(db->d_sc + SC_ERRPK, 0xFF, 8),
                              fseg(db->d_sc + SC_ERRPK + 2, 0, (SC_COUNT - SC_ERRPK - 2) * 4)}));
    if (ntab) CK(dev_fill(db->st_ins, 0, 4 * (m + 1) * ntab, s));
    DevDb v = make_devdb(db);
    v.n = (uint32_t)m;
    v.type = db->s_type;
    v.poff = db->s_poff;
    v.pw = db->s_pw;
    v.ts = nullptr;
    const uint32_t g = grid_for(m, 256, 148 * 16);
    ingest_kernel<S><<<g, 256, 0, s>>>(v, db->s_pw, words, nullptr, db->type_mask, db->st_ins, (uint32_t)(m + 1),
                                       db->d_sc, nullptr, nullptr, nullptr);
    TRY(pull_sc(db, s));
    CK(cudaStreamSynchronize(s));
    if (db->h_sc[SC_ERR])
        return fail(db, err_code(db) <= 2 ? GPUTX_EUNKNOWN_TYPE : GPUTX_EINVAL,
                    "pool arrival " + std::to_string(err_idx(db)) + " rejected (code " +
                        std::to_string(err_code(db)) + ")");
    // 2. append to the pool with timestamps next_ts + i
    const uint32_t n0 = (uint32_t)db->pool_n;
    pool_append_kernel<<<g, 256, 0, s>>>(db->s_type, db->s_poff, db->s_pw, db->st_ins, (uint32_t)m, n0,
                                         (uint32_t)db->pool_words, (uint32_t)db->next_ts, ntab,
                                         0u, db->d_type, db->d_poff, db->d_pw, db->d_ts,
                                         db->d_pins, (uint32_t)db->max_bulk);
    // 3. the arrivals' access records, sorted by (item, ts), merged into the pool's
    DevDb a = make_devdb(db);
    a.n = (uint32_t)m;
    a.type = db->d_type + n0;
    a.poff = db->d_poff + n0;
    a.idx_base = n0;
    emit_count_kernel<S><<<g, 256, 0, s>>>(a, db->d_cnt);
    scan_u32(db, db->d_cnt, db->d_rec_off, nullptr, m, db->d_sc + SC_NREC);
    emit_write_kernel<S><<<g, 256, 0, s>>>(a, db->d_rec_off, db->d_rec_a);
    const uint64_t* srt = radix_sort_u64(db->d_rec_a, db->d_rec_b, db->d_sc + SC_NREC,
                                         std::min<uint64_t>(db->max_rec, m * MAX_REC), KEY_ITEM_SHIFT, db->item_bits,
                                         db->sort_ws, db->epoch, s);
    const uint64_t tot = db->pool_nrec + std::min<uint64_t>(db->max_rec, m * MAX_REC);
    pool_merge_kernel<<<grid_for(tot, 256, 148 * 8), 256, 0, s>>>(db->d_prec, (uint32_t)db->pool_nrec, srt,
                                                                  db->d_sc + SC_NREC, db->d_prec2);
    std::swap(db->d_prec, db->d_prec2);
    db->launches += 6;
    TRY(pull_sc(db, s));
    CK(cudaStreamSynchronize(s));
    db->pool_nrec += db->h_sc[SC_NREC];
    db->pool_n += m;
    db->pool_words += words;
    return GPUTX_OK;
}

template <int S>
gputx_status pool_step_schema(gputx_db* db, gputx_stats* stats) {
    cudaStream_t s = db->stream;
    const uint64_t n = db->pool_n, nrec = db->pool_nrec;
    const uint32_t ntab = (uint32_t)db->ins.size();
    const uint32_t g = grid_for(std::max(n, nrec), 256, 148 * 16);
    db->launches = 0;
    cudaEventRecord(db->ev[0], s);
    CK(dev_fill(db->d_sc, 0, SC_COUNT * 4, s));
    // 0-set of the pool: one pass of head checks over the sorted records (no rank fixpoint)
    pool_zs_init_kernel<<<g, 256, 0, s>>>(db->d_prec, (uint32_t)nrec, db->d_lock, db->d_fna, db->d_zflag, (uint32_t)n);
    pool_zs_mark_kernel<<<g, 256, 0, s>>>(db->d_prec, (uint32_t)nrec, db->d_lock, db->d_fna);
    pool_zs_check_kernel<<<g, 256, 0, s>>>(db->d_prec, (uint32_t)nrec, db->d_lock, db->d_fna, db->d_zflag);
    scan_u32(db, db->d_zflag, db->d_rec_off, nullptr, n, db->d_sc + SC_XTOTAL);
    pool_list_kernel<<<g, 256, 0, s>>>(db->d_zflag, db->d_rec_off, (uint32_t)n, db->d_list);
    // insert rows of the executed transactions: positions in ts order (appended per step)
    if (ntab) {
        pool_ins_mask_kernel<<<g, 256, 0, s>>>(db->d_zflag, db->d_pins, (uint32_t)n, (uint32_t)db->max_bulk, ntab,
                                              db->d_ins_off);
        for (uint32_t t = 0; t < ntab; ++t)
            scan_u32(db, db->d_ins_off + t * (n + 1), db->d_ins_off + t * (n + 1), nullptr, n, db->d_sc + SC_INS0 + t);
    }
    db->launches += 5;
    cudaEventRecord(db->ev[4], s);
    // one lock-free round (Property 1): the whole 0-set in parallel
    CK(dev_fill(db->d_status, 0, n, s));
    CK(dev_fill(db->d_out, 0, n * db->out_stride, s));
    db->n = n;
    db->has_ts = true;
    db->ins_dense = false;              // pool rows: positions scanned over the executed 0-set
    DevDb v = make_devdb(db);
    pool_exec_kernel<S><<<grid_for(S == S_TPCC ? n * 32 : n, 256, 148 * 8), 256, 0, s>>>(v, db->d_list,
                                                                                       db->d_sc + SC_XTOTAL);
    cudaEventRecord(db->ev[6], s);
    pool_results_kernel<<<g, 256, 0, s>>>(db->d_list, db->d_sc + SC_XTOTAL, db->d_ts, db->d_status, db->d_out,
                                          db->out_stride, db->d_rts, db->d_rstatus, db->d_rout);
    count_aborts_kernel<<<grid_for(n / 4 + 1, 256, 148 * 4), 256, 0, s>>>(db->d_status, (uint32_t)n,
                                                                          db->d_sc + SC_COMMITTED);
    // remove the executed transactions and their records (stable: ts order and the
    // records' (item, ts) order are preserved; record idx renumbered)
    pool_keep_kernel<<<g, 256, 0, s>>>(db->d_zflag, db->d_poff, (uint32_t)n, db->d_cnt, db->d_rpos);
    scan_u32(db, db->d_cnt, db->d_npos, nullptr, n, db->d_sc + SC_POOL_KEPT);
    scan_u32(db, db->d_rpos, db->d_noff, nullptr, n, db->d_sc + SC_POOL_WORDS);
    pool_compact_kernel<<<g, 256, 0, s>>>(db->d_zflag, db->d_npos, db->d_noff, (uint32_t)n, ntab,
                                          (uint32_t)db->max_bulk, db->d_type, db->d_poff, db->d_pw, db->d_ts,
                                          db->d_pins, db->q_type, db->q_poff, db->q_pw, db->q_ts, db->q_ins,
                                          db->d_sc + SC_POOL_KEPT, db->d_sc + SC_POOL_WORDS);
    pool_rec_keep_kernel<<<g, 256, 0, s>>>(db->d_prec, (uint32_t)nrec, db->d_zflag, db->d_cnt);
    scan_u32(db, db->d_cnt, db->d_rpos, nullptr, nrec, db->d_sc + SC_NREC);
    pool_rec_compact_kernel<<<g, 256, 0, s>>>(db->d_prec, (uint32_t)nrec, db->d_cnt, db->d_rpos, db->d_npos,
                                              db->d_prec2);
    db->launches += 10;
    cudaEventRecord(db->ev[7], s);
    TRY(pull_sc(db, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    std::swap(db->d_type, db->q_type);
    std::swap(db->d_poff, db->q_poff);
    std::swap(db->d_pw, db->q_pw);
    std::swap(db->d_ts, db->q_ts);
    std::swap(db->d_pins, db->q_ins);
    std::swap(db->d_prec, db->d_prec2);
    const uint64_t ex = db->h_sc[SC_XTOTAL];
    db->pool_exec = ex;
    if (S == S_TM1 && ex) db->rows_dirty = true;
    db->pool_n = db->h_sc[SC_POOL_KEPT];
    db->pool_words = db->h_sc[SC_POOL_WORDS];
    db->pool_nrec = db->h_sc[SC_NREC];
    for (auto& t : db->ins) t.rows += db->h_sc[SC_INS0 + t.table_id];
    db->executed = false;          // gputx_read_results is for bulks; pool results: gputx_pool_read
    if (stats) {
        memset(stats, 0, sizeof(*stats));
        stats->n = ex;
        stats->zero_set = ex;
        stats->records = nrec;
        stats->aborted = db->h_sc[SC_COMMITTED];
        stats->committed = ex - stats->aborted;
        stats->launches = db->launches;
        stats->strategy = GPUTX_KSET;
        float a = 0, b = 0, c = 0, tot = 0;
        cudaEventElapsedTime(&a, db->ev[0], db->ev[4]);
        cudaEventElapsedTime(&b, db->ev[4], db->ev[6]);
        cudaEventElapsedTime(&c, db->ev[6], db->ev[7]);
        cudaEventElapsedTime(&tot, db->ev[0], db->ev[7]);
        stats->ms_rank = a;       // 0-set extraction (head checks + list + insert positions)
        stats->ms_exec = b;
        stats->ms_merge = c;      // results + compaction of the pool
        stats->ms_total = tot;
    }
    return GPUTX_OK;
}

// TM-1 row groups (schema.cuh): built from the columns, and the columns' mutable fields
// refreshed from them before any read of the database image
gputx_status tm1_rows_pack(gputx_db* db) {
    if (db->schema != S_TM1) return GPUTX_OK;
    const DevDb v = make_devdb(db);
    tm1_pack_kernel<<<grid_for(db->cfg.dims[0], 256, 148 * 8), 256, 0, db->stream>>>(v);
    CK(cudaGetLastError());
    db->rows_dirty = false;
    return GPUTX_OK;
}
gputx_status tm1_rows_sync(gputx_db* db) {
    if (db->schema != S_TM1 || !db->rows_dirty) return GPUTX_OK;
    const DevDb v = make_devdb(db);
    tm1_unpack_kernel<<<grid_for(db->cfg.dims[0], 256, 148 * 8), 256, 0, db->stream>>>(v);
    CK(cudaGetLastError());
    db->rows_dirty = false;
    return GPUTX_OK;
}

Col* find_col(gputx_db* db, const char* name) {
    for (auto& c : db->cols)
        if (!strcmp(c.spec.name, name)) return &c;
    return nullptr;
}

}  // namespace

// =====================================================================================
// C ABI
// =====================================================================================
extern "C" {

uint32_t gputx_out_stride(gputx_schema schema) {
    return schema == GPUTX_TPCB ? 8 : schema == GPUTX_TM1 ? 40 : schema == GPUTX_TPCC ? 200
         : schema == GPUTX_MICRO ? 4 : 0;
}

const char* gputx_last_error(const gputx_db* db) { return db ? db->err.c_str() : "null handle"; }

gputx_status gputx_open_db(const gputx_db_config* cfg, gputx_db** out) {
    if (!out) return GPUTX_EINVAL;
    *out = nullptr;
    if (!cfg) return GPUTX_EINVAL;
    if ((cfg->alloc == nullptr) != (cfg->free == nullptr)) return GPUTX_EINVAL;
    const int schema = (int)cfg->schema;
    if (schema < 1 || schema > 4) return GPUTX_EINVAL;
    if (cfg->max_bulk == 0 || cfg->max_bulk > (1u << 24)) return GPUTX_EINVAL;
    const uint32_t* d = cfg->dims;
    if (schema == S_TPCB && (!d[0] || !d[1] || !d[2])) return GPUTX_EINVAL;
    if (schema == S_TM1 && !d[0]) return GPUTX_EINVAL;
    // micro benchmark: N tuples, 1 <= T <= 32 types, x <= 1000 units of 100 sin calls; unsharded
    if (schema == S_MICRO && (!d[0] || !d[1] || d[1] > MICRO_MAX_TYPES || d[2] > 1000 || cfg->nshards > 1))
        return GPUTX_EINVAL;
    if (schema == S_TPCC && (!d[0] || !d[1] || !d[2] || !d[3])) return GPUTX_EINVAL;
    gputx_db* db = new gputx_db();
    db->cfg = *cfg;
    db->schema = schema;
    db->ntypes = ntypes_of(schema, d);
    db->type_mask = db->ntypes >= 32 ? 0xFFFFFFFFu : (1u << db->ntypes) - 1;
    db->max_bulk = cfg->max_bulk;
    db->out_stride = gputx_out_stride(cfg->schema);
    // PART partition size: PAPER.md:461 tuned 128 on its GPU; on B200 TM-1 runs fastest with
    // one subscriber per partition (maximum parallelism; tools/probe_part_tm1.py: PART total
    // 0.51 ms at 1 vs 3.45 ms at 128 on the 1M/1M NURand bulk), the micro benchmark keeps 128
    db->part_size = cfg->part_size ? cfg->part_size : schema == S_TM1 ? 1 : 128;
    db->nshards = cfg->nshards ? cfg->nshards : 1;
    db->shard = cfg->shard;
    if (db->nshards > MAX_SHARDS || db->shard >= db->nshards) { delete db; return GPUTX_EINVAL; }
    db->packed = (cfg->flags & GPUTX_FLAG_PACKED_OUT) != 0;
    if (db->packed && db->nshards > 1) { delete db; return GPUTX_EINVAL; }   // fixed-stride exchange records
    db->nroot = d[0];                       // branches / subscribers / warehouses
    if (db->nroot < db->nshards) { delete db; return GPUTX_EINVAL; }
    db->root_lo = (uint32_t)(((uint64_t)db->shard * db->nroot + db->nshards - 1) / db->nshards);
    db->root_hi = (uint32_t)(((uint64_t)(db->shard + 1) * db->nroot + db->nshards - 1) / db->nshards);
    auto bail = [&](gputx_status s) { *out = db; gputx_close_db(db); *out = nullptr; return s; };
    if (cudaSetDevice(cfg->device) != cudaSuccess) return bail(GPUTX_ECUDA);
    cudaDeviceGetAttribute(&db->nsm, cudaDevAttrMultiProcessorCount, cfg->device);
    if (cfg->stream) {
        db->stream = (cudaStream_t)cfg->stream;
    } else {
        if (cudaStreamCreateWithFlags(&db->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(GPUTX_ECUDA);
        db->own_stream = true;
    }
    // sizes
    uint64_t n_items = 0, max_words_per = 0, max_rec_per = 0;
    if (schema == S_TPCB) {
        n_items = (uint64_t)d[0] * d[2] + (uint64_t)d[0] * d[1] + d[0];
        max_words_per = 4; max_rec_per = 3;
        db->nparts = d[0];
    } else if (schema == S_TM1) {
        n_items = TM1_STRIDE * d[0];
        max_words_per = 7; max_rec_per = 3;
        db->nparts = (uint32_t)((d[0] + db->part_size - 1) / db->part_size);
    } else if (schema == S_MICRO) {
        n_items = d[0];
        max_words_per = 1; max_rec_per = 1;
        db->nparts = (uint32_t)((d[0] + db->part_size - 1) / db->part_size);
    } else {
        const uint64_t WD = (uint64_t)d[0] * d[1];
        n_items = 2 * WD + d[0] + WD * d[2] + (uint64_t)d[0] * d[3];
        max_words_per = 49; max_rec_per = 16;
        db->nparts = d[0];
    }
    db->n_items = n_items;
    db->item_bits = bits_for(n_items - 1);
    if (db->item_bits > 34) return bail(GPUTX_EINVAL);
    db->part_bits = bits_for(db->nparts ? db->nparts - 1 : 0);
    db->max_words = max_words_per * db->max_bulk;
    db->max_rec = max_rec_per * db->max_bulk;       // records (K-SET/TPL) and fragments (PART) share buffers
    gputx_status st;
    // columns
    for (auto& cs : column_specs(schema, d)) {
        Col c;
        c.spec = cs;
        if ((st = dalloc(db, (uint8_t**)&c.d, cs.count * cs.elem)) != GPUTX_OK) return bail(st);
        dev_fill(c.d, 0, cs.count * cs.elem, db->stream);
        db->cols.push_back(c);
    }
    // insert tables
    for (auto& is : insert_specs(schema)) {
        InsTable t;
        t.name = is.table;
        t.table_id = is.table_id;
        t.per_txn = is.per_txn;
        t.cap = (cfg->insert_capacity ? cfg->insert_capacity : 8) * db->max_bulk * is.per_txn;
        for (auto* cn : is.cols) {
            InsCol ic;
            ic.name = cn;
            if ((st = dalloc(db, (uint32_t**)&ic.d, t.cap)) != GPUTX_OK) return bail(st);
            t.cols.push_back(ic);
        }
        db->ins.push_back(t);
    }
    const uint64_t NB = db->max_bulk;
    const uint64_t cntn = std::max(NB, db->max_rec) + 2;
    if ((st = dalloc(db, &db->d_type, NB)) || (st = dalloc(db, &db->d_poff, NB + 1)) ||
        (st = dalloc(db, &db->d_pw, db->max_words + 16)) || (st = dalloc(db, &db->d_status, NB)) ||
        (st = dalloc(db, &db->d_out, NB * db->out_stride)) || (st = dalloc(db, &db->d_ins_off, 4 * (NB + 1))) ||
        (st = dalloc(db, &db->d_rec_a, db->max_rec)) || (st = dalloc(db, &db->d_rec_b, db->max_rec)) ||
        (st = dalloc(db, &db->d_cnt, cntn)) || (st = dalloc(db, &db->d_rec_off, NB + 2)) ||
        (st = dalloc(db, &db->d_D, NB)) || (st = dalloc(db, &db->d_perm, NB)) ||
        (st = dalloc(db, &db->d_g, NB + 1)) || (st = dalloc(db, &db->d_done, NB + 1)) ||
        (st = dalloc(db, &db->d_ptype, NB)) || (st = dalloc(db, &db->d_pp, NB * 8)) ||
        (st = dalloc(db, &db->d_trace, 8 * (NB + 1))) ||
        (st = dalloc(db, &db->d_gcnt, NB * db->ntypes + 2)) || (st = dalloc(db, &db->d_goff, NB * db->ntypes + 2)) ||
        (st = dalloc(db, &db->d_lock, n_items)) || (st = dalloc(db, &db->d_lkey, db->max_rec)) ||
        (st = dalloc(db, &db->d_part_off, (uint64_t)db->nparts + 2)) || (st = dalloc(db, &db->d_sc, SC_COUNT)) ||
        (st = dalloc(db, &db->d_bar, 1)) || (st = dalloc(db, &db->d_tickets, 256)) ||
        (st = dalloc(db, &db->d_ts, NB + 1)) || (st = dalloc(db, &db->d_order, NB + 1)))
        return bail(st);
    if (schema == S_TPCB && (st = dalloc(db, &db->d_undo, NB * UNDO_SLOTS))) return bail(st);
    if (db->packed && (st = dalloc(db, &db->d_out_off, NB + 1))) return bail(st);
    if (schema == S_TM1) {
        const uint64_t P = d[0];
        if ((st = dalloc(db, &db->tm1_sub, P * TM1_SUBROW)) || (st = dalloc(db, &db->tm1_ai, 4 * P * TM1_AIROW)) ||
            (st = dalloc(db, &db->tm1_sf, 4 * P * TM1_SFROW)) || (st = dalloc(db, &db->tm1_cf, 4 * P * TM1_CFROW)))
            return bail(st);
    }
    if (db->nshards > 1) {             // exchange arena: raw cudaMalloc (IPC-exportable)
        const uint32_t sf = gputx_shard_stride((gputx_schema)schema, 0), sr = gputx_shard_stride((gputx_schema)schema, 1);
        db->fwd_cap = (uint32_t)NB;
        db->ret_cap = (uint32_t)NB;
        db->ret_base = AR_HDR + (uint64_t)db->fwd_cap * sf;
        db->arena_words = db->ret_base + (uint64_t)db->ret_cap * sr;
        if (cudaMalloc((void**)&db->arena, db->arena_words * 4) != cudaSuccess) return bail(GPUTX_ENOMEM);
        dev_fill(db->arena, 0, db->arena_words * 4, db->stream);
        if ((st = dalloc(db, &db->d_done_ctas, 1))) return bail(st);
        dev_fill(db->d_done_ctas, 0, 4, db->stream);
    }
    if (db->nshards > 1 &&
        ((st = dalloc(db, &db->d_src, NB + 1)) || (st = dalloc(db, &db->d_home_pos, NB + 1)) ||
         (st = dalloc(db, &db->d_xflag, NB + 1)) || (st = dalloc(db, &db->s_type, NB + 1)) ||
         (st = dalloc(db, &db->s_poff, NB + 1)) || (st = dalloc(db, &db->s_pw, db->max_words + 16)) ||
         (st = dalloc(db, &db->s_ts, NB + 1)) || (st = dalloc(db, &db->d_hstatus, NB + 1)) ||
         (st = dalloc(db, &db->d_hout, NB * db->out_stride + 16))))
        return bail(st);
    // look-back state: sized for the largest tiled pass
    // (>= 4096 entries: the rank kernel also keeps one aggregate per CTA here)
    const uint64_t tiles = std::max<uint64_t>((std::max(db->max_rec, NB * db->ntypes) + 2) / 2048 + 4, 4096);
    if ((st = dalloc(db, &db->lb_scan2.flag, tiles)) || (st = dalloc(db, &db->lb_scan2.agg, tiles)) ||
        (st = dalloc(db, &db->lb_scan2.inc, tiles)))
        return bail(st);
    dev_fill(db->lb_scan2.flag, 0, tiles * 4, db->stream);
    if ((st = dalloc(db, &db->lb_scan.flag, tiles)) || (st = dalloc(db, &db->lb_scan.agg, tiles)) ||
        (st = dalloc(db, &db->lb_scan.inc, tiles)) || (st = dalloc(db, &db->lb_rank.flag, tiles)) ||
        (st = dalloc(db, &db->lb_rank.agg, tiles)) || (st = dalloc(db, &db->lb_rank.inc, tiles)) ||
        (st = dalloc(db, &db->lb_tpl.flag, tiles)) || (st = dalloc(db, &db->lb_tpl.agg, tiles)) ||
        (st = dalloc(db, &db->lb_tpl.inc, tiles)))
        return bail(st);
    {
        const uint64_t rt = db->max_rec / RK_WT + 2;
        if ((st = dalloc(db, &db->rank_memo.aggA, rt)) || (st = dalloc(db, &db->rank_memo.carD, rt)) ||
            (st = dalloc(db, &db->rank_memo.dirty, rt / 32 + 1)) ||
            (st = dalloc(db, &db->rank_memo.recpos, db->max_rec + 1)) ||
            (st = dalloc(db, &db->d_rtrace, RANK_TRACE_SLOTS)))
            return bail(st);
    }
    db->sort_ws.max_tiles = db->max_rec / (RS_THREADS * 8) + 2;     // sized for the smallest tile
    // keys per thread of a sort tile: 12 for TPC-B's 12 M records (0.70 / 0.60 / 0.65 ms at
    // 8 / 12 / 16) and TPC-C's (0.34 / 0.29 / 0.31 ms), 16 else
    db->sort_ws.items = schema == S_TPCB || schema == S_TPCC ? 12 : RS_ITEMS;
    if (const char* e = getenv("GPUTX_SORT_ITEMS")) db->sort_ws.items = (uint32_t)atoi(e);
    if ((st = dalloc(db, &db->sort_ws.hist, RS_MAXPASS * 256)) ||
        (st = dalloc(db, &db->sort_ws.status, db->sort_ws.max_tiles * 256)) ||
        (st = dalloc(db, &db->sort_ws.tickets, 64)))
        return bail(st);
    dev_fill(db->lb_scan.flag, 0, tiles * 4, db->stream);
    dev_fill(db->lb_rank.flag, 0, tiles * 4, db->stream);
    dev_fill(db->lb_tpl.flag, 0, tiles * 4, db->stream);
    dev_fill(db->sort_ws.status, 0, db->sort_ws.max_tiles * 256 * 8, db->stream);
    dev_fill(db->d_bar, 0, sizeof(GridBar), db->stream);
    dev_fill(db->d_sc, 0, SC_COUNT * 4, db->stream);
    dev_fill(db->d_lock, 0, n_items * 4, db->stream);
    // counters come back through mapped (zero-copy) host memory, written by a kernel: a
    // D2H copy would queue on the copy engine behind a large result transfer of
    // gputx_run_bulks and stall the next bulk's synchronous steps (1.67 vs 1.05 ms / bulk)
    if (cudaHostAlloc((void**)&db->h_sc, SC_COUNT * 4, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&db->h_sc_dev, db->h_sc, 0) != cudaSuccess)
        return bail(GPUTX_ENOMEM);
    for (auto& e : db->ev) cudaEventCreate(&e);
    for (auto& e : db->ev_sub) cudaEventCreate(&e);
    for (auto& e : db->ev_x) cudaEventCreate(&e);
    db->rank_grid = coop_grid(db, rank_kernel, RK_THREADS, 0);
    // sweeps per warp-tile per rank pass, measured per schema (profiles/round1.md):
    // TM-1 / TPC-B chains are mostly root-local (sweeps close them in the tile), TPC-C's cross tiles
    const bool add_rule = (cfg->flags & GPUTX_FLAG_ADD_RULE) != 0;
    // TPC-B with the ADD rule: 1 in-tile sweep (its tiles settle at once; 0.75 -> 0.70 ms)
    db->rank_local = schema == S_TPCC || (schema == S_TPCB && add_rule) ? 1 : 4;
    if (const char* e = getenv("GPUTX_RANK_LOCAL")) db->rank_local = (uint32_t)std::max(1, atoi(e));
    // TPC-C: each pass raises most of the long W_YTD chains' suffix, so nearly every tile is
    // dirty every pass and the marking costs more than it saves (profiles/round1.md)
    db->rank_dirty = schema == S_TPCC ? 0 : 1;
    if (const char* e = getenv("GPUTX_RANK_DIRTY")) db->rank_dirty = (uint32_t)atoi(e);
    // Root-local sweeps where roots are small next to a warp's share of the records: TM-1
    // transactions never cross subscribers (2 passes: settle + confirm; 0.80 -> 0.21 ms),
    // TPC-B crosses branches only through remote accounts (7 -> 4 passes, 2.9 -> 2.1 ms).
    // TPC-C's 64 warehouses are far larger than a warp's share: CTA-range passes instead.
    // (TPC-B with the ADD rule: the grid-wide scan balances better than whole branches
    //  per warp, 0.97 -> 0.70 ms; profiles/round1.md)
    db->rank_root = schema == S_TPCC || (schema == S_TPCB && add_rule) ? 0 : 1;
    if (const char* e = getenv("GPUTX_RANK_ROOT")) db->rank_root = (uint32_t)atoi(e);
    if (const char* e = getenv("GPUTX_RANK_STREAM")) db->rank_stream = (uint32_t)atoi(e);
    if (const char* e = getenv("GPUTX_RANK_SPINE")) db->rank_spine = (uint32_t)atoi(e);
    // TPC-C: 128 k-transaction windows (measured: 2^12 .. 2^17 -> rank 19.6 .. 10.8 ms at
    // 1 M transactions, profiles/round1.md)
    db->rank_window = schema == S_TPCC ? 17 : 0;
    if (const char* e = getenv("GPUTX_RANK_WINDOW")) db->rank_window = (uint32_t)atoi(e);
    db->rank_window_grid = coop_grid(db, rank_window_kernel<false>, RK_THREADS, 0);
    // one 16-CTA cluster with hardware barriers was measured slower than the full
    // cooperative grid with the aggregate reuse (kernels.cuh rank_window_kernel)
    db->rank_window_cluster = 0;
    if (const char* e = getenv("GPUTX_RANK_WCLUSTER")) db->rank_window_cluster = (uint32_t)atoi(e);
    if (db->rank_window_cluster > 8 &&
        cudaFuncSetAttribute(rank_window_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        db->rank_window_cluster = 8;
    if (db->rank_window) {
        gputx_status st2;
        if ((st2 = dalloc(db, &db->d_wseg, (db->max_bulk >> db->rank_window) + 4)) || (st2 = dalloc(db, &db->d_wst, n_items + 1)))
            return bail(st2);
    }
    db->rank_root_grid = schema == S_TPCB ? coop_grid(db, rank_root_kernel<S_TPCB>, RK_THREADS, 0)
                         : schema == S_TM1 ? coop_grid(db, rank_root_kernel<S_TM1>, RK_THREADS, 0)
                         : schema == S_MICRO ? coop_grid(db, rank_root_kernel<S_MICRO>, RK_THREADS, 0)
                                           : coop_grid(db, rank_root_kernel<S_TPCC>, RK_THREADS, 0);
    // a round's memory instructions are spread over ceil(|k-set| / Q) SMs; a TPC-C
    // NewOrder issues ~10x the memory instructions of a TM-1 / TPC-B transaction
    db->kset_q = schema == S_TPCC ? 8 : schema == S_TPCB || schema == S_MICRO ? 32 : 128;   // TPC-C: one warp per txn, 8 warps
    db->kset_cluster = schema == S_TPCB ? 16 : 8;
    if (const char* e = getenv("GPUTX_KSET_Q")) db->kset_q = (uint32_t)std::max(1, atoi(e));
    if (const char* e = getenv("GPUTX_KSET_DIAG")) db->kset_diag = (uint32_t)atoi(e);
    // K-SET runs: rounds of up to runmax transactions run inside CTA 0 (kernels.cuh "Runs")
    if (const char* e = getenv("GPUTX_KSET_RUNMAX")) db->kset_diag = (db->kset_diag & 0xFFFFu) | ((uint32_t)atoi(e) << 16);
    db->sync_stages = getenv("GPUTX_SYNC") != nullptr;
    if (const char* e = getenv("GPUTX_TPL_PERSISTENT")) db->tpl_persistent = atoi(e) != 0;
    if (const char* e = getenv("GPUTX_WATCHDOG_MS")) {   // spin watchdog of every device wait loop
        const unsigned long long ns = (unsigned long long)std::max(1, atoi(e)) * 1000000ull;
        cudaMemcpyToSymbol(g_watchdog_ns, &ns, sizeof(ns));
    }
    if (const char* e = getenv("GPUTX_TPL_SLEEP")) {
        const uint32_t cap = (uint32_t)atoi(e);
        cudaMemcpyToSymbol(g_tpl_sleep_cap, &cap, 4);
    }
    // K-SET executor: thread-block clusters of kset_cluster CTAs (rounds of <= that many
    // CTAs are separated by the hardware cluster barrier); 0 disables clusters
    if (const char* e = getenv("GPUTX_KSET_CLUSTER")) db->kset_cluster = (uint32_t)std::max(0, atoi(e));
    if (const char* e = getenv("GPUTX_KSET_DF")) db->kset_df = atoi(e);
    if (const char* e = getenv("GPUTX_KSET_OWN")) db->kset_own = atoi(e);
    if (const char* e = getenv("GPUTX_KSET_CHAIN")) db->kset_chain = atoi(e);
    if (const char* e = getenv("GPUTX_CHAIN_RUNS")) db->chain_runs = atoi(e);
    if (const char* e = getenv("GPUTX_OWN_PIPE")) db->own_pipe = atoi(e);
    // diag 16384 (tests: arbitrary owners) needs (item, ts)-sorted records for the dependency pass
    if (schema == S_TM1 && (db->kset_diag & 16384u)) db->rank_stream = 0;
    if (const char* e = getenv("GPUTX_KSET_DF_AHEAD")) db->kset_df_ahead = (uint32_t)atoi(e);
    if (const char* e = getenv("GPUTX_KSET_DF_GRID")) db->kset_df_grid = (uint32_t)atoi(e);
    // (sized on the plain variant; the explicit-ts / sharded variant gets the same attributes)
    const void* kfn = schema == S_TPCB ? kset_fn<S_TPCB>(false) : schema == S_TM1 ? kset_fn<S_TM1>(false)
                    : schema == S_MICRO ? kset_fn<S_MICRO>(false)
                                                                                  : kset_fn<S_TPCC>(false);
    const int kblock = schema == S_TPCB ? kset_block<S_TPCB>() : schema == S_TM1 ? kset_block<S_TM1>()
                     : schema == S_MICRO ? kset_block<S_MICRO>()
                                                                                 : kset_block<S_TPCC>();
    {
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kfn, kblock, 0);
        db->kset_grid = std::max(1, per) * db->nsm;
    }
    while (db->kset_cluster) {
        if (db->kset_cluster > 8) {
            const void* kfn_ts = schema == S_TPCB ? kset_fn<S_TPCB>(true) : schema == S_TM1 ? kset_fn<S_TM1>(true)
                    : schema == S_MICRO ? kset_fn<S_MICRO>(true)
                                                                                           : kset_fn<S_TPCC>(true);
            cudaFuncSetAttribute(kfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaFuncSetAttribute(kfn_ts, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        }
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(std::max<uint32_t>(db->kset_cluster, db->kset_grid / db->kset_cluster * db->kset_cluster));
        lc.blockDim = dim3(kblock);
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = db->kset_cluster;
        at.val.clusterDim.y = 1;
        at.val.clusterDim.z = 1;
        lc.attrs = &at;
        lc.numAttrs = 1;
        int nclusters = 0;
        const cudaError_t ce = cudaOccupancyMaxActiveClusters(&nclusters, kfn, &lc);
        if (getenv("GPUTX_DEBUG"))
            fprintf(stderr, "gputx: cluster %u query: %s, %d clusters\n", db->kset_cluster, cudaGetErrorString(ce),
                    nclusters);
        if (ce != cudaSuccess || nclusters < 1) {
            cudaGetLastError();
            db->kset_cluster /= 2;           // try smaller clusters; 1 -> 0: counter hand-offs only
            if (db->kset_cluster < 2) db->kset_cluster = 0;
            continue;
        }
        db->kset_grid = std::min(db->kset_grid, nclusters * (int)db->kset_cluster);
        // the explicit-ts / sharded variant has its own cooperative grid
        const void* kfn_ts = schema == S_TPCB ? kset_fn<S_TPCB>(true) : schema == S_TM1 ? kset_fn<S_TM1>(true)
                    : schema == S_MICRO ? kset_fn<S_MICRO>(true)
                                                                                       : kset_fn<S_TPCC>(true);
        int per_ts = 0, ncl_ts = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_ts, kfn_ts, kblock, 0);
        db->kset_grid_ts = std::max(1, per_ts) * db->nsm;
        if (cudaOccupancyMaxActiveClusters(&ncl_ts, kfn_ts, &lc) == cudaSuccess && ncl_ts >= 1)
            db->kset_grid_ts = std::min(db->kset_grid_ts, ncl_ts * (int)db->kset_cluster);
        db->kset_grid_ts = std::min(db->kset_grid_ts, db->kset_grid);
        cudaGetLastError();
        break;
    }
    if (const char* e = getenv("GPUTX_KSET_GRID")) db->exec_grid_override = (uint32_t)std::min(atoi(e), db->kset_grid);
    if (!db->kset_grid_ts) db->kset_grid_ts = db->kset_grid;
    if (getenv("GPUTX_DEBUG"))
        fprintf(stderr, "gputx: schema %d kset grid %d (ts variant %d) block %d cluster %u Q %u rank grid %d local %u\n",
                schema, db->kset_grid, db->kset_grid_ts, kblock, db->kset_cluster, db->kset_q, db->rank_grid,
                db->rank_local);
    if (cudaStreamSynchronize(db->stream) != cudaSuccess) return bail(GPUTX_ECUDA);
    *out = db;
    return GPUTX_OK;
}

gputx_status gputx_column_info(const gputx_db* db, uint32_t index, const char** name, uint32_t* elem_bytes,
                               uint64_t* count) {
    if (!db || index >= db->cols.size()) return GPUTX_EINVAL;
    if (name) *name = db->cols[index].spec.name;
    if (elem_bytes) *elem_bytes = db->cols[index].spec.elem;
    if (count) *count = db->cols[index].spec.count;
    return GPUTX_OK;
}

gputx_status gputx_load_column(gputx_db* db, const char* name, const void* host, uint64_t bytes) {
    if (!db || !name || !host) return GPUTX_EINVAL;
    if (db->sealed) return fail(db, GPUTX_ESTATE, "load_column after seal");
    Col* c = find_col(db, name);
    if (!c) return fail(db, GPUTX_EINVAL, std::string("unknown column ") + name);
    const uint64_t need = c->spec.count * c->spec.elem;
    if (bytes != need)
        return fail(db, GPUTX_EINVAL, std::string("column ") + name + ": expected " + std::to_string(need) + " bytes");
    CK(cudaMemcpyAsync(c->d, host, bytes, cudaMemcpyHostToDevice, db->stream));
    CK(cudaStreamSynchronize(db->stream));
    c->loaded = true;
    if (!strcmp(name, "sub_nbr")) db->h_nbr.assign((const uint64_t*)host, (const uint64_t*)host + c->spec.count);
    if (!strcmp(name, "c_last")) db->h_last.assign((const uint16_t*)host, (const uint16_t*)host + c->spec.count);
    if (!strcmp(name, "c_first")) db->h_first.assign((const uint64_t*)host, (const uint64_t*)host + c->spec.count);
    return GPUTX_OK;
}

gputx_status gputx_seal(gputx_db* db) {
    if (!db) return GPUTX_EINVAL;
    if (db->sealed) return fail(db, GPUTX_ESTATE, "already sealed");
    gputx_status st;
    if (db->schema == S_TM1) {
        // static sub_nbr -> s_id index (open addressing, load <= 0.5)
        const uint64_t P = db->cfg.dims[0];
        uint64_t cap = 1;
        while (cap < 2 * P) cap <<= 1;
        std::vector<uint64_t> keys(cap, 0);
        std::vector<uint32_t> vals(cap, 0);
        if (db->h_nbr.size() != P) db->h_nbr.assign(P, 0);
        for (uint64_t s = 0; s < P; ++s) {
            const uint64_t k = db->h_nbr[s];
            if (!k) continue;
            uint64_t h = nbr_hash(k) & (cap - 1);
            while (keys[h] != 0 && keys[h] != k) h = (h + 1) & (cap - 1);
            keys[h] = k;
            vals[h] = (uint32_t)(s + 1);
        }
        db->hmask = cap - 1;
        if ((st = dalloc(db, &db->d_hkeys, cap)) || (st = dalloc(db, &db->d_hvals, cap))) return st;
        CK(cudaMemcpyAsync(db->d_hkeys, keys.data(), cap * 8, cudaMemcpyHostToDevice, db->stream));
        CK(cudaMemcpyAsync(db->d_hvals, vals.data(), cap * 4, cudaMemcpyHostToDevice, db->stream));
        CK(cudaStreamSynchronize(db->stream));
        db->h_nbr.clear();
        db->h_nbr.shrink_to_fit();
    }
    if (db->schema == S_TPCC) {
        // static (w, d, c_last) -> customers ordered by (c_first, c)
        const uint64_t W = db->cfg.dims[0], D = db->cfg.dims[1], C = db->cfg.dims[2];
        const uint64_t WD = W * D;
        if (db->h_last.size() != WD * C) db->h_last.assign(WD * C, 0);
        if (db->h_first.size() != WD * C) db->h_first.assign(WD * C, 0);
        std::vector<uint32_t> sorted(WD * C);
        std::vector<uint32_t> off(WD * 1000 + 1, 0);
        std::vector<uint32_t> idx(C);
        for (uint64_t wd = 0; wd < WD; ++wd) {
            const uint64_t b = wd * C;
            for (uint32_t c = 0; c < C; ++c) idx[c] = c;
            std::sort(idx.begin(), idx.end(), [&](uint32_t x, uint32_t y) {
                const uint16_t lx = db->h_last[b + x], ly = db->h_last[b + y];
                if (lx != ly) return lx < ly;
                const uint64_t fx = db->h_first[b + x], fy = db->h_first[b + y];
                if (fx != fy) return fx < fy;
                return x < y;
            });
            uint32_t k = 0;
            for (uint32_t last = 0; last < 1000; ++last) {
                off[wd * 1000 + last] = (uint32_t)(b + k);
                while (k < C && db->h_last[b + idx[k]] == last) { sorted[b + k] = idx[k]; ++k; }
            }
            for (; k < C; ++k) sorted[b + k] = idx[k];     // names >= 1000 (not reachable)
        }
        off[WD * 1000] = (uint32_t)(WD * C);
        if ((st = dalloc(db, &db->d_name_sorted, WD * C)) || (st = dalloc(db, &db->d_name_off, WD * 1000 + 1))) return st;
        CK(cudaMemcpyAsync(db->d_name_sorted, sorted.data(), WD * C * 4, cudaMemcpyHostToDevice, db->stream));
        CK(cudaMemcpyAsync(db->d_name_off, off.data(), (WD * 1000 + 1) * 4, cudaMemcpyHostToDevice, db->stream));
        CK(cudaStreamSynchronize(db->stream));
        db->h_last.clear();
        db->h_first.clear();
    }
    TRY(tm1_rows_pack(db));
    // pristine copy for reset
    for (auto& c : db->cols) {
        const uint64_t b = c.spec.count * c.spec.elem;
        if ((st = dalloc(db, (uint8_t**)&c.pristine, b)) != GPUTX_OK) return st;
        CK(cudaMemcpyAsync(c.pristine, c.d, b, cudaMemcpyDeviceToDevice, db->stream));
    }
    CK(cudaStreamSynchronize(db->stream));
    db->sealed = true;
    return GPUTX_OK;
}

gputx_status gputx_register_types(gputx_db* db, const uint32_t* ids, uint32_t k) {
    if (!db || (k && !ids)) return GPUTX_EINVAL;
    uint32_t mask = 0;
    for (uint32_t j = 0; j < k; ++j) {
        if (ids[j] >= db->ntypes) return fail(db, GPUTX_EUNKNOWN_TYPE, "type " + std::to_string(ids[j]) + " not compiled");
        if (mask & (1u << ids[j])) return fail(db, GPUTX_EDUP_TYPE, "type " + std::to_string(ids[j]) + " listed twice");
        mask |= 1u << ids[j];
    }
    db->type_mask = mask;
    return GPUTX_OK;
}

gputx_status gputx_submit_bulk(gputx_db* db, const gputx_bulk* b, uint64_t* first_ts) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !b) return GPUTX_EINVAL;
    NVTX_SCOPE("gputx.submit");
    if (db->nshards > 1) return fail(db, GPUTX_ESTATE, "sharded handle: submit with gputx_shard_pack + gputx_shard_submit");
    TRY(submit_check(db, b));
    cudaStream_t s = db->stream;
    const uint64_t n = b->n;
    uint32_t n_words = 0;
    if (n && !b->on_device) n_words = b->param_off[n];
    if (n_words > db->max_words) return fail(db, GPUTX_ECAPACITY, "too many parameter words");
    if (!b->ts && db->next_ts + n >= (1ull << 32)) return fail(db, GPUTX_ECAPACITY, "timestamp space exhausted");
    db->has_ts = b->ts != nullptr;
    db->have_x = false;
    cudaEventRecord(db->ev_sub[0], s);
    if (n) {   // (device bulks: ordered on the handle's stream; the words' count is read there)
        const cudaMemcpyKind kind = b->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        if (b->on_device) {
            CK(dev_copy2(db->d_type, b->type, n, db->d_poff, b->param_off, (n + 1) * 4, s));
        } else {
            CK(cudaMemcpyAsync(db->d_type, b->type, n, kind, s));
            CK(cudaMemcpyAsync(db->d_poff, b->param_off, (n + 1) * 4, kind, s));
        }
        if (n_words && !b->on_device) CK(cudaMemcpyAsync(db->d_pw, b->param_words, (uint64_t)n_words * 4, kind, s));
        if (b->ts) CK(cudaMemcpyAsync(db->d_ts, b->ts, n * 4, kind, s));
    }
    db->first_ts = db->next_ts;
    TRY(finish_submit(db, n, n_words, n && b->on_device ? b->param_words : nullptr));
    if (n && b->on_device) ++db->launches;     // (the copy kernel, before finish_submit's reset)
    if (!b->ts) db->next_ts += n;
    if (first_ts) *first_ts = db->first_ts;
    return GPUTX_OK;
}

uint32_t gputx_shard_stride(gputx_schema schema, int result) {
    if (result) return 1 + gputx_out_stride(schema) / 4;
    return schema == GPUTX_TPCB ? 3 + 4 : schema == GPUTX_TM1 ? 3 + 7 : schema == GPUTX_TPCC ? 3 + 49 : 0;
}

gputx_status gputx_shard_pack(gputx_db* db, const gputx_bulk* b, uint32_t* send, uint64_t send_cap, uint64_t* counts) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !b || !counts) return GPUTX_EINVAL;
    if (db->nshards < 2) return fail(db, GPUTX_ESTATE, "not a sharded handle");
    TRY(submit_check(db, b));
    if (b->n && !b->ts) return fail(db, GPUTX_EINVAL, "sharded bulks need global timestamps (gputx_bulk.ts)");
    cudaStream_t s = db->stream;
    const uint64_t n = b->n;
    uint32_t n_words = 0;
    if (n) {
        if (b->on_device) {   // ordered on the handle's stream (the caller's buffers may come from it)
            CK(cudaMemcpyAsync(db->h_sc + SC_COUNT - 1, b->param_off + n, 4, cudaMemcpyDeviceToHost, db->stream));
            CK(cudaStreamSynchronize(db->stream));
            n_words = db->h_sc[SC_COUNT - 1];
        } else {
            n_words = b->param_off[n];
        }
    }
    if (n_words > db->max_words) return fail(db, GPUTX_ECAPACITY, "too many parameter words");
    const uint32_t stride = gputx_shard_stride((gputx_schema)db->schema, 0);
    cudaEventRecord(db->ev_sub[0], s);
    CK(dev_fill(db->d_sc, 0, SC_COUNT * 4, s));
    if (n) {
        const cudaMemcpyKind kind = b->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        CK(cudaMemcpyAsync(db->s_type, b->type, n, kind, s));
        CK(cudaMemcpyAsync(db->s_poff, b->param_off, (n + 1) * 4, kind, s));
        if (n_words) CK(cudaMemcpyAsync(db->s_pw, b->param_words, (uint64_t)n_words * 4, kind, s));
        CK(cudaMemcpyAsync(db->s_ts, b->ts, n * 4, kind, s));
        const DevDb v = make_devdb(db);
        const uint32_t g = grid_for(n, 256, 148 * 8);
        CK(dev_fill(db->d_sc + SC_ERRPK, 0xFF, 8, s));
        shard_validate_kernel<<<g, 256, 0, s>>>(db->s_poff, (uint32_t)n, n_words, stride - 3, db->d_sc);
        if (db->schema == S_TPCB) shard_count_kernel<S_TPCB><<<g, 256, 0, s>>>(v, db->s_type, db->s_poff, db->s_pw, (uint32_t)n, db->d_cnt);
        else if (db->schema == S_TM1) shard_count_kernel<S_TM1><<<g, 256, 0, s>>>(v, db->s_type, db->s_poff, db->s_pw, (uint32_t)n, db->d_cnt);
        else shard_count_kernel<S_TPCC><<<g, 256, 0, s>>>(v, db->s_type, db->s_poff, db->s_pw, (uint32_t)n, db->d_cnt);
        scan_u32(db, db->d_cnt, db->d_rec_off, nullptr, n, db->d_sc + SC_XTOTAL);
        if (db->schema == S_TPCB) shard_pair_kernel<S_TPCB><<<g, 256, 0, s>>>(v, db->s_type, db->s_poff, db->s_pw, (uint32_t)n, db->d_rec_off, db->d_rec_a, db->d_sc);
        else if (db->schema == S_TM1) shard_pair_kernel<S_TM1><<<g, 256, 0, s>>>(v, db->s_type, db->s_poff, db->s_pw, (uint32_t)n, db->d_rec_off, db->d_rec_a, db->d_sc);
        else shard_pair_kernel<S_TPCC><<<g, 256, 0, s>>>(v, db->s_type, db->s_poff, db->s_pw, (uint32_t)n, db->d_rec_off, db->d_rec_a, db->d_sc);
        db->launches += 2;
        const uint64_t* pairs = radix_sort_u64(db->d_rec_a, db->d_rec_b, db->d_sc + SC_XTOTAL,
                                               std::min<uint64_t>(n * (db->nshards - 1), db->max_rec), 32,
                                               bits_for(db->nshards - 1), db->sort_ws, db->epoch, s);
        TRY(pull_sc(db, s));
        CK(cudaStreamSynchronize(s));
        if (db->h_sc[SC_ERR])
            return fail(db, GPUTX_EINVAL, "home transaction " + std::to_string(err_idx(db)) + ": bad param_off");
        const uint64_t np = db->h_sc[SC_XTOTAL];
        for (uint32_t q = 0; q < db->nshards; ++q) counts[q] = db->h_sc[SC_DEST0 + q];
        if (np > send_cap) return fail(db, GPUTX_ECAPACITY, "send buffer holds " + std::to_string(send_cap) +
                                                                 " records, need " + std::to_string(np));
        if (np) {
            if (!send) return GPUTX_EINVAL;
            shard_pack_kernel<<<grid_for(np, 256, 148 * 8), 256, 0, s>>>(pairs, db->d_sc + SC_XTOTAL, db->s_type,
                                                                         db->s_poff, db->s_pw, db->s_ts, stride, send);
            ++db->launches;
            CK(cudaStreamSynchronize(s));      // send is complete on return (the caller moves it)
        }
    } else {
        for (uint32_t q = 0; q < SC_COUNT; ++q) db->h_sc[q] = 0;
    }
    for (uint32_t q = 0; q < db->nshards; ++q) counts[q] = db->h_sc[SC_DEST0 + q];
    db->nh = n;
    db->staged = true;
    return GPUTX_OK;
}

gputx_status gputx_shard_submit(gputx_db* db, const uint32_t* recv, uint64_t n_recv, uint64_t* n_local) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db) return GPUTX_EINVAL;
    if (!db->staged) return fail(db, GPUTX_ESTATE, "gputx_shard_pack first");
    if (n_recv && !recv) return GPUTX_EINVAL;
    const uint64_t n = db->nh + n_recv;
    if (n > db->max_bulk) return fail(db, GPUTX_ECAPACITY, "home + received transactions exceed max_bulk");
    cudaStream_t s = db->stream;
    const uint32_t stride = gputx_shard_stride((gputx_schema)db->schema, 0);
    uint32_t n_words = 0;
    if (n) {
        const uint32_t g = grid_for(n, 256, 148 * 8);
        const uint32_t nh = (uint32_t)db->nh;
        merge_keys_kernel<<<g, 256, 0, s>>>(db->s_ts, nh, recv, (uint32_t)n_recv, stride, db->d_rec_a);
        CK(dev_fill(db->d_sc, 0, SC_COUNT * 4, s));
        uint32_t nn = (uint32_t)n;
        CK(cudaMemcpyAsync(db->d_sc + SC_XTOTAL, &nn, 4, cudaMemcpyHostToDevice, s));
        const uint64_t* keys = radix_sort_u64(db->d_rec_a, db->d_rec_b, db->d_sc + SC_XTOTAL, n, 32, 32, db->sort_ws,
                                              db->epoch, s);
        merge_meta_kernel<<<g, 256, 0, s>>>(keys, nn, nh, db->s_type, db->s_poff, db->s_ts, recv, stride, db->d_type,
                                            db->d_ts, db->d_src, db->d_home_pos, db->d_cnt);
        scan_u32(db, db->d_cnt, db->d_poff, nullptr, n, db->d_sc + SC_XTOTAL);
        merge_params_kernel<<<g, 256, 0, s>>>(keys, nn, nh, db->s_poff, db->s_pw, recv, stride, db->d_poff, db->d_pw,
                                              (uint32_t)db->max_words);
        db->launches += 4 + 4;
        CK(cudaMemcpyAsync(&n_words, db->d_sc + SC_XTOTAL, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (n_words > db->max_words) return fail(db, GPUTX_ECAPACITY, "too many parameter words");
    }
    db->has_ts = true;
    db->staged = false;
    db->returned = false;
    TRY(finish_submit(db, n, n_words));
    if (n_local) *n_local = n;
    return GPUTX_OK;
}

gputx_status gputx_shard_return_pack(gputx_db* db, uint32_t* send, uint64_t send_cap, uint64_t* counts) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !counts) return GPUTX_EINVAL;
    if (db->nshards < 2) return fail(db, GPUTX_ESTATE, "not a sharded handle");
    if (!db->executed) return fail(db, GPUTX_ESTATE, "no executed bulk");
    cudaStream_t s = db->stream;
    const uint32_t ow = db->out_stride / 4;
    CK(dev_fill(db->d_sc + SC_DEST0, 0, MAX_SHARDS * 4, s));
    CK(dev_fill(db->d_sc + SC_XTOTAL, 0, 4, s));
    if (db->n) {
        const uint32_t g = grid_for(db->n, 256, 148 * 8);
        const DevDb v = make_devdb(db);
        ret_count_kernel<<<g, 256, 0, s>>>(db->d_src, (uint32_t)db->n, db->d_cnt);
        scan_u32(db, db->d_cnt, db->d_rec_off, nullptr, db->n, db->d_sc + SC_XTOTAL);
        if (db->schema == S_TPCB) ret_pair_kernel<S_TPCB><<<g, 256, 0, s>>>(v, db->d_rec_off, db->d_rec_a, db->d_sc);
        else if (db->schema == S_TM1) ret_pair_kernel<S_TM1><<<g, 256, 0, s>>>(v, db->d_rec_off, db->d_rec_a, db->d_sc);
        else ret_pair_kernel<S_TPCC><<<g, 256, 0, s>>>(v, db->d_rec_off, db->d_rec_a, db->d_sc);
        const uint64_t* pairs = radix_sort_u64(db->d_rec_a, db->d_rec_b, db->d_sc + SC_XTOTAL, db->n, 32,
                                               bits_for(db->nshards - 1), db->sort_ws, db->epoch, s);
        TRY(pull_sc(db, s));
        CK(cudaStreamSynchronize(s));
        const uint64_t np = db->h_sc[SC_XTOTAL];
        for (uint32_t q = 0; q < db->nshards; ++q) counts[q] = db->h_sc[SC_DEST0 + q];
        if (np > send_cap) return fail(db, GPUTX_ECAPACITY, "send buffer holds " + std::to_string(send_cap) +
                                                                 " records, need " + std::to_string(np));
        if (np) {
            if (!send) return GPUTX_EINVAL;
            ret_pack_kernel<<<grid_for(np, 256, 148 * 8), 256, 0, s>>>(pairs, db->d_sc + SC_XTOTAL, db->d_ts,
                                                                       db->d_out, ow, send);
            CK(cudaStreamSynchronize(s));      // send is complete on return (the caller moves it)
        }
    } else {
        for (uint32_t q = 0; q < SC_COUNT; ++q) db->h_sc[q] = 0;
    }
    for (uint32_t q = 0; q < db->nshards; ++q) counts[q] = db->h_sc[SC_DEST0 + q];
    return GPUTX_OK;
}

// ------------------------------------------------------------- peer-memory exchange (fused)
struct PeerBlob {
    char magic[8];
    uint32_t version, shard, nshards, device;
    uint64_t pid, ptr, words, ret_base;
    uint32_t fwd_cap, ret_cap;
    cudaIpcMemHandle_t h;
};
static_assert(sizeof(PeerBlob) <= GPUTX_PEER_BLOB_BYTES, "blob size");

gputx_status gputx_shard_export(gputx_db* db, void* blob) {
    if (!db || !blob) return GPUTX_EINVAL;
    if (db->nshards < 2 || !db->arena) return fail(db, GPUTX_ESTATE, "not a sharded handle");
    PeerBlob b{};
    memcpy(b.magic, "GPTXPEER", 8);
    b.version = 1;
    b.shard = db->shard;
    b.nshards = db->nshards;
    b.device = (uint32_t)db->cfg.device;
    b.pid = (uint64_t)getpid();
    b.ptr = (uint64_t)(uintptr_t)db->arena;
    b.words = db->arena_words;
    b.ret_base = db->ret_base;
    b.fwd_cap = db->fwd_cap;
    b.ret_cap = db->ret_cap;
    CK(cudaIpcGetMemHandle(&b.h, db->arena));
    memset(blob, 0, GPUTX_PEER_BLOB_BYTES);
    memcpy(blob, &b, sizeof(b));
    return GPUTX_OK;
}

gputx_status gputx_shard_connect(gputx_db* db, const void* blobs) {
    if (!db || !blobs) return GPUTX_EINVAL;
    if (db->nshards < 2 || !db->arena) return fail(db, GPUTX_ESTATE, "not a sharded handle");
    if (db->p2p) return fail(db, GPUTX_ESTATE, "already connected");
    CK(cudaSetDevice(db->cfg.device));
    PeerTable pt{};
    for (uint32_t q = 0; q < db->nshards; ++q) {
        PeerBlob b;
        memcpy(&b, (const uint8_t*)blobs + (uint64_t)q * GPUTX_PEER_BLOB_BYTES, sizeof(b));
        if (memcmp(b.magic, "GPTXPEER", 8) || b.version != 1 || b.shard != q || b.nshards != db->nshards ||
            b.ret_base >= b.words)
            return fail(db, GPUTX_EINVAL, "peer blob " + std::to_string(q) + " does not match this handle");
        pt.ret_base[q] = b.ret_base;
        pt.fwd_cap[q] = b.fwd_cap;
        pt.ret_cap[q] = b.ret_cap;
        if (q == db->shard) {
            pt.arena[q] = db->arena;
        } else if (b.pid == (uint64_t)getpid()) {       // same process: the pointer itself
            if ((int)b.device != db->cfg.device) {
                const cudaError_t e = cudaDeviceEnablePeerAccess((int)b.device, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    return fail(db, GPUTX_ENCCL, std::string("peer access: ") + cudaGetErrorString(e));
                cudaGetLastError();
            }
            pt.arena[q] = (uint32_t*)(uintptr_t)b.ptr;
        } else {                                       // another process: CUDA IPC over NVLink
            void* p = nullptr;
            const cudaError_t e = cudaIpcOpenMemHandle(&p, b.h, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) return fail(db, GPUTX_ENCCL, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
            db->ipc_open.push_back(p);
            pt.arena[q] = (uint32_t*)p;
        }
    }
    db->pt = pt;
    db->p2p = true;
    return GPUTX_OK;
}

gputx_status gputx_shard_connect_local(gputx_db* const* dbs, uint32_t n) {
    if (!dbs || n < 2 || n > MAX_SHARDS) return GPUTX_EINVAL;
    std::vector<uint8_t> blobs((size_t)n * GPUTX_PEER_BLOB_BYTES);
    for (uint32_t q = 0; q < n; ++q) {
        if (!dbs[q] || dbs[q]->shard != q || dbs[q]->nshards != n) return GPUTX_EINVAL;
        TRY(gputx_shard_export(dbs[q], blobs.data() + (size_t)q * GPUTX_PEER_BLOB_BYTES));
    }
    for (uint32_t q = 0; q < n; ++q) TRY(gputx_shard_connect(dbs[q], blobs.data()));
    return GPUTX_OK;
}

extern "C++" {
template <int S>
void p2p_dispatch_launch(gputx_db* db, uint32_t nh) {
    const DevDb v = make_devdb(db);
    const uint32_t g = std::max<uint32_t>(1, grid_for(nh, 256, 148 * 8));
    p2p_dispatch_kernel<S><<<g, 256, 0, db->stream>>>(v, db->s_type, db->s_poff, db->s_pw, db->s_ts, nh, db->pt,
                                                      db->shard, db->nshards,
                                                      gputx_shard_stride((gputx_schema)db->schema, 0), db->xepoch,
                                                      db->d_done_ctas);
    ++db->launches;
}
}  // extern "C++"

gputx_status gputx_shard_dispatch(gputx_db* db, const gputx_bulk* b) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !b) return GPUTX_EINVAL;
    NVTX_SCOPE("gputx.shard_dispatch");
    if (!db->p2p) return fail(db, GPUTX_ESTATE, "gputx_shard_connect first");
    cudaStream_t s = db->stream;
    ++db->xepoch;                      // every shard dispatches once per bulk: epochs agree
    db->have_x = true;
    cudaEventRecord(db->ev_x[0], s);
    cudaEventRecord(db->ev_sub[0], s);
    db->launches = 0;
    gputx_status err = submit_check(db, b);
    if (err == GPUTX_OK && b->n && !b->ts) err = fail(db, GPUTX_EINVAL, "sharded bulks need global timestamps");
    const uint64_t n = err == GPUTX_OK ? b->n : 0;
    uint32_t n_words = 0;
    if (n) {
        if (b->on_device) {
            CK(cudaMemcpyAsync(db->h_sc + SC_COUNT - 1, b->param_off + n, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            n_words = db->h_sc[SC_COUNT - 1];
        } else {
            n_words = b->param_off[n];
        }
        if (n_words > db->max_words) err = fail(db, GPUTX_ECAPACITY, "too many parameter words");
    }
    uint32_t nh = 0;
    if (err == GPUTX_OK && n) {
        const cudaMemcpyKind kind = b->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        CK(cudaMemcpyAsync(db->s_type, b->type, n, kind, s));
        CK(cudaMemcpyAsync(db->s_poff, b->param_off, (n + 1) * 4, kind, s));
        if (n_words) CK(cudaMemcpyAsync(db->s_pw, b->param_words, (uint64_t)n_words * 4, kind, s));
        CK(cudaMemcpyAsync(db->s_ts, b->ts, n * 4, kind, s));
        CK(dev_fill_multi(s, {fseg(db->d_sc, 0, SC_ERRPK * 4), fseg(db->d_sc + SC_ERRPK, 0xFF, 8),
                              fseg(db->d_sc + SC_ERRPK + 2, 0, (SC_COUNT - SC_ERRPK - 2) * 4)}));
        const uint32_t stride = gputx_shard_stride((gputx_schema)db->schema, 0);
        shard_validate_kernel<<<grid_for(n, 256, 148 * 8), 256, 0, s>>>(db->s_poff, (uint32_t)n, n_words, stride - 3,
                                                                        db->d_sc);
        TRY(pull_sc(db, s));
        CK(cudaStreamSynchronize(s));
        if (db->h_sc[SC_ERR]) err = fail(db, GPUTX_EINVAL, "home transaction " + std::to_string(err_idx(db)) +
                                                               ": bad param_off");
        else nh = (uint32_t)n;
    }
    // always publish (an empty contribution on error), so that no peer waits forever
    if (db->schema == S_TPCB) p2p_dispatch_launch<S_TPCB>(db, nh);
    else if (db->schema == S_TM1) p2p_dispatch_launch<S_TM1>(db, nh);
    else p2p_dispatch_launch<S_TPCC>(db, nh);
    CK(cudaGetLastError());
    if (err != GPUTX_OK) return err;
    db->nh = nh;
    db->staged = true;
    return GPUTX_OK;
}

gputx_status gputx_shard_receive(gputx_db* db, uint64_t* n_local) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db) return GPUTX_EINVAL;
    NVTX_SCOPE("gputx.shard_receive");
    if (!db->p2p || !db->staged) return fail(db, GPUTX_ESTATE, "gputx_shard_dispatch first");
    cudaStream_t s = db->stream;
    CK(dev_fill(db->d_sc + SC_DEADLOCK, 0, 4, s));
    p2p_wait_kernel<<<1, 32, 0, s>>>(db->arena, AR_FWD_FLAGS, AR_FWD_CNT, db->shard, db->nshards, db->xepoch,
                                     db->d_sc, db->d_sc + SC_P2P);
    TRY(pull_sc(db, s));
    CK(cudaStreamSynchronize(s));
    if (db->h_sc[SC_DEADLOCK]) {
        db->poisoned = true;
        return fail(db, GPUTX_EDEADLOCK, "a peer shard did not publish its records (watchdog)");
    }
    if (db->h_sc[SC_P2P + 1] & 1u) return fail(db, GPUTX_ECAPACITY, "exchange arena full (forward records)");
    const uint64_t nr = db->h_sc[SC_P2P];
    gputx_status r = gputx_shard_submit(db, db->arena + AR_HDR, nr, n_local);
    // ms_exchange = dispatch .. received records merged and ingested, + return .. collected
    cudaEventRecord(db->ev_x[1], s);
    return r;
}

extern "C++" {
template <int S>
void p2p_return_launch(gputx_db* db) {
    const DevDb v = make_devdb(db);
    const uint32_t g = std::max<uint32_t>(1, grid_for(db->n, 256, 148 * 8));
    p2p_return_kernel<S><<<g, 256, 0, db->stream>>>(v, db->pt, db->shard, db->nshards, db->out_stride / 4,
                                                    db->xepoch, db->d_done_ctas);
    ++db->launches;
}
}  // extern "C++"

gputx_status gputx_shard_return(gputx_db* db) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db) return GPUTX_EINVAL;
    if (!db->p2p) return fail(db, GPUTX_ESTATE, "gputx_shard_connect first");
    if (!db->executed) return fail(db, GPUTX_ESTATE, "no executed bulk");
    cudaEventRecord(db->ev_x[2], db->stream);
    if (db->schema == S_TPCB) p2p_return_launch<S_TPCB>(db);
    else if (db->schema == S_TM1) p2p_return_launch<S_TM1>(db);
    else p2p_return_launch<S_TPCC>(db);
    CK(cudaGetLastError());
    return GPUTX_OK;
}

gputx_status gputx_shard_collect(gputx_db* db) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db) return GPUTX_EINVAL;
    if (!db->p2p || !db->executed) return fail(db, GPUTX_ESTATE, "gputx_shard_return first");
    cudaStream_t s = db->stream;
    p2p_wait_kernel<<<1, 32, 0, s>>>(db->arena, AR_RET_FLAGS, AR_RET_CNT, db->shard, db->nshards, db->xepoch,
                                     db->d_sc, db->d_sc + SC_P2P);
    TRY(pull_sc(db, s));
    CK(cudaStreamSynchronize(s));
    if (db->h_sc[SC_DEADLOCK]) {
        db->poisoned = true;
        return fail(db, GPUTX_EDEADLOCK, "a peer shard did not return its outputs (watchdog)");
    }
    if (db->h_sc[SC_P2P + 1] & 2u) return fail(db, GPUTX_ECAPACITY, "exchange arena full (returned outputs)");
    const uint64_t nr = db->h_sc[SC_P2P];
    TRY(gputx_shard_return_merge(db, db->arena + db->ret_base, nr));
    cudaEventRecord(db->ev_x[3], s);
    return GPUTX_OK;
}

gputx_status gputx_shard_return_merge(gputx_db* db, const uint32_t* recv, uint64_t n_recv) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db) return GPUTX_EINVAL;
    if (db->nshards < 2) return fail(db, GPUTX_ESTATE, "not a sharded handle");
    if (!db->executed) return fail(db, GPUTX_ESTATE, "no executed bulk");
    if (n_recv && !recv) return GPUTX_EINVAL;
    cudaStream_t s = db->stream;
    CK(dev_fill_multi(s, {fseg(db->d_sc, 0, SC_ERRPK * 4), fseg(db->d_sc + SC_ERRPK, 0xFF, 8),
                              fseg(db->d_sc + SC_ERRPK + 2, 0, (SC_COUNT - SC_ERRPK - 2) * 4)}));
    if (n_recv) {
        ret_merge_kernel<<<grid_for(n_recv, 256, 148 * 8), 256, 0, s>>>(recv, (uint32_t)n_recv, db->out_stride / 4,
                                                                         db->d_ts, db->d_src, (uint32_t)db->n,
                                                                         db->d_out, db->d_sc);
    }
    if (db->nh) {
        home_gather_kernel<<<grid_for(db->nh, 256, 148 * 8), 256, 0, s>>>(db->d_home_pos, (uint32_t)db->nh,
                                                                           db->d_status, db->d_out, db->out_stride,
                                                                           db->d_hstatus, db->d_hout);
    }
    TRY(pull_sc(db, s));
    CK(cudaStreamSynchronize(s));
    if (db->h_sc[SC_ERR])
        return fail(db, GPUTX_EINVAL, "returned result " + std::to_string(err_idx(db)) +
                                          " matches no home transaction");
    db->returned = true;
    return GPUTX_OK;
}

// the launch half of gputx_execute / gputx_execute_async: every kernel of the strategy,
// the abort count and the counter pull, enqueued on the handle's stream
gputx_status execute_launch(gputx_db* db, gputx_strategy st) {
    NVTX_SCOPE("gputx.execute");
    if (!db->submitted) return fail(db, GPUTX_ESTATE, "nothing submitted");
    if (st != GPUTX_TPL && st != GPUTX_PART && st != GPUTX_KSET && st != GPUTX_AUTO && st != GPUTX_TPL_RELAXED &&
        st != GPUTX_PART_RELAXED)
        return fail(db, GPUTX_EINVAL, "bad strategy");
    if ((st == GPUTX_TPL_RELAXED || st == GPUTX_PART_RELAXED) && db->nshards > 1)
        return fail(db, GPUTX_EINVAL, "relaxed strategies are single-GPU");
    if (db->deferred) {
        // only K-SET's owner-local path guards every parameter read against a failed ingest;
        // any other execution takes the verdict first (the round trip the flag saves)
        const bool guarded = st == GPUTX_KSET && (db->schema == S_TM1 ? kset_use_own<S_TM1>(db)
                                                                       : kset_use_own<S_MICRO>(db));
        if (!guarded) {
            db->guard = false;
            db->deferred = false;
            TRY(pull_sc(db, db->stream));
            CK(cudaStreamSynchronize(db->stream));
            const gputx_status vs = submit_verdict(db);
            if (vs != GPUTX_OK) {                  // (the failed bulk takes no timestamps)
                db->submitted = false;
                if (!db->has_ts) db->next_ts = db->first_ts;
                return vs;
            }
        }
    }
    db->has_order = false;
    db->chosen = st == GPUTX_AUTO ? (int)GPUTX_KSET : (int)st;   // AUTO: overwritten by run_auto
    cudaStream_t s = db->stream;
    cudaEventRecord(db->ev[0], s);
    const uint64_t n = db->n;
    gputx_status r = GPUTX_OK;
    if (n) {
        // status and (unless TPC-B, whose procedures write every record) the output records, one launch
        const bool zo = db->schema != S_TPCB && !(db->kset_diag & 4096u);
        CK(dev_fill_multi(s, {fseg(db->d_status, 0, n), fseg(db->d_out, 0, zo ? db->out_bytes : 0)}));
        ++db->launches;
        if (db->schema == S_TPCB) r = execute_schema<S_TPCB>(db, st);
        else if (db->schema == S_TM1) r = execute_schema<S_TM1>(db, st);
        else if (db->schema == S_MICRO) r = execute_schema<S_MICRO>(db, st);
        else r = execute_schema<S_TPCC>(db, st);
    } else {
        for (int k = 1; k < 7; ++k) cudaEventRecord(db->ev[k], s);
    }
    cudaEventRecord(db->ev[7], s);
    db->submitted = false;
    if (r != GPUTX_OK) return r;
    if (n) {                                  // (status is 4-byte aligned: cudaMalloc)
        count_aborts_kernel<<<grid_for(n / 4 + 1, 256, 148 * 4), 256, 0, s>>>(db->d_status, (uint32_t)n,
                                                                              db->d_sc + SC_COMMITTED);
        ++db->launches;
    }
    TRY(pull_sc(db, s));
    db->exec_pending = true;
    db->exec_st = (int)st;
    return GPUTX_OK;
}

// the completion half: wait for the stream, device-side errors, stats
gputx_status execute_finish(gputx_db* db, gputx_stats* stats) {
    db->exec_pending = false;
    const gputx_strategy st = (gputx_strategy)db->exec_st;
    cudaStream_t s = db->stream;
    const uint64_t n = db->n;
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    if (db->schema == S_TM1 && n) db->rows_dirty = true;
    if (db->deferred) {                        // the submit's verdict (the bulk ran as empty if it failed)
        db->deferred = false;
        db->guard = false;
        const gputx_status vs = submit_verdict(db);
        db->submitted = false;
        if (vs != GPUTX_OK) {
            db->executed = false;
            if (!db->has_ts) db->next_ts = db->first_ts;   // (the failed bulk takes no timestamps)
            return vs;
        }
        db->out_bytes = db->packed ? (uint64_t)db->h_sc[SC_OUTBYTES] : n * db->out_stride;
    }
    const bool ranked = (st == GPUTX_KSET || st == GPUTX_AUTO) && n;
    const gputx_strategy eff = (gputx_strategy)db->chosen;
    if (ranked) db->rank_epoch += db->h_sc[SC_PASSES] + 1;
    for (auto& t : db->ins) { t.rows += t.pending; t.pending = 0; }
    db->executed = true;
    db->last_strategy = (int)eff;
    if (ranked && db->h_sc[SC_NOCONV]) return fail(db, GPUTX_ECUDA, "rank did not converge");
    if (db->h_sc[SC_DEADLOCK]) {
        db->poisoned = true;
        return fail(db, GPUTX_EDEADLOCK, "spin watchdog tripped (a device wait exceeded GPUTX_WATCHDOG_MS); "
                                         "database poisoned until gputx_reset");
    }
    if (stats) {
        memset(stats, 0, sizeof(*stats));
        stats->n = n;
        stats->launches = db->launches;
        stats->strategy = (uint64_t)eff;
        stats->cross = (eff == GPUTX_PART || st == GPUTX_AUTO) ? db->h_sc[SC_CROSS] : 0;
        stats->records = st == GPUTX_PART ? 0 : db->h_sc[SC_NREC];
        stats->fragments = eff == GPUTX_PART ? db->h_sc[SC_NFRAG] : 0;
        if (ranked) {
            stats->depth = db->h_sc[SC_MAXD];
            stats->ksets = (uint64_t)db->h_sc[SC_MAXD] + 1;
            stats->zero_set = db->h_sc[SC_ZERO];
            stats->rank_passes = db->h_sc[SC_PASSES];
        }
        if (eff == GPUTX_PART || eff == GPUTX_PART_RELAXED) {
            stats->parts = db->nparts;
            stats->max_chain = db->h_sc[SC_MAXCHAIN];
        }
        if (eff == GPUTX_PART_RELAXED) stats->cross = db->h_sc[SC_XTOTAL];
        float ms[8] = {0};
        for (int k = 1; k < 8; ++k) cudaEventElapsedTime(&ms[k], db->ev[k - 1], db->ev[k]);
        stats->ms_emit = ms[2];
        stats->ms_sort = ms[3];
        stats->ms_rank = ms[4];
        stats->ms_group = ms[5];
        stats->ms_exec = ms[6];
        stats->ms_merge = ms[7];
        float tot = 0;
        cudaEventElapsedTime(&tot, db->ev[0], db->ev[7]);
        stats->ms_total = tot;
        const uint64_t ab = n ? db->h_sc[SC_COMMITTED] : 0;    // aborts, counted on the device
        stats->aborted = ab;
        stats->committed = n - ab;
        float mi = 0;
        if (cudaEventElapsedTime(&mi, db->ev_sub[0], db->ev_sub[1]) == cudaSuccess) stats->ms_ingest = mi;
        if (db->have_x) {
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, db->ev_x[0], db->ev_x[1]);
            cudaEventElapsedTime(&b, db->ev_x[2], db->ev_x[3]);
            stats->ms_exchange = a + b;
        }
        stats->out_bytes = db->nshards > 1 ? db->nh * db->out_stride : db->out_bytes;
        stats->flags = (db->h_sc[SC_NOCLUSTER] ? GPUTX_STAT_CLUSTER_FALLBACK : 0) |
                       ((ranked && eff == GPUTX_KSET && db->kset_ran_df) ? GPUTX_STAT_KSET_DATAFLOW : 0) |
                       ((ranked && eff == GPUTX_KSET && db->kset_ran_own) ? GPUTX_STAT_KSET_OWNER : 0) |
                       ((ranked && eff == GPUTX_KSET && db->kset_ran_chain) ? GPUTX_STAT_KSET_CHAIN : 0);
        cudaGetLastError();
    }
    return GPUTX_OK;
}


gputx_status gputx_execute(gputx_db* db, gputx_strategy st, gputx_stats* stats) {
    if (!db) return GPUTX_EINVAL;
    if (db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    TRY(execute_launch(db, st));
    return execute_finish(db, stats);
}

gputx_status gputx_execute_async(gputx_db* db, gputx_strategy st) {
    if (!db) return GPUTX_EINVAL;
    if (db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    return execute_launch(db, st);
}

gputx_status gputx_wait(gputx_db* db, gputx_stats* stats) {
    if (!db) return GPUTX_EINVAL;
    if (!db->exec_pending) return fail(db, GPUTX_ESTATE, "no asynchronous execute pending");
    return execute_finish(db, stats);
}

gputx_status gputx_read_results(gputx_db* db, uint8_t* status, void* out, uint64_t out_bytes) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    const uint8_t* ds = nullptr;
    const void* dout = nullptr;
    uint64_t n = 0;
    TRY(gputx_results_device(db, &ds, &dout, &n));
    const uint64_t need = db->nshards > 1 || !db->packed ? n * db->out_stride : db->out_bytes;
    if (out && out_bytes < need) return fail(db, GPUTX_ECAPACITY, "output buffer too small");
    if (status && n) CK(cudaMemcpyAsync(status, ds, n, cudaMemcpyDeviceToHost, db->stream));
    if (out && n) CK(cudaMemcpyAsync(out, dout, need, cudaMemcpyDeviceToHost, db->stream));
    CK(cudaStreamSynchronize(db->stream));
    return GPUTX_OK;
}

gputx_status gputx_read_out_offsets(gputx_db* db, uint32_t* host, uint64_t n, uint64_t* bytes) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db) return GPUTX_EINVAL;
    if (!db->packed) return fail(db, GPUTX_EINVAL, "fixed-stride outputs (no GPUTX_FLAG_PACKED_OUT)");
    if (!db->submitted && !db->executed) return fail(db, GPUTX_ESTATE, "no submitted bulk");
    if (host && n != db->n + 1) return fail(db, GPUTX_EINVAL, "offsets are u32[n + 1]");
    if (host) CK(cudaMemcpy(host, db->d_out_off, (db->n + 1) * 4, cudaMemcpyDeviceToHost));
    if (bytes) *bytes = db->out_bytes;
    return GPUTX_OK;
}

gputx_status gputx_results_device(gputx_db* db, const uint8_t** status, const void** out, uint64_t* n) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db) return GPUTX_EINVAL;
    if (!db->executed) return fail(db, GPUTX_ESTATE, "no executed bulk");
    if (db->nshards > 1) {
        if (!db->returned) return fail(db, GPUTX_ESTATE, "sharded: gputx_shard_return_merge first");
        if (status) *status = db->d_hstatus;
        if (out) *out = db->d_hout;
        if (n) *n = db->nh;
        return GPUTX_OK;
    }
    if (status) *status = db->d_status;
    if (out) *out = db->d_out;
    if (n) *n = db->n;
    return GPUTX_OK;
}

gputx_status gputx_read_column(gputx_db* db, const char* name, void* host, uint64_t bytes) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !name || !host) return GPUTX_EINVAL;
    TRY(tm1_rows_sync(db));
    Col* c = find_col(db, name);
    if (!c) return fail(db, GPUTX_EINVAL, std::string("unknown column ") + name);
    if (bytes != c->spec.count * c->spec.elem) return fail(db, GPUTX_EINVAL, "size mismatch");
    CK(cudaMemcpyAsync(host, c->d, bytes, cudaMemcpyDeviceToHost, db->stream));
    CK(cudaStreamSynchronize(db->stream));
    return GPUTX_OK;
}

gputx_status gputx_insert_rows(gputx_db* db, const char* table, uint64_t* rows) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !table || !rows) return GPUTX_EINVAL;
    for (auto& t : db->ins)
        if (t.name == table) { *rows = t.rows; return GPUTX_OK; }
    return fail(db, GPUTX_EINVAL, std::string("unknown table ") + table);
}

gputx_status gputx_read_insert_column(gputx_db* db, const char* table, const char* column, void* host, uint64_t bytes) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !table || !column) return GPUTX_EINVAL;
    for (auto& t : db->ins) {
        if (t.name != table) continue;
        for (auto& c : t.cols) {
            if (c.name != column) continue;
            if (bytes != t.rows * 4) return fail(db, GPUTX_EINVAL, "size mismatch");
            if (bytes) {
                CK(cudaMemcpyAsync(host, c.d, bytes, cudaMemcpyDeviceToHost, db->stream));
                CK(cudaStreamSynchronize(db->stream));
            }
            return GPUTX_OK;
        }
    }
    return fail(db, GPUTX_EINVAL, std::string("unknown insert column ") + table + "." + column);
}

gputx_status gputx_read_depths(gputx_db* db, uint32_t* host, uint64_t n) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !host) return GPUTX_EINVAL;
    if (!db->has_depth || n != db->n) return fail(db, GPUTX_ESTATE, "no K-SET depths for this bulk");
    if (n) CK(cudaMemcpy(host, db->d_D, n * 4, cudaMemcpyDeviceToHost));
    return GPUTX_OK;
}

gputx_status gputx_read_round_ns(gputx_db* db, uint64_t* host, uint64_t rounds) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !host) return GPUTX_EINVAL;
    if (!db->trace_rounds || !db->has_perm) return fail(db, GPUTX_ESTATE, "round tracing off or no K-SET bulk");
    if (rounds > db->n) return fail(db, GPUTX_EINVAL, "more rounds than transactions");
    if (rounds) CK(cudaMemcpy(host, db->d_trace, rounds * 8 * 8, cudaMemcpyDeviceToHost));
    return GPUTX_OK;
}

gputx_status gputx_read_rank_ns(gputx_db* db, uint64_t* host, uint64_t passes) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !host) return GPUTX_EINVAL;
    if (!db->trace_rounds || !db->has_depth) return fail(db, GPUTX_ESTATE, "tracing off or no K-SET bulk");
    if (passes > RANK_TRACE_SLOTS / 8) return fail(db, GPUTX_EINVAL, "too many passes");
    if (passes) CK(cudaMemcpy(host, db->d_rtrace, passes * 64, cudaMemcpyDeviceToHost));
    return GPUTX_OK;
}

gputx_status gputx_trace_rounds(gputx_db* db, int on) {
    if (!db) return GPUTX_EINVAL;
    db->trace_rounds = on != 0;
    return GPUTX_OK;
}

gputx_status gputx_read_perm(gputx_db* db, uint32_t* host, uint64_t n) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !host) return GPUTX_EINVAL;
    if (db->has_depth && !db->has_perm && db->executed && n == db->n && n) {
        // the chain executor needs no (depth, type) order: group it on demand
        cudaStream_t s = db->stream;
        const uint32_t T = db->ntypes;
        const uint32_t P = db->group_p ? std::min(db->group_p, T) : T;
        const uint32_t gg = grid_for((db->n + GR_TILE - 1) / GR_TILE, 1, 148 * 4);
        group_zero_kernel<<<148 * 4, 256, 0, s>>>(db->d_gcnt, db->d_sc, T);
        group_kernel<0, 0><<<gg, 256, 0, s>>>(db->d_D, db->d_type, (uint32_t)db->n, T, db->d_gcnt, nullptr, nullptr,
                                              nullptr, nullptr, nullptr, nullptr, P);
        scan_u32(db, db->d_gcnt, db->d_goff, db->d_sc + SC_NKEYS, db->n * T + 1, nullptr);
        group_kernel<1, 0><<<gg, 256, 0, s>>>(db->d_D, db->d_type, (uint32_t)db->n, T, db->d_gcnt, db->d_goff,
                                              db->d_perm, nullptr, nullptr, nullptr, nullptr, P);
        CK(cudaStreamSynchronize(s));
        db->has_perm = true;
    }
    if (!db->has_perm || n != db->n) return fail(db, GPUTX_ESTATE, "no K-SET order for this bulk");
    if (n) CK(cudaMemcpy(host, db->d_perm, n * 4, cudaMemcpyDeviceToHost));
    return GPUTX_OK;
}

gputx_status gputx_pool_submit(gputx_db* db, const gputx_bulk* b, uint64_t* first_ts) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !b) return GPUTX_EINVAL;
    if (!db->sealed) return fail(db, GPUTX_ESTATE, "pool submit before seal");
    if (db->packed) return fail(db, GPUTX_EINVAL, "the transaction pool returns fixed-stride outputs");
    if (db->submitted) return fail(db, GPUTX_ESTATE, "a bulk is submitted; execute it first");
    if (db->poisoned) return fail(db, GPUTX_ESTATE, "database poisoned by a deadlock; reset first");
    if (db->nshards > 1) return fail(db, GPUTX_ESTATE, "the pool is single-GPU (unsharded handles)");
    if (b->ts) return fail(db, GPUTX_EINVAL, "pool arrivals take ts = next_ts + i (gputx_bulk.ts must be NULL)");
    const uint64_t m = b->n;
    if (db->pool_n + m > db->max_bulk) return fail(db, GPUTX_ECAPACITY, "pool would exceed max_bulk");
    if (m && (!b->type || !b->param_off || !b->param_words)) return GPUTX_EINVAL;
    if (db->next_ts + m >= (1ull << 24)) return fail(db, GPUTX_ECAPACITY, "timestamp space (24 bits) exhausted; reset");
    TRY(pool_alloc(db));
    if (first_ts) *first_ts = db->next_ts;
    if (!m) return GPUTX_OK;
    cudaStream_t s = db->stream;
    uint32_t words = 0;
    if (b->on_device) {
        CK(cudaMemcpyAsync(db->h_sc + SC_COUNT - 1, b->param_off + m, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        words = db->h_sc[SC_COUNT - 1];
    } else {
        words = b->param_off[m];
    }
    if (db->pool_words + words > db->max_words) return fail(db, GPUTX_ECAPACITY, "pool parameter words exceed capacity");
    const cudaMemcpyKind kind = b->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpyAsync(db->s_type, b->type, m, kind, s));
    CK(cudaMemcpyAsync(db->s_poff, b->param_off, (m + 1) * 4, kind, s));
    if (words) CK(cudaMemcpyAsync(db->s_pw, b->param_words, (uint64_t)words * 4, kind, s));
    gputx_status r;
    if (db->schema == S_TPCB) r = pool_submit_schema<S_TPCB>(db, m, words);
    else if (db->schema == S_TM1) r = pool_submit_schema<S_TM1>(db, m, words);
    else if (db->schema == S_MICRO) r = pool_submit_schema<S_MICRO>(db, m, words);
    else r = pool_submit_schema<S_TPCC>(db, m, words);
    if (r == GPUTX_OK) db->next_ts += m;
    return r;
}

gputx_status gputx_pool_step(gputx_db* db, gputx_stats* stats, uint64_t* executed) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db) return GPUTX_EINVAL;
    NVTX_SCOPE("gputx.pool_step");
    if (db->submitted) return fail(db, GPUTX_ESTATE, "a bulk is submitted; execute it first");
    if (db->poisoned) return fail(db, GPUTX_ESTATE, "database poisoned by a deadlock; reset first");
    if (!db->pool_n) {
        db->pool_exec = 0;
        if (executed) *executed = 0;
        if (stats) memset(stats, 0, sizeof(*stats));
        return GPUTX_OK;
    }
    gputx_status r;
    if (db->schema == S_TPCB) r = pool_step_schema<S_TPCB>(db, stats);
    else if (db->schema == S_TM1) r = pool_step_schema<S_TM1>(db, stats);
    else if (db->schema == S_MICRO) r = pool_step_schema<S_MICRO>(db, stats);
    else r = pool_step_schema<S_TPCC>(db, stats);
    if (r == GPUTX_OK && executed) *executed = db->pool_exec;
    return r;
}

gputx_status gputx_pool_read(gputx_db* db, uint32_t* ts, uint8_t* status, void* out, uint64_t cap, uint64_t* n) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db) return GPUTX_EINVAL;
    const uint64_t k = db->pool_exec;
    if (n) *n = k;
    if (k > cap) return fail(db, GPUTX_ECAPACITY, "result buffers hold fewer than the step's transactions");
    cudaStream_t s = db->stream;
    if (k && ts) CK(cudaMemcpyAsync(ts, db->d_rts, k * 4, cudaMemcpyDeviceToHost, s));
    if (k && status) CK(cudaMemcpyAsync(status, db->d_rstatus, k, cudaMemcpyDeviceToHost, s));
    if (k && out) CK(cudaMemcpyAsync(out, db->d_rout, k * db->out_stride, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return GPUTX_OK;
}

// Snapshot: the whole current database in one host buffer.
//   "GPTXSNAP" u32 version=1 u32 schema u32 dims[4] u32 ncols u32 ntables
//   per column : u32 name_len, name, u32 elem_bytes, u64 count, count*elem bytes
//   per table  : u32 name_len, name, u32 ncols, u64 rows, per column: u32 name_len, name, rows*4 bytes
gputx_status gputx_snapshot(gputx_db* db, void* buf, uint64_t* bytes) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !bytes) return GPUTX_EINVAL;
    if (!db->sealed) return fail(db, GPUTX_ESTATE, "snapshot before seal");
    uint64_t need = 8 + 4 * 8;
    for (auto& c : db->cols) need += 4 + strlen(c.spec.name) + 4 + 8 + c.spec.count * c.spec.elem;
    for (auto& t : db->ins) {
        need += 4 + t.name.size() + 4 + 8;
        for (auto& c : t.cols) need += 4 + c.name.size() + t.rows * 4;
    }
    if (!buf) { *bytes = need; return GPUTX_OK; }
    if (*bytes < need) { *bytes = need; return fail(db, GPUTX_ECAPACITY, "snapshot buffer too small"); }
    TRY(tm1_rows_sync(db));
    uint8_t* o = (uint8_t*)buf;
    auto put = [&](const void* p, uint64_t k) { memcpy(o, p, k); o += k; };
    auto u32 = [&](uint32_t v) { put(&v, 4); };
    auto u64 = [&](uint64_t v) { put(&v, 8); };
    put("GPTXSNAP", 8);
    u32(1);
    u32((uint32_t)db->schema);
    for (int k = 0; k < 4; ++k) u32(db->cfg.dims[k]);
    u32((uint32_t)db->cols.size());
    u32((uint32_t)db->ins.size());
    for (auto& c : db->cols) {
        u32((uint32_t)strlen(c.spec.name));
        put(c.spec.name, strlen(c.spec.name));
        u32(c.spec.elem);
        u64(c.spec.count);
        CK(cudaMemcpyAsync(o, c.d, c.spec.count * c.spec.elem, cudaMemcpyDeviceToHost, db->stream));
        o += c.spec.count * c.spec.elem;
    }
    for (auto& t : db->ins) {
        u32((uint32_t)t.name.size());
        put(t.name.data(), t.name.size());
        u32((uint32_t)t.cols.size());
        u64(t.rows);
        for (auto& c : t.cols) {
            u32((uint32_t)c.name.size());
            put(c.name.data(), c.name.size());
            if (t.rows) CK(cudaMemcpyAsync(o, c.d, t.rows * 4, cudaMemcpyDeviceToHost, db->stream));
            o += t.rows * 4;
        }
    }
    CK(cudaStreamSynchronize(db->stream));
    *bytes = need;
    return GPUTX_OK;
}

// ------------------------------------------------------------------ overlapped bulk stream
gputx_status pipe_alloc(gputx_db* db) {
    if (db->st_h2d) return GPUTX_OK;
    CK(cudaStreamCreateWithFlags(&db->st_h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&db->st_d2h, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        for (cudaEvent_t* e : {&db->ev_in[k], &db->ev_in_free[k], &db->ev_res[k], &db->ev_res_free[k]})
            CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        gputx_status st;
        if ((st = dalloc(db, &db->in_type[k], db->max_bulk + 1)) || (st = dalloc(db, &db->in_poff[k], db->max_bulk + 1)) ||
            (st = dalloc(db, &db->in_pw[k], db->max_words + 16)) || (st = dalloc(db, &db->res_status[k], db->max_bulk + 1)) ||
            (st = dalloc(db, &db->res_out[k], db->max_bulk * db->out_stride + 16)))
            return st;
        CK(cudaEventRecord(db->ev_in_free[k], db->stream));
        CK(cudaEventRecord(db->ev_res_free[k], db->stream));
    }
    return GPUTX_OK;
}

// bytes of a host bulk's output records (GPUTX_FLAG_PACKED_OUT sizes, include/gputx.h)
// for the schemas without parameter-dependent sizes
uint64_t host_out_bytes(const gputx_db* db, const uint8_t* type, uint64_t n) {
    if (!db->packed) return n * db->out_stride;
    if (db->schema == S_MICRO) return 4 * n;
    if (db->schema == S_TPCB) return 8 * n;
    // TM-1: GSD 40, GND 32, GAD 16, the rest 0 -- the type bytes counted 16 at a time (SSE2
    // compare + movemask + popcount: the host enqueues the next bulk while this one runs)
    uint64_t c0 = 0, c1 = 0, c2 = 0, i = 0;
    const __m128i z0 = _mm_setzero_si128(), z1 = _mm_set1_epi8(1), z2 = _mm_set1_epi8(2);
    for (; i + 16 <= n; i += 16) {
        const __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i*>(type + i));
        c0 += __builtin_popcount(_mm_movemask_epi8(_mm_cmpeq_epi8(v, z0)));
        c1 += __builtin_popcount(_mm_movemask_epi8(_mm_cmpeq_epi8(v, z1)));
        c2 += __builtin_popcount(_mm_movemask_epi8(_mm_cmpeq_epi8(v, z2)));
    }
    for (; i < n; ++i) { c0 += type[i] == 0; c1 += type[i] == 1; c2 += type[i] == 2; }
    return 40 * c0 + 32 * c1 + 16 * c2;
}

// Pipelined gputx_run_bulks (TM-1 / micro, K-SET with owner-local rounds): every bulk's
// submit and execute are enqueued without a host round trip.  Ingest errors cannot be
// returned before the execute is enqueued, so the kernels that read parameters treat a
// bulk whose ingest flagged an error as empty (DevDb.err) and the run's poison word makes
// every later bulk fail at ingest; the counters of bulk i land in mapped host slot i and
// are checked after the one synchronisation at the end (the first failing bulk's error is
// returned, as in the synchronous loop).  Per-bulk stats carry counts, not phase times.
gputx_status run_bulks_pipe(gputx_db* db, const gputx_bulk* bulks, uint64_t k, uint8_t* const* status,
                            void* const* out, gputx_stats* stats) {
    cudaStream_t s = db->stream;
    if (db->slots_cap < k) {
        if (db->h_slots) cudaFreeHost(db->h_slots);
        db->h_slots = nullptr;
        db->slots_cap = 0;
        const uint64_t cap = std::max<uint64_t>(k, 64);
        if (cudaHostAlloc((void**)&db->h_slots, cap * SC_COUNT * 4, cudaHostAllocMapped | cudaHostAllocPortable) !=
                cudaSuccess ||
            cudaHostGetDevicePointer((void**)&db->h_slots_dev, db->h_slots, 0) != cudaSuccess)
            return fail(db, GPUTX_ENOMEM, "run_bulks counter slots");
        db->slots_cap = cap;
    }
    if (!db->d_poison) TRY(dalloc(db, &db->d_poison, 1));
    CK(dev_fill(db->d_poison, 0, 4, s));
    std::vector<uint64_t> nb(k), ob(k), fts(k);
    auto h2d = [&](uint64_t i) -> gputx_status {
        const gputx_bulk& b = bulks[i];
        const int sl = (int)(i & 1);
        CK(cudaStreamWaitEvent(db->st_h2d, db->ev_in_free[sl], 0));
        if (b.n) {
            CK(cudaMemcpyAsync(db->in_type[sl], b.type, b.n, cudaMemcpyHostToDevice, db->st_h2d));
            CK(cudaMemcpyAsync(db->in_poff[sl], b.param_off, (b.n + 1) * 4, cudaMemcpyHostToDevice, db->st_h2d));
            const uint64_t w = b.param_off[b.n];
            if (w) CK(cudaMemcpyAsync(db->in_pw[sl], b.param_words, w * 4, cudaMemcpyHostToDevice, db->st_h2d));
        }
        CK(cudaEventRecord(db->ev_in[sl], db->st_h2d));
        return GPUTX_OK;
    };
    // GPUTX_PIPE_TRACE: per bulk, event times (ms from the first) of H2D end, exec start,
    // exec end and D2H end, printed after the run
    static const bool ptrace = getenv("GPUTX_PIPE_TRACE") != nullptr;
    std::vector<cudaEvent_t> pev;
    auto pmark = [&](cudaStream_t st_) {
        if (!ptrace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st_);
        pev.push_back(e);
    };
    if (ptrace) pmark(s);
    gputx_status hst = GPUTX_OK;               // a host-detected error stops enqueueing
    uint64_t done = 0;
    int last = 0;
    db->pipe = true;
    if (k) hst = h2d(0);
    for (uint64_t i = 0; i < k && hst == GPUTX_OK; ++i) {
        const int sl = (int)(i & 1);
        last = sl;
        if (i + 1 < k && (hst = h2d(i + 1)) != GPUTX_OK) break;
        if ((hst = submit_check(db, &bulks[i])) != GPUTX_OK) break;
        CK(cudaStreamWaitEvent(s, db->ev_in[sl], 0));
        CK(cudaStreamWaitEvent(s, db->ev_res_free[sl], 0));
        std::swap(db->d_type, db->in_type[sl]);
        std::swap(db->d_poff, db->in_poff[sl]);
        std::swap(db->d_pw, db->in_pw[sl]);
        std::swap(db->d_status, db->res_status[sl]);
        std::swap(db->d_out, db->res_out[sl]);
        CK(cudaEventRecord(db->ev_in_free[sl], s));
        pmark(s);                              // exec start (its inputs and result slot ready)
        const uint64_t n = bulks[i].n;
        const uint32_t words = n ? bulks[i].param_off[n] : 0;
        // submit without the round trip (finish_submit's device half)
        db->has_ts = false;
        db->first_ts = db->next_ts;
        fts[i] = db->first_ts;
        db->n = n;
        db->launches = 0;
        db->has_depth = db->has_perm = false;
        db->executed = false;
        CK(dev_fill_multi(s, {fseg(db->d_sc, 0, SC_ERRPK * 4), fseg(db->d_sc + SC_ERRPK, 0xFF, 8),
                              fseg(db->d_sc + SC_ERRPK + 2, 0, (SC_COUNT - SC_ERRPK - 2) * 4)}));
        // (records counted by emit: its failed-bulk guard zeroes them and sets the poison word)
        db->rec_at_ingest = false;
        if (n) {
            if (db->schema == S_TM1) launch_ingest<S_TM1>(db, words, nullptr);
            else launch_ingest<S_MICRO>(db, words, nullptr);
            if (db->packed) scan_u32(db, db->d_out_off, db->d_out_off, nullptr, n, db->d_sc + SC_OUTBYTES);
        }
        db->ins_dense = false;
        db->out_bytes = host_out_bytes(db, bulks[i].type, n);
        db->submitted = true;
        db->next_ts += n;
        db->pull_target = db->h_slots_dev + i * SC_COUNT;
        hst = execute_launch(db, GPUTX_KSET);
        db->exec_pending = false;
        db->pull_target = nullptr;
        if (hst != GPUTX_OK) break;
        nb[i] = n;
        ob[i] = db->out_bytes;
        done = i + 1;
        CK(cudaEventRecord(db->ev_res[sl], s));
        pmark(s);                              // exec end
        CK(cudaStreamWaitEvent(db->st_d2h, db->ev_res[sl], 0));
        if (n && status && status[i]) CK(cudaMemcpyAsync(status[i], db->d_status, n, cudaMemcpyDeviceToHost, db->st_d2h));
        if (n && out && out[i] && db->out_bytes)
            CK(cudaMemcpyAsync(out[i], db->d_out, db->out_bytes, cudaMemcpyDeviceToHost, db->st_d2h));
        CK(cudaEventRecord(db->ev_res_free[sl], db->st_d2h));
        pmark(db->st_d2h);                     // D2H end
        std::swap(db->d_status, db->res_status[sl]);
        std::swap(db->d_out, db->res_out[sl]);
    }
    db->pipe = false;
    db->pull_target = nullptr;
    for (int sl = 0; sl < 2; ++sl) CK(cudaStreamWaitEvent(s, db->ev_res_free[sl], 0));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    if (ptrace) {                              // rows: exec start, exec end, D2H end per bulk
        for (size_t j = 1; j < pev.size(); ++j) {
            float ms = 0;
            cudaEventElapsedTime(&ms, pev[0], pev[j]);
            fprintf(stderr, "%s%.3f", (j - 1) % 3 == 0 ? "\n[pipe] " : " ", ms);
            cudaEventDestroy(pev[j]);
        }
        fprintf(stderr, "\n");
        if (!pev.empty()) cudaEventDestroy(pev[0]);
    }
    if (done) {                                // gputx_read_results: the last bulk's results
        std::swap(db->d_status, db->res_status[last]);
        std::swap(db->d_out, db->res_out[last]);
    }
    if (done && db->schema == S_TM1) db->rows_dirty = true;   // (the row groups changed)
    // the bulks' counters, in order: the first failing bulk stops the run
    for (uint64_t i = 0; i < done; ++i) {
        const uint32_t* h = db->h_slots + i * SC_COUNT;
        db->rank_epoch += h[SC_PASSES] + 1;
        if (h[SC_ERR]) {
            static const char* what[] = {"", "type id out of range", "type not registered", "wrong parameter count",
                                         "parameter out of range", "bad param_off", "timestamps not increasing",
                                         "home partition not owned by this shard", "too many parameter words",
                                         "an earlier bulk of the run failed"};
            const uint64_t pk = (uint64_t)h[SC_ERRPK] | ((uint64_t)h[SC_ERRPK + 1] << 32);
            const uint32_t e = (uint32_t)(pk & 0xFF), bad = (uint32_t)(pk >> 8);
            db->n = 0;
            db->submitted = false;
            db->executed = false;
            db->next_ts = fts[i];              // the failed bulk and the ones after it take no ts
            return fail(db, e <= 2 ? GPUTX_EUNKNOWN_TYPE : GPUTX_EINVAL,
                        "bulk " + std::to_string(i) + ", transaction " + std::to_string(bad) + ": " +
                            what[e <= 9 ? e : 0]);
        }
        if (h[SC_DEADLOCK]) {
            db->poisoned = true;
            return fail(db, GPUTX_EDEADLOCK, "spin watchdog tripped (bulk " + std::to_string(i) + ")");
        }
        if (stats) {
            gputx_stats& st = stats[i];
            memset(&st, 0, sizeof(st));
            st.n = nb[i];
            st.strategy = GPUTX_KSET;
            st.records = h[SC_NREC];
            st.depth = h[SC_MAXD];
            st.ksets = (uint64_t)h[SC_MAXD] + 1;
            st.zero_set = h[SC_ZERO];
            st.rank_passes = h[SC_PASSES];
            st.aborted = nb[i] ? h[SC_COMMITTED] : 0;
            st.committed = nb[i] - st.aborted;
            st.out_bytes = ob[i];
            st.flags = GPUTX_STAT_KSET_OWNER | GPUTX_STAT_PIPELINED;
        }
    }
    if (done) {
        db->executed = true;
        db->last_strategy = (int)GPUTX_KSET;
        if (db->schema == S_TM1) db->rows_dirty = true;
    }
    return hst;
}

gputx_status gputx_run_bulks(gputx_db* db, const gputx_bulk* bulks, uint64_t k, gputx_strategy st,
                             uint8_t* const* status, void* const* out, gputx_stats* stats) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || (k && !bulks)) return GPUTX_EINVAL;
    if (db->nshards > 1) return fail(db, GPUTX_ESTATE, "sharded handles: use the shard calls");
    for (uint64_t i = 0; i < k; ++i) {
        if (bulks[i].on_device || bulks[i].ts) return fail(db, GPUTX_EINVAL, "run_bulks takes host bulks without ts");
        if (bulks[i].n > db->max_bulk) return fail(db, GPUTX_ECAPACITY, "bulk larger than max_bulk");
        if (bulks[i].n && (!bulks[i].type || !bulks[i].param_off || !bulks[i].param_words)) return GPUTX_EINVAL;
        if (bulks[i].n && bulks[i].param_off[bulks[i].n] > db->max_words)
            return fail(db, GPUTX_ECAPACITY, "too many parameter words");
    }
    TRY(pipe_alloc(db));
    // the pipelined loop: TM-1 / micro K-SET (owner-local rounds; no inserts, no host-side
    // decisions between ingest and execute); GPUTX_PIPE=0 keeps the synchronous loop
    static const bool pipe_env = !getenv("GPUTX_PIPE") || atoi(getenv("GPUTX_PIPE")) != 0;
    if (pipe_env && st == GPUTX_KSET && k &&
        ((db->schema == S_TM1 && kset_use_own<S_TM1>(db)) || (db->schema == S_MICRO && kset_use_own<S_MICRO>(db))))
        return run_bulks_pipe(db, bulks, k, status, out, stats);
    cudaStream_t s = db->stream;
    // No device-to-device copies on the way (they would queue behind the other copy stream's
    // transfer on the copy engines): each slot's input buffers are SWAPPED in as the engine's
    // bulk buffers, and its result buffers swapped in for the next bulk's results.
    auto h2d = [&](uint64_t i) -> gputx_status {
        const gputx_bulk& b = bulks[i];
        const int sl = (int)(i & 1);
        CK(cudaStreamWaitEvent(db->st_h2d, db->ev_in_free[sl], 0));
        if (b.n) {
            CK(cudaMemcpyAsync(db->in_type[sl], b.type, b.n, cudaMemcpyHostToDevice, db->st_h2d));
            CK(cudaMemcpyAsync(db->in_poff[sl], b.param_off, (b.n + 1) * 4, cudaMemcpyHostToDevice, db->st_h2d));
            const uint64_t w = b.param_off[b.n];
            if (w) CK(cudaMemcpyAsync(db->in_pw[sl], b.param_words, w * 4, cudaMemcpyHostToDevice, db->st_h2d));
        }
        CK(cudaEventRecord(db->ev_in[sl], db->st_h2d));
        return GPUTX_OK;
    };
    if (k) TRY(h2d(0));
    int last = 0;
    static const bool ptrace = getenv("GPUTX_PIPE_TRACE") != nullptr;
    std::vector<cudaEvent_t> pev;
    auto pmark = [&](cudaStream_t st_) {
        if (!ptrace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st_);
        pev.push_back(e);
    };
    for (uint64_t i = 0; i < k; ++i) {
        const int sl = (int)(i & 1);
        last = sl;
        if (i + 1 < k) TRY(h2d(i + 1));              // next bulk's copy overlaps this one's execution
        TRY(submit_check(db, &bulks[i]));
        pmark(s);
        CK(cudaStreamWaitEvent(s, db->ev_in[sl], 0));       // bulk i has landed in slot sl
        CK(cudaStreamWaitEvent(s, db->ev_res_free[sl], 0)); // bulk i-2's results left slot sl
        std::swap(db->d_type, db->in_type[sl]);
        std::swap(db->d_poff, db->in_poff[sl]);
        std::swap(db->d_pw, db->in_pw[sl]);
        std::swap(db->d_status, db->res_status[sl]);
        std::swap(db->d_out, db->res_out[sl]);
        // the buffers now in slot sl held bulk i-1 (already executed): free for bulk i+1's copy
        CK(cudaEventRecord(db->ev_in_free[sl], s));
        const uint64_t n = bulks[i].n;
        db->has_ts = false;
        db->first_ts = db->next_ts;
        TRY(finish_submit(db, n, n ? bulks[i].param_off[n] : 0));
        db->next_ts += n;
        pmark(s);
        TRY(gputx_execute(db, st, stats ? &stats[i] : nullptr));
        pmark(s);
        // results stay in the engine's d_status / d_out until the next bulk swaps them out; the
        // D2H reads them from there on its own stream, overlapping the next execution
        CK(cudaEventRecord(db->ev_res[sl], s));
        CK(cudaStreamWaitEvent(db->st_d2h, db->ev_res[sl], 0));
        pmark(db->st_d2h);
        if (n && status && status[i]) CK(cudaMemcpyAsync(status[i], db->d_status, n, cudaMemcpyDeviceToHost, db->st_d2h));
        if (n && out && out[i])
            CK(cudaMemcpyAsync(out[i], db->d_out, db->out_bytes, cudaMemcpyDeviceToHost, db->st_d2h));
        CK(cudaEventRecord(db->ev_res_free[sl], db->st_d2h));
        pmark(db->st_d2h);
        // the next bulk gets the other slot's result buffers (swap below) -- these stay put
        std::swap(db->d_status, db->res_status[sl]);
        std::swap(db->d_out, db->res_out[sl]);
    }
    // the handle's stream is ordered after the last result copy (an event recorded on it
    // after this call covers the whole run), then wait for it
    for (int sl = 0; sl < 2; ++sl) CK(cudaStreamWaitEvent(s, db->ev_res_free[sl], 0));
    CK(cudaStreamSynchronize(s));
    if (ptrace) {
        for (size_t j = 0; j < pev.size(); ++j) {
            float ms = 0;
            cudaEventElapsedTime(&ms, pev[0], pev[j]);
            fprintf(stderr, "%s%s%.3f", j % 5 == 0 ? "\n[pipe] " : " ", j % 5 == 0 ? "" : "", ms);
        }
        fprintf(stderr, "\n[pipe] columns: pre-wait, exec-start, exec-end, d2h-start, d2h-end\n");
        for (auto e : pev) cudaEventDestroy(e);
    }
    if (k) {                                   // gputx_read_results: the last bulk's results
        std::swap(db->d_status, db->res_status[last]);
        std::swap(db->d_out, db->res_out[last]);
    }
    return GPUTX_OK;
}

gputx_status gputx_read_serial_order(gputx_db* db, uint32_t* host, uint64_t n) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db || !host) return GPUTX_EINVAL;
    if (n == 0 && db->n == 0) return GPUTX_OK;                    // an empty bulk: the empty order
    if (!db->has_order || n != db->n) return fail(db, GPUTX_ESTATE, "no relaxed-strategy execution of this bulk");
    if (n) CK(cudaMemcpy(host, db->d_order, n * 4, cudaMemcpyDeviceToHost));
    return GPUTX_OK;
}

gputx_status gputx_pool_pending(const gputx_db* db, uint64_t* n) {
    if (!db || !n) return GPUTX_EINVAL;
    *n = db->pool_n;
    return GPUTX_OK;
}

gputx_status gputx_set_grouping(gputx_db* db, uint32_t p) {
    if (!db) return GPUTX_EINVAL;
    if (p > db->ntypes) return fail(db, GPUTX_EINVAL, "more type groups than types");
    db->group_p = p;
    return GPUTX_OK;
}

gputx_status gputx_set_chooser(gputx_db* db, uint64_t w0_bar, uint64_t d_bar, uint64_t c_bar) {
    if (!db) return GPUTX_EINVAL;
    db->ch_w0 = w0_bar;
    db->ch_d = d_bar;
    db->ch_c = c_bar;
    return GPUTX_OK;
}

gputx_status gputx_reset(gputx_db* db) {
    if (db && db->exec_pending) return fail(db, GPUTX_ESTATE, "an asynchronous execute is pending: gputx_wait first");
    if (!db) return GPUTX_EINVAL;
    if (!db->sealed) return fail(db, GPUTX_ESTATE, "reset before seal");
    for (auto& c : db->cols)
        CK(cudaMemcpyAsync(c.d, c.pristine, c.spec.count * c.spec.elem, cudaMemcpyDeviceToDevice, db->stream));
    for (auto& t : db->ins) { t.rows = 0; t.pending = 0; }
    TRY(tm1_rows_pack(db));
    CK(cudaStreamSynchronize(db->stream));
    db->poisoned = false;
    db->submitted = false;
    db->executed = false;
    db->deferred = db->guard = false;
    db->next_ts = 0;
    db->pool_n = db->pool_words = db->pool_nrec = db->pool_exec = 0;
    return GPUTX_OK;
}

gputx_status gputx_set_launch(gputx_db* db, uint32_t exec_block, uint32_t exec_grid, uint32_t narrow_max) {
    if (!db) return GPUTX_EINVAL;
    if (exec_grid && (int)exec_grid > db->kset_grid) return fail(db, GPUTX_EINVAL, "grid exceeds co-resident CTAs");
    (void)exec_block;
    (void)narrow_max;
    db->exec_grid_override = exec_grid;
    return GPUTX_OK;
}

void gputx_close_db(gputx_db* db) {
    if (!db) return;
    if (db->stream) cudaStreamSynchronize(db->stream);
    for (auto& c : db->cols) { dfree(db, c.d); dfree(db, c.pristine); }
    for (auto& t : db->ins)
        for (auto& c : t.cols) dfree(db, c.d);
    void* ps[] = {db->d_type, db->d_poff, db->d_pw, db->d_status, db->d_out, db->d_ins_off, db->d_hkeys, db->d_hvals,
                  db->d_name_sorted, db->d_name_off, db->d_rec_a, db->d_rec_b, db->d_cnt, db->d_rec_off, db->d_D,
                  db->d_perm, db->d_g, db->d_done, db->d_ptype, db->d_pp, db->d_trace, db->d_gcnt, db->d_goff, db->d_lock, db->d_lkey, db->d_part_off, db->d_sc, db->d_bar,
                  db->d_tickets, db->lb_scan.flag, db->lb_scan.agg, db->lb_scan.inc, db->lb_rank.flag,
                  db->lb_rank.agg, db->lb_rank.inc, db->lb_tpl.flag, db->lb_tpl.agg, db->lb_tpl.inc,
                  db->sort_ws.hist, db->sort_ws.status, db->sort_ws.tickets, db->rank_memo.aggA,
                  db->rank_memo.carD, db->rank_memo.dirty, db->rank_memo.recpos, db->d_rtrace, db->d_ts,
                  db->d_src, db->d_home_pos, db->d_xflag, db->s_type, db->s_poff, db->s_pw, db->s_ts,
                  db->d_hstatus, db->d_hout, db->d_wseg, db->d_wst};
    for (void* p : ps) dfree(db, p);
    dfree(db, db->d_order);
    dfree(db, db->tm1_sub); dfree(db, db->tm1_ai); dfree(db, db->tm1_sf); dfree(db, db->tm1_cf);
    dfree(db, db->d_undo);
    dfree(db, db->d_out_off);
    dfree(db, db->lb_scan2.flag); dfree(db, db->lb_scan2.agg); dfree(db, db->lb_scan2.inc);
    dfree(db, db->d_lastw); dfree(db, db->d_sp); dfree(db, db->d_lcnt); dfree(db, db->d_loff); dfree(db, db->d_lfill);
    dfree(db, db->d_links); dfree(db, db->d_heads); dfree(db, db->d_ccur); dfree(db, db->d_clast);
    dfree(db, db->d_cpub); dfree(db, db->d_cdone);
    dfree(db, db->lb_seg.flag); dfree(db, db->lb_seg.agg); dfree(db, db->lb_seg.inc);
    dfree(db, db->d_oseg); dfree(db, db->d_prog); dfree(db, db->d_oout); dfree(db, db->d_own); dfree(db, db->d_wait); dfree(db, db->d_pub); dfree(db, db->d_owait);
    void* pp[] = {db->d_prec, db->d_prec2, db->d_pins, db->q_ins, db->st_ins, db->q_type, db->q_poff, db->q_pw,
                  db->q_ts, db->d_zflag, db->d_fna, db->d_list, db->d_npos, db->d_noff, db->d_rpos, db->d_rts,
                  db->d_rstatus, db->d_rout};
    for (void* p : pp) dfree(db, p);          // (pool staging s_* is in ps above)
    if (db->h_sc) cudaFreeHost(db->h_sc);
    if (db->h_slots) cudaFreeHost(db->h_slots);
    dfree(db, db->d_poison);
    for (auto& e : db->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : db->ev_sub)
        if (e) cudaEventDestroy(e);
    for (auto& e : db->ev_x)
        if (e) cudaEventDestroy(e);
    for (int k = 0; k < 2; ++k) {
        for (cudaEvent_t e : {db->ev_in[k], db->ev_in_free[k], db->ev_res[k], db->ev_res_free[k]})
            if (e) cudaEventDestroy(e);
        dfree(db, db->in_type[k]); dfree(db, db->in_poff[k]); dfree(db, db->in_pw[k]);
        dfree(db, db->res_status[k]); dfree(db, db->res_out[k]);
    }
    if (db->st_h2d) cudaStreamDestroy(db->st_h2d);
    for (void* p : db->ipc_open) cudaIpcCloseMemHandle(p);
    if (db->arena) cudaFree(db->arena);
    dfree(db, db->d_done_ctas);
    if (db->st_d2h) cudaStreamDestroy(db->st_d2h);
    if (db->own_stream && db->stream) cudaStreamDestroy(db->stream);
    delete db;
}

}  // extern "C"
