/*
 * gputx.h — C ABI of the B200-native GPUTx bulk transaction engine.
 *
 * Implements the bulk execution model of He & Yu, "High-Throughput Transaction
 * Executions on Graphics Processors", PVLDB 4(5) 2011 (arXiv 1103.3105):
 *   - a bulk of stored-procedure transactions <id, type, params> (§3.2)
 *   - executed on the GPU so that the final database and every transaction's
 *     output equal serial execution in increasing timestamp order
 *     (Definition 1, §3.1)
 *   - under one of three strategies (§5):
 *       GPUTX_TPL  two-phase locking with ts-ordered counter locks (§5.1, App. C Fig. 11)
 *       GPUTX_PART one thread per partition, partitions run serially (§5.2)
 *       GPUTX_KSET k-set by k-set execution of the T-dependency graph (§4, §5.3)
 *
 * Conventions (every function):
 *   - returns gputx_status; nothing throws or aborts across the ABI; on error
 *     gputx_last_error(db) describes it (valid until the next call on db).
 *   - a gputx_db owns ALL device memory it uses; callers own every pointer they pass
 *     and may reuse it as soon as the call returns.
 *   - a handle is not thread-safe: one host thread per handle.
 *   - "host" pointers are ordinary (pinned or pageable) host memory; "device"
 *     pointers are CUDA device memory of cfg.device.
 *   - all work is ordered on the handle's stream (cfg.stream or a library stream).
 *
 * Schemas, type ids and parameter words (u32, little-endian; 0-based ids except
 * TM-1 s_id in [1, P]):
 *   TPC-B     type 0 deposit    [aid, tid, bid, delta(i32)]
 *   TM-1 type 0 GSD [s_id]   1 GND [s_id, sf, st, et]   2 GAD [s_id, ai]
 *                             3 USD [s_id, sf, bit1, data_a]   4 UL [nbr_lo, nbr_hi, vlr]
 *                             5 ICF [nbr_lo, nbr_hi, sf, st, et, numx_lo, numx_hi]
 *                             6 DCF [nbr_lo, nbr_hi, sf, st]
 *                             (nbr = sub_nbr string, 15 BCD digits; the lookup
 *                             half of the split transaction, runs at submit)
 *   TPC-C     type 0 NewOrder [w, d, c, ol_cnt, (i, supply_w, qty) x ol_cnt]
 *                             type 1 Payment  [w, d, cw, cd, by_name, c_or_last, h_amount]
 *                             (by-name customer lookup, runs at submit)
 *   MICRO     dims = (N tuples, T types <= 32, x, 0); type t in [0, T): [tuple]
 *                             reads the tuple (f32 bits, column "tuple"), applies 100*x "sin
 *                             calls" of type t (u = fma(v, 15/16 - t/128, (t - 15.5)/1024),
 *                             v = u * (1 + u^2 (C3 + u^2 C5)), IEEE fma/mul, DESIGN.md R-M1),
 *                             writes it back; never aborts.  Unsharded only.
 *
 * Output records (fixed stride per schema, zero for aborted transactions):
 *   TPC-B  8 B : i64 account balance after the deposit
 *   TM-1  40 B : GSD  [0]u64 sub_nbr [8]u64 hex [16]u32 msc [20]u32 vlr [24]u16 bits [26]u8[10] byte2
 *                GND  [0]u32 count [8,16,24]u64 numberx of the qualifying rows in start-time order
 *                GAD  [0]u8 data1 [1]u8 data2 [4]u32 data3 [8]u64 data4
 *   MICRO  4 B : u32 bits of the value written back
 *   TPC-C 200 B: NewOrder [0]u32 o_id [4]u32 ol_cnt [8]i64 total, line l at 16+12l:
 *                         [0]i32 s_quantity before the update [4]i32 amount [8]u8 brand 'B'
 *                Payment  [0]u32 c_id [4]u32 c_credit(1=BC) [8]i64 c_balance after
 * Status: 0 commit, 1 logical abort (no writes; two-phase procedures).
 */
#ifndef GPUTX_H
#define GPUTX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gputx_db gputx_db;                         /* opaque */

typedef enum {
    GPUTX_OK = 0,
    GPUTX_EINVAL = 1,        /* bad argument, bad column, malformed transaction        */
    GPUTX_ENOMEM = 2,        /* device or host allocation failed                         */
    GPUTX_EDUP_TYPE = 3,     /* register_types: a type id listed twice                    */
    GPUTX_EUNKNOWN_TYPE = 4, /* type id not compiled for the schema / not registered      */
    GPUTX_ESTATE = 5,        /* call out of order (e.g. submit twice, execute unsealed)   */
    GPUTX_ECAPACITY = 6,     /* bulk > max_bulk, output buffer short, insert table full   */
    GPUTX_ECROSS = 7,        /* PART: a cross-partition type with no fragment split       */
    GPUTX_EDEADLOCK = 8,     /* a spin watchdog tripped (K-SET round wait, grid barrier, TPL lock); db poisoned until reset */
    GPUTX_ECUDA = 9,         /* CUDA runtime error                                        */
    GPUTX_ENCCL = 10         /* inter-GPU exchange: a peer's arena cannot be mapped       */
} gputx_status;

typedef enum { GPUTX_TPL = 0, GPUTX_PART = 1, GPUTX_KSET = 2,
               GPUTX_AUTO = 3, /* Algorithm 1, see gputx_set_chooser */
               /* Relaxed timestamp constraint (Appendix G):
                * the result equals serial execution in SOME order (serializability), not
                * necessarily ts order; the order used is gputx_read_serial_order's.        */
               GPUTX_TPL_RELAXED = 4,  /* Figure 10 spin locks (CAS), acquired in item order,
                                          strict 2PL; order = lock-point order               */
               GPUTX_PART_RELAXED = 5  /* sort-free PART: per-partition counters give each
                                          transaction its position, a prefix sum the starts
                                          (PAPER.md:523); cross-partition transactions then run
                                          under TPL_RELAXED. Single-GPU only.  */
} gputx_strategy;
typedef enum { GPUTX_TPCB = 1, GPUTX_TM1 = 2, GPUTX_TPCC = 3,
               GPUTX_MICRO = 4  /* the paper's micro benchmark (§6.1), see below */ } gputx_schema;

/* Device-memory hooks: every device allocation of the handle goes through
 * alloc(bytes, stream, ctx) / free(ptr, stream, ctx) when they are set -- e.g. PyTorch's
 * caching allocator, so the engine shares the framework's memory pool -- else cudaMalloc. */
typedef void* (*gputx_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*gputx_free_fn)(void* ptr, void* stream, void* ctx);

typedef struct {
    gputx_schema schema;
    uint32_t dims[4];         /* TPC-B: branches, tellers/branch, accounts/branch, 0
                                 TM-1 : subscribers P, 0, 0, 0
                                 TPC-C: warehouses W, districts/W D, customers/district C, items I */
    uint64_t max_bulk;        /* transactions per bulk, <= 1<<24 (timestamp field width)            */
    uint64_t insert_capacity; /* merged insert tables hold this many full bulks; 0 => 8            */
    uint32_t part_size;       /* PART: TM-1 subscribers / micro tuples per partition; 0 => TM-1 1,  */
                              /* micro 128 (PAPER.md:461 tuned 128 on its GPU; B200: DESIGN.md)    */
    int device;               /* CUDA device ordinal                                                */
    void* stream;             /* cudaStream_t to order all work on; NULL => a library-owned stream  */
    uint32_t flags;           /* GPUTX_FLAG_* below; 0 = the paper's R/W conflict rule              */
    uint32_t shard;           /* this handle's shard in [0, nshards)                                */
    uint32_t nshards;         /* 0 or 1: unsharded; 2..8: one handle per GPU, see "Sharding" below  */
    gputx_alloc_fn alloc;     /* NULL => cudaMalloc / cudaFree (both or neither)                     */
    gputx_free_fn free;
    void* alloc_ctx;
} gputx_db_config;

/* gputx_db_config.flags
 * GPUTX_FLAG_ADD_RULE: a domain-specific conflict rule (PAPER.md:475(c)):
 *   columns that their transaction types only increment and no output reads (TPC-B teller
 *   and branch balances, TPC-C W_YTD and D_YTD) are accessed in mode ADD; two adds of one
 *   item do not conflict (an add still conflicts with reads and writes).  K-SET depths and
 *   TPL lock keys follow the rule; the final database and every output stay equal to
 *   serial execution in ts order (the increments are atomic and commutative). */
#define GPUTX_FLAG_ADD_RULE 1u
/* GPUTX_FLAG_PACKED_OUT: variable-size output records.  Transaction i's record is the
 * first gputx_out_size(type, params) bytes of its fixed-stride record (the rest of that
 * record is always zero), at byte offset out_off[i] = sum of the sizes before it, so a
 * bulk's outputs are one dense array of out_off[n] bytes instead of n * gputx_out_stride:
 * the result transfer the paper counts in the bulk time carries only
 * what the procedures return.  Sizes (multiples of 8; micro 4):
 *   TPC-B 8; micro 4; TM-1 GSD 40, GND 32, GAD 16, USD / UL / ICF / DCF 0;
 *   TPC-C NewOrder 16 + 12 x ol_cnt rounded up to 8, Payment 16.
 * The offsets are computed at submit (gputx_read_out_offsets); gputx_read_results,
 * gputx_results_device and gputx_run_bulks then move out_off[n] bytes.  Not with sharding
 * or the transaction pool (EINVAL there). */
#define GPUTX_FLAG_PACKED_OUT 2u
/* GPUTX_FLAG_DEFERRED_CHECK (TM-1 and micro, unsharded): gputx_submit_bulk enqueues the
 * validation without waiting for its verdict (no host round trip between submit and
 * execute).  Validation errors (EINVAL, EUNKNOWN_TYPE, ECAPACITY for parameter words) are
 * then returned by the following gputx_execute / gputx_wait instead, and the database is
 * unchanged: K-SET's owner-local path executes a failed bulk as empty; every other strategy
 * takes the verdict before it launches anything.  submit still returns the host-detectable
 * errors (ESTATE, bulk larger than max_bulk, null pointers). */
#define GPUTX_FLAG_DEFERRED_CHECK 4u

typedef struct {
    const uint8_t* type;        /* u8[n]                                                */
    const uint32_t* param_off;  /* u32[n+1], param_off[0] == 0                          */
    const uint32_t* param_words;/* u32[param_off[n]]                                    */
    uint64_t n;
    int on_device;              /* 0: host pointers (copied H2D at submit);
                                   1: device pointers already resident in HBM           */
    const uint32_t* ts;         /* u32[n] global timestamps, strictly increasing, or NULL
                                   (then ts = first_ts + i); REQUIRED sharded */
} gputx_bulk;

typedef struct {
    uint64_t n, committed, aborted;
    uint64_t depth;          /* d: depth of the T-dependency graph (K-SET) */
    uint64_t ksets;          /* d + 1 (K-SET)                                            */
    uint64_t zero_set;       /* w0 = |0-set| (K-SET)                        */
    uint64_t records;        /* access records emitted (K-SET, TPL)                     */
    uint64_t rank_passes;    /* rank passes to the fixpoint (K-SET; TPC-C: summed over windows; TM-1: 1) */
    uint64_t parts;          /* partitions (PART)                                       */
    uint64_t fragments;      /* executed fragments (PART)                               */
    uint64_t max_chain;      /* longest partition (PART)                                */
    uint64_t launches;       /* kernels this library launched for the bulk (submit + execute) */
    double ms_emit, ms_sort, ms_rank, ms_group, ms_exec, ms_merge, ms_total;
    uint64_t cross;          /* c: transactions with fragments in more than one PART partition
                                (filled by PART and AUTO, else 0)             */
    uint64_t strategy;       /* the strategy that ran (GPUTX_AUTO: the one Algorithm 1 chose) */
    double ms_ingest;        /* device time of the last submit on the handle's stream: H2D/D2D of the
                                signatures, validation, split lookups, insert counts  */
    double ms_exchange;      /* sharded: device time of the cross-shard exchange of this bulk (pack,
                                peer transfer, merge by ts; return of fragment outputs), else 0   */
    uint64_t flags;          /* GPUTX_STAT_* bits below                                          */
    uint64_t out_bytes;      /* bytes of this bulk's output records: n * gputx_out_stride, or the
                                packed size with GPUTX_FLAG_PACKED_OUT (what a result read moves) */
} gputx_stats;

/* gputx_stats.flags */
#define GPUTX_STAT_CLUSTER_FALLBACK 1u   /* K-SET executor was launched without its cluster shape
                                            (e.g. by a profiler) and used counter hand-offs only */
#define GPUTX_STAT_KSET_DATAFLOW 2u      /* K-SET ran the dataflow executor (per-item completion
                                            counters, k-set-order dispatch) instead of rounds  */
#define GPUTX_STAT_KSET_CHAIN 16u        /* TPC-B K-SET over spine chains: one thread per branch
                                            chain, members in k-set order, cross-chain waits  */
#define GPUTX_STAT_PIPELINED 8u         /* gputx_run_bulks ran the bulk without a host round trip
                                            (TM-1 / micro K-SET): counts are set, phase times 0 */
#define GPUTX_STAT_KSET_OWNER 4u         /* K-SET ran owner-local rounds: every warp executes the
                                            k-sets of its own transactions (root key -> warp),
                                            waiting only for cross-warp predecessors (default
                                            for TM-1 / TPC-B / micro under the R/W rule)       */

/* Create a database handle for cfg->schema with empty (zero) columns on cfg->device.
 * Errors: EINVAL (bad schema/dims/max_bulk), ENOMEM, ECUDA.  *out is NULL on error. */
gputx_status gputx_open_db(const gputx_db_config* cfg, gputx_db** out);

/* Copy one column of the initial image from host memory ("the necessary
 * data columns and indexes are copied from the main memory to the GPU memory").
 * name/bytes must match the schema's column list (gputx_column_info); EINVAL otherwise.
 * Only before gputx_seal. */
gputx_status gputx_load_column(gputx_db* db, const char* name, const void* host, uint64_t bytes);

/* Column catalog ("system catalog"): index -> name, element bytes and row
 * count. Returns EINVAL past the last column. */
gputx_status gputx_column_info(const gputx_db* db, uint32_t index, const char** name,
                               uint32_t* elem_bytes, uint64_t* count);

/* Finish loading: build the static indexes (TM-1 sub_nbr hash, TPC-C (w,d,c_last)
 * index), keep a pristine device copy for gputx_reset.  ESTATE if called twice. */
gputx_status gputx_seal(gputx_db* db);

/* Enable k compiled-in stored procedures (registering = adding a case of
 * the combined switch kernel).  Errors: EDUP_TYPE, EUNKNOWN_TYPE; nothing changes on
 * error.  Unless called, every type of the schema is enabled. */
gputx_status gputx_register_types(gputx_db* db, const uint32_t* type_ids, uint32_t k);

/* Submit one bulk.  Copies/reads the signatures, assigns ts =
 * first_ts + i, validates every transaction and resolves the static lookups.
 * Synchronous.  Errors (nothing enqueued): ECAPACITY (n > max_bulk), EINVAL /
 * EUNKNOWN_TYPE (first bad transaction in the message), ESTATE (unsealed, or a bulk
 * already submitted and not executed).  *first_ts may be NULL. */
gputx_status gputx_submit_bulk(gputx_db* db, const gputx_bulk* bulk, uint64_t* first_ts);

/* Execute the submitted bulk with the given strategy to completion (synchronous) and
 * merge the insert buffers.  stats may be NULL.  Errors: ESTATE (nothing
 * submitted), EDEADLOCK (a device wait exceeded the spin watchdog, GPUTX_WATCHDOG_MS,
 * default 10 s: the handle is poisoned until gputx_reset), ECAPACITY (insert table full), ECUDA. */
gputx_status gputx_execute(gputx_db* db, gputx_strategy strategy, gputx_stats* stats);

/* gputx_execute in two halves, so the caller's thread is free while the bulk runs (and a
 * device timer can bracket exactly the bulk's kernels).  gputx_execute_async enqueues every
 * kernel of the strategy on the handle's stream and returns; host-detectable errors
 * (ESTATE nothing submitted, EINVAL bad strategy) are returned here, nothing is enqueued
 * then.  (GPUTX_AUTO and the sharded / relaxed paths still synchronise inside for their
 * device-computed decisions.)  gputx_wait synchronises and returns what gputx_execute would
 * have: the device-side errors (EDEADLOCK, ECUDA) and the stats (may be NULL).  Until
 * gputx_wait, every other call on the handle except gputx_close_db returns ESTATE. */
gputx_status gputx_execute_async(gputx_db* db, gputx_strategy strategy);
gputx_status gputx_wait(gputx_db* db, gputx_stats* stats);

/* A stream of k HOST bulks executed back to back with the transfers overlapped: bulk i+1's
 * H2D copy and bulk i-1's D2H of results run on two copy streams while bulk i executes
 * (double-buffered device slots).  Equivalent to k x (gputx_submit_bulk + gputx_execute +
 * gputx_read_results) -- same results, same errors (the first failing bulk stops the run);
 * the paper counts the transfers in the bulk time and keeps them below 5% (PAPER.md:449,
 * 515).  status[i] (u8[n_i]) and out[i] (n_i * gputx_out_stride bytes; with
 * GPUTX_FLAG_PACKED_OUT the bulk's packed outputs, at most that) are caller-owned host
 * buffers (pinned for real overlap; entries may be NULL); stats: k entries or NULL.
 * Returns after the last result has landed; every bulk takes ts = next_ts + position. */
gputx_status gputx_run_bulks(gputx_db* db, const gputx_bulk* bulks, uint64_t k, gputx_strategy strategy,
                             uint8_t* const* status, void* const* out, gputx_stats* stats);

/* Thresholds of the strategy chooser, Algorithm 1 (Appendix D
 * "Choosing the suitable execution strategy").  GPUTX_AUTO first builds the
 * T-dependency graph's structural parameters of the submitted bulk:
 *   w0 = |0-set| and d = depth, from the K-SET emit / sort / rank phases, and
 *   c  = transactions whose PART fragments lie in more than one partition;
 * then runs   w0 >= w0_bar            -> K-SET (reusing the ranks)
 *             c <= c_bar or d >= d_bar -> PART
 *             otherwise               -> TPL  (reusing the sorted access records).
 * Defaults, calibrated on B200 with tools/calibrate_chooser.py (the paper calibrates its
 * thresholds; profiles/round1_chooser_calibration.json): w0_bar = 64 x #SMs
 * (9,472 on B200; PAPER.md:414 ties it to the GPU's processors), d_bar = 0, c_bar = 0 --
 * i.e. K-SET for a wide 0-set, else PART; with d_bar = 0 the default NEVER returns TPL.
 * That is a calibration outcome, not a property of TPL: TPL was the fastest strategy on 5
 * of the 13 calibration bulks.  Four of them (TM-1, TM-1 uniform, TPC-B ADD, TPC-C ADD) have
 * w0 >= 9,472, where line 2 returns K-SET before TPL is considered; TPC-C (w0 = 624,
 * d = 7,990) would pick TPL only with d_bar > 7,990, which loses more on the TPC-B sweep
 * bulks (PART-best, d up to 99,466) than it gains -- Algorithm 1's three thresholds cannot
 * separate them (DESIGN.md §4 "Strategy chooser"). 
 * Errors: EINVAL (null handle). */
gputx_status gputx_set_chooser(gputx_db* db, uint64_t w0_bar, uint64_t d_bar, uint64_t c_bar);

/* Type grouping inside each k-set (Appendix D "Branch divergence"):
 * transactions of one k-set are ordered by p groups of type ids (type * p / T, the high
 * part of the id -- what (log2 p)/b passes of a b-bit radix partitioning on the type give),
 * so a warp's lanes take at most a few branches of the combined switch.  p = 0 (default)
 * or p = T: one group per type (full grouping; on B200 it is the same single counting-sort
 * pass as depth-only grouping); p = 1: depth only, types mixed in ts order (the paper's
 * "basic execution").  The best p is found by calibration (tools/calibrate_grouping.py,
 * PAPER.md:404 "we run calibration to determine the number of passes").
 * Errors: EINVAL (p > T). */
gputx_status gputx_set_grouping(gputx_db* db, uint32_t p);

/* Copy the last executed bulk's results to host: status u8[n] (may be NULL) and the
 * output records (n * gputx_out_stride bytes, or out_off[n] with GPUTX_FLAG_PACKED_OUT;
 * out may be NULL).  ECAPACITY if out_bytes
 * is short, ESTATE before the first execute.  Sharded: the n home transactions passed to
 * gputx_shard_pack, in that order, after gputx_shard_return_merge. */
gputx_status gputx_read_results(gputx_db* db, uint8_t* status, void* out, uint64_t out_bytes);

/* Device pointers to the last bulk's status u8[n] and output records; valid until the
 * next submit.  For callers that keep results in HBM. */
gputx_status gputx_results_device(gputx_db* db, const uint8_t** status, const void** out,
                                  uint64_t* n);

uint32_t gputx_out_stride(gputx_schema schema);

/* GPUTX_FLAG_PACKED_OUT: the submitted bulk's output offsets u32[n + 1] (out_off[n] = the
 * bytes of its packed outputs) to host; *bytes (may be NULL) = out_off[n].  Without the
 * flag the records are fixed-stride and this returns EINVAL.  ESTATE before a submit. */
gputx_status gputx_read_out_offsets(gputx_db* db, uint32_t* host, uint64_t n, uint64_t* bytes);

/* Snapshot one current column to host (exact bytes of the column). */
gputx_status gputx_read_column(gputx_db* db, const char* name, void* host, uint64_t bytes);

/* Merged insert tables (TPC-B "history"; TPC-C "order", "new_order", "order_line",
 * "history"): row count, and one column (u32/i32 per row) copied to host. */
gputx_status gputx_insert_rows(gputx_db* db, const char* table, uint64_t* rows);
gputx_status gputx_read_insert_column(gputx_db* db, const char* table, const char* column,
                                      void* host, uint64_t bytes);

/* Diagnostics of the last execute: K-SET depth per transaction (u32[n]); the
 * k-set execution order perm (u32[n]); TPL lock key per access record in emission
 * order (u32[records]).  ESTATE when the last strategy did not compute them. */
gputx_status gputx_read_depths(gputx_db* db, uint32_t* host, uint64_t n);
gputx_status gputx_read_perm(gputx_db* db, uint32_t* host, uint64_t n);

/* The serialization order of the last execute under GPUTX_TPL_RELAXED / GPUTX_PART_RELAXED:
 * u32 order[n], a permutation of the bulk's transactions such that executing them one at a
 * time in this order (each keeping its own ts for time fields) gives exactly the database,
 * statuses and outputs the relaxed execution produced.  ESTATE for other strategies. */
gputx_status gputx_read_serial_order(gputx_db* db, uint32_t* host, uint64_t n);

/* K-SET round tracing (diagnostics): when on, the executor records device times (ns,
 * %globaltimer) per round k: [8k] CTA 0 starts, [8k+1] CTA 0 has signalled, [8k+2] and
 * [8k+3] the same for CTA 1 (0 if it did not take part), [8k+4], [8k+5] polls CTA 0 / 1
 * spent waiting for round k-1.  gputx_read_round_ns copies 8 * rounds u64 (rounds <= n)
 * of the last K-SET execute.  ESTATE if tracing was off. */
gputx_status gputx_trace_rounds(gputx_db* db, int on);
gputx_status gputx_read_round_ns(gputx_db* db, uint64_t* host, uint64_t rounds);

/* Rank-pass tracing (same switch): per pass p of the last K-SET rank fixpoint, u64
 * [8p] pass start, [8p+1] last CTA done aggregating, [8p+2] past barrier 1, [8p+3]
 * last CTA done sweeping, [8p+4] past barrier 2 (ns, %globaltimer), [8p+5] tiles swept,
 * [8p+6] tile sweeps.  Copies 8 * passes u64 (passes <= 1024).  ESTATE if tracing was
 * off or the last execute was not K-SET; EINVAL for passes > 1024. */
gputx_status gputx_read_rank_ns(gputx_db* db, uint64_t* host, uint64_t passes);

/* ---- Sharding (multi-GPU) ----------------------------------------------
 * Tables are partitioned by root key (TPC-B branch, TPC-C warehouse, TM-1 subscriber):
 * shard r owns roots [ceil(r*R/G), ceil((r+1)*R/G)) of R, so root x lives on x*G/R.  Each
 * handle holds the whole image but only its roots are ever read or written; the union of
 * the shards' roots is the database.  A cross-shard transaction is split into fragments
 * with no data flow between them (PART's split, DESIGN.md R-S9), each run on the shard
 * that owns its root: every shard runs its fragments in global ts order, which projects
 * the serial order onto its items, so the union equals serial execution (Definition 1).
 * Per bulk, every shard calls, in this order (the caller moves the buffers between
 * shards, e.g. NCCL all-to-all over NVLink):
 *   1. gputx_shard_pack(db, home, send, cap, counts): stage the home bulk (transactions
 *      whose home root is local, global ts required) and write, for every other shard q,
 *      counts[q] records [ts, type, len, params, 0-padding] (gputx_shard_stride(schema, 0)
 *      u32 words each) to the device buffer send, grouped by q in increasing q, each group
 *      in ts order.  counts: host u64[nshards].  ECAPACITY if cap (records) is short.
 *   2. gputx_shard_submit(db, recv, n_recv, &n_local): recv = the records the peers sent
 *      to this shard (device, any order of groups); the local bulk is home + received
 *      transactions in ts order.  ECROSS if a home transaction's root is not local.
 *   3. gputx_execute (any strategy; ranks and locks are shard-local).
 *   4. gputx_shard_return_pack(db, send, cap, counts): the outputs of the peers'
 *      transactions, [ts, out words] (gputx_shard_stride(schema, 1) words), grouped by
 *      home shard.
 *   5. gputx_shard_return_merge(db, recv, n_recv): OR the returned fragment outputs into
 *      the home records (fragments write disjoint fields).  Then gputx_read_results.
 * The pack calls are synchronous: their send buffer is complete when they return.  The
 * caller must have completed the writes into recv (e.g. synchronized the stream its
 * exchange ran on) before calling gputx_shard_submit / gputx_shard_return_merge, which
 * read it on the handle's stream. */
uint32_t gputx_shard_stride(gputx_schema schema, int result);

/* The same exchange FUSED into the library over peer memory (no host
 * staging and no collective call): every shard owns an exchange arena in its HBM; the
 * kernel that packs a shard's cross-shard records writes each one straight into the owner
 * shard's arena (P2P stores over NVLink / NVSwitch, or same-device stores when shards share
 * a GPU) and its last CTA publishes the bulk's epoch to every peer; the receiving shard's
 * stream waits for all peers' epochs on the device (spin watchdog -> EDEADLOCK), merges the
 * received records by ts and ingests the local bulk.  Fragment outputs return the same way.
 *   connect once: blob = gputx_shard_export(db) on every shard (GPUTX_PEER_BLOB_BYTES; a
 *     CUDA IPC handle of the arena), all-gathered by the caller in shard order (any host
 *     plumbing, e.g. torch.distributed.all_gather_object), then gputx_shard_connect(db,
 *     blobs); handles of ONE process: gputx_shard_connect_local(dbs, n).
 *   per bulk, on every shard: gputx_shard_dispatch(db, home) -> gputx_shard_receive(db,
 *     &n_local) -> gputx_execute -> gputx_shard_return(db) -> gputx_shard_collect(db) ->
 *     gputx_read_results.  In one process, call dispatch on every handle before receive on
 *     any (receive waits for all peers), and return on every handle before collect.
 * dispatch always publishes (an empty contribution if it fails validation), so peers never
 * hang on a failing shard.  ECAPACITY if an arena's record area is full (it holds max_bulk
 * records); ENCCL if a peer's arena cannot be mapped. */
#define GPUTX_PEER_BLOB_BYTES 128
gputx_status gputx_shard_export(gputx_db* db, void* blob);
gputx_status gputx_shard_connect(gputx_db* db, const void* blobs);
gputx_status gputx_shard_connect_local(gputx_db* const* dbs, uint32_t n);
gputx_status gputx_shard_dispatch(gputx_db* db, const gputx_bulk* home);
gputx_status gputx_shard_receive(gputx_db* db, uint64_t* n_local);
gputx_status gputx_shard_return(gputx_db* db);
gputx_status gputx_shard_collect(gputx_db* db);
gputx_status gputx_shard_pack(gputx_db* db, const gputx_bulk* home, uint32_t* send, uint64_t send_cap,
                              uint64_t* counts);
gputx_status gputx_shard_submit(gputx_db* db, const uint32_t* recv, uint64_t n_recv, uint64_t* n_local);
gputx_status gputx_shard_return_pack(gputx_db* db, uint32_t* send, uint64_t send_cap, uint64_t* counts);
gputx_status gputx_shard_return_merge(gputx_db* db, const uint32_t* recv, uint64_t n_recv);

/* ---- Streaming K-SET over a live transaction pool (SURVEY.md
 * §8(f) NEXT-2) ---------------------------------------------------------------------------
 * Transactions arrive in the pool in submission order (ts = next_ts + i, the auto-increment
 * id of PAPER.md:95) and wait there until they are in the pool's 0-set: no earlier pool
 * transaction conflicts with them.  Each step executes exactly that 0-set in one lock-free
 * round (Property 1) and removes it: "It iteratively pick the 0-set as a bulk
 * for execution ... the transactions in 1-set become the 0-set".  The
 * k-sets are maintained incrementally: an arrival's access records are radix-sorted and
 * merged into the pool's sorted record array, and the 0-set is found by one pass of
 * group-head checks, without a rank fixpoint.  Every executed transaction
 * precedes, in ts, every pending transaction it conflicts with, so once the pool drains the
 * database and every transaction's (status, output) equal serial execution in ts order
 * (Definition 1).  Insert rows are appended at execution time, in ts order within a step.
 *   gputx_pool_submit(db, arrivals, &first_ts): validate + resolve lookups (as
 *       gputx_submit_bulk) and append; EINVAL if arrivals->ts is set, ECAPACITY if the pool
 *       would exceed max_bulk transactions, ESTATE while a bulk is submitted / sharded handles.
 *   gputx_pool_step(db, stats, &executed): execute the current 0-set (stats: n = executed,
 *       ms_rank = 0-set extraction, ms_exec = the round, ms_merge = pool compaction).
 *   gputx_pool_read(db, ts, status, out, cap, &n): host copies of the last step's executed
 *       transactions in ts order: u32 ts[n], u8 status[n], out[n * gputx_out_stride]; any of
 *       the three may be NULL; ECAPACITY if cap < n (n is still returned).
 *   gputx_pool_pending(db, &n): transactions still in the pool.
 * gputx_submit_bulk returns ESTATE while the pool is not empty; gputx_reset empties it. */
gputx_status gputx_pool_submit(gputx_db* db, const gputx_bulk* arrivals, uint64_t* first_ts);
gputx_status gputx_pool_step(gputx_db* db, gputx_stats* stats, uint64_t* executed);
gputx_status gputx_pool_read(gputx_db* db, uint32_t* ts, uint8_t* status, void* out, uint64_t cap, uint64_t* n);
gputx_status gputx_pool_pending(const gputx_db* db, uint64_t* n);

/* Snapshot of the current database (every column and the merged insert tables) into one
 * caller-owned host buffer; 2-call size query: buf == NULL sets *bytes to the size needed.
 * Layout: "GPTXSNAP" u32 version(1) u32 schema u32 dims[4] u32 ncols u32 ntables; per column
 * u32 name_len, name, u32 elem_bytes, u64 count, the column's bytes; per insert table u32
 * name_len, name, u32 ncols, u64 rows, per column u32 name_len, name, rows * 4 bytes.
 * ECAPACITY (and *bytes = needed) if *bytes is short; ESTATE before seal. */
gputx_status gputx_snapshot(gputx_db* db, void* buf, uint64_t* bytes);

/* Restore the pristine image (columns and insert tables) by a device copy. */
gputx_status gputx_reset(gputx_db* db);

void gputx_close_db(gputx_db* db);
const char* gputx_last_error(const gputx_db* db);

/* Launch-shape overrides for tests of grid-shape independence (0 = default):
 * exec_grid = CTAs of the persistent K-SET executor (<= co-resident); others reserved. */
gputx_status gputx_set_launch(gputx_db* db, uint32_t exec_block, uint32_t exec_grid,
                              uint32_t narrow_max);

#ifdef __cplusplus
}
#endif
#endif /* GPUTX_H */
