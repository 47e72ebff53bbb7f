/* Drives libgputx.so through the C ABI only (no Python): TPC-B tiny-ish + TM-1-like
 * K-SET run with round tracing, to time the executor's hand-offs outside Python. */
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
#include "../include/gputx.h"

static uint64_t rng = 88172645463325252ull;
static uint64_t xr(void) { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; }

int main(void) {
    /* TPC-B with 4 branches: ~n/4 rounds of ~4 txns each?  Use B=2000 branches, n=200k:
       d ~ 100 + rounds of ~2000 txns -> multi-CTA rounds. */
    gputx_db_config cfg; memset(&cfg, 0, sizeof cfg);
    cfg.schema = GPUTX_TPCB; cfg.dims[0] = 2000; cfg.dims[1] = 10; cfg.dims[2] = 1000; cfg.max_bulk = 200000;
    gputx_db* db; int st = gputx_open_db(&cfg, &db); if (st) { printf("open %d\n", st); return 1; }
    for (uint32_t i = 0;; ++i) {
        const char* name; uint32_t el; uint64_t cnt;
        if (gputx_column_info(db, i, &name, &el, &cnt)) break;
        void* z = calloc(cnt, el); gputx_load_column(db, name, z, cnt * el); free(z);
    }
    gputx_seal(db);
    uint64_t n = cfg.max_bulk;
    uint8_t* type = calloc(n, 1); uint32_t* off = malloc((n + 1) * 4); uint32_t* pw = malloc(n * 16);
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t b = xr() % 2000, t = b * 10 + xr() % 10, a = b * 1000 + xr() % 1000;
        off[i] = i * 4; pw[4 * i] = a; pw[4 * i + 1] = t; pw[4 * i + 2] = b; pw[4 * i + 3] = (uint32_t)(xr() % 1000);
    }
    off[n] = n * 4;
    gputx_bulk bk = {type, off, pw, n, 0};
    gputx_trace_rounds(db, 1);
    gputx_stats s;
    for (int it = 0; it < 3; ++it) {
        gputx_submit_bulk(db, &bk, NULL);
        st = gputx_execute(db, GPUTX_KSET, &s);
        if (st) { printf("exec %d %s\n", st, gputx_last_error(db)); return 1; }
    }
    uint64_t nk = s.ksets;
    uint64_t* tr = malloc(nk * 64);
    gputx_read_round_ns(db, tr, nk);
    double sum = 0; for (uint64_t k = 0; k + 1 < nk; ++k) sum += (double)(tr[8 * (k + 1)] - tr[8 * k]);
    printf("C ABI TPC-B: ksets %llu exec_ms %.3f mean round %.2f us\n", (unsigned long long)nk, s.ms_exec, sum / 1e3 / (nk - 1));
    gputx_close_db(db);
    return 0;
}
