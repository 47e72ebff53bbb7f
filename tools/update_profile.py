"""Rewrite the "Current state" section of profiles/round1.md from profiles/round1_*.json,
profiles/ncu_traffic.json and the tables of tools/profile_tables.py (/tmp/tables.md)."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = lambda *a: os.path.join(ROOT, *a)
old = open(P("profiles", "round1.md")).read()
tables = open("/tmp/tables.md").read()
bench_t, launch_t = tables.split("\n\n", 1)
ref = json.loads(open(P("profiles", "round1_ref_tm1.json")).read())
dflt = json.loads(open(P("profiles", "round1_bench_default.json")).read())
nt = json.load(open(P("profiles", "ncu_traffic.json")))
PEAK = dflt["roofline"]["peak"]
READ = {
    ("tm1", "kset_exec_kernel"): ("51.6 MB", "~3× sector amplification (4-8 B column accesses move 32-B sectors); 195 dependent rounds at ~2.6 µs: critical-path bound"),
    ("tm1", "rank_stream_tm1_kernel"): ("17.8 MB", "the serial walk of the hottest NURand (subscriber, component) roots bounds it; D writes stay in L2"),
    ("tm1", "rs_pass_kernel"): ("19.5 MB", "one of 3 passes over 1.2 M records: look-back latency, not bandwidth"),
    ("tm1", "group_kernel"): ("40 MB", "scatter of ids + 8 parameter words"),
    ("tpcb_add", "rank_kernel"): ("304 MB", "2 grid passes over 12 M records (+ the first pass's recpos prologue)"),
    ("tpcc_add", "rank_window_kernel"): ("4873 MB", "458 window passes; each touches one 2^17-transaction window (L2-resident)"),
    ("tpcb", "kset_exec_kernel"): ("404 MB", "4,196 rounds of ≤ 1,000 deposits: critical-path bound"),
}
rows = []
for (wl, k), (alg, why) in READ.items():
    if wl in nt and k in nt[wl]:
        e = nt[wl][k]
        frac = e["dram_bytes_per_launch"] / (e["ncu_us_per_launch"] * 1e-6) / 1e9 / PEAK
        rows.append(f"| {wl} `{k}` | {e['ncu_us_per_launch']:.1f} | {e['dram_bytes_per_launch'] / 1e6:.1f} MB | "
                    f"{100 * frac:.1f} % | {alg} | {e['l2_hit_pct']:.0f} % | {why} |")
r = dflt["roofline"]
new = f"""## Current state (end of round 1): `tools/gpu_final.sh` → `profiles/round1_bench_*.json`

`python -m pytest tests -m gpu`: 92 passed, 1 skipped (the TM-1 case of the AUTO→TPL
branch: Algorithm 1 never returns TPL when c = 0); `smoke()` ok.  The sharded bench path
ran with 2 ranks on the one GPU (gloo exchange; a functional check, numbers meaningless):
TPC-C and TPC-B ok (`profiles/round1_bench_n2_*.json`).

bench.py lines (device-resident inputs, L2 flushed before every timed step, 5 timed + 3
warm-up bulks; M txn/s; phases of the K-SET step in ms; AUTO = Algorithm 1 with the
default thresholds, the strategy it chose in brackets; the last column is the dominant
kernel's algorithmic bytes ÷ its CUDA-event time, and the ncu DRAM bytes where a capture
exists):

{bench_t}

Default bench line (`profiles/round1_bench_default.json`, TM-1 NURand K-SET, seed 1):
{dflt['value'] / 1e6:.1f} M txn/s device-resident, e2e {dflt['e2e']['value'] / 1e6:.1f} M txn/s
(13.7 MB H2D + 41 MB D2H per step), {dflt['gpu_launches']} kernel launches in the timed
region, SM clock {dflt['clocks']['sm_mhz']:.0f} MHz (no throttle reason), roofline
`{r['kernel']}` {r['achieved']:.0f} GB/s = {100 * r['frac']:.2f} % of {PEAK:.0f} GB/s (ncu DRAM fraction
{100 * (r['ncu_dram_frac'] or 0):.1f} %), critical path {r['critical_path']['rounds']} rounds at
{r['critical_path']['us_per_round']:.2f} µs.  cpu_baseline (the oracle, 1 host core of
"{dflt['cpu_baseline']['cpu']}", {dflt['cpu_baseline']['sample']}): {dflt['cpu_baseline']['value'] / 1e6:.1f} M txn/s.
Reference arm (`--impl reference`): {ref['value'] / 1e6:.1f} M txn/s.

**ncu `--set full` (one launch each, cold cache; raw pages `profiles/ncu_raw_*.csv`,
summarised in `profiles/ncu_traffic.json`, which bench.py reads for `roofline.traffic`):**

| workload / kernel | ncu µs | DRAM bytes (read+write) | ncu DRAM fraction | algorithmic bytes | L2 hit | reading |
|---|---:|---:|---:|---:|---:|---|
""" + "\n".join(rows) + f"""

**Launch shares, default bench (`profiles/round1_launches_tm1_final.csv`, ncu
`gpu__time_duration.sum`, 2 timed + 3 warm-up bulks, all strategies + e2e loop):**

{launch_t}
"""
start = old.index("## Current state")
end = old.index("Changes in this session", start)
open(P("profiles", "round1.md"), "w").write(old[:start] + new + "\n" + old[end:])
