"""Markdown tables for profiles/roundN.md from a gpu_final.sh output directory.
   python tools/profile_tables.py gpurun_out/final"""
import glob
import json
import os
import subprocess
import sys

d = sys.argv[1]
rows = ["| workload | K-SET | PART | TPL | AUTO (chose) | e2e K-SET | sort | rank (passes) | group | exec (rounds, µs/round) | dominant kernel: algorithmic GB/s = frac; ncu DRAM bytes |",
        "|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---|"]
for f in sorted(glob.glob(os.path.join(d, "bench_*.json"))):
    if "default" in f or "_n2_" in f:
        continue
    try:
        x = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    st, ph, rf, g = x["strategies"], x["phases_ms"], x["roofline"], x["graph"]
    cp = rf.get("critical_path") or {}
    a = st.get("auto", {})
    tr = f"{rf['traffic'] / 1e6:.1f} MB" if rf.get("traffic") else "—"
    rows.append(f"| {x['config']['workload']} | {st['kset']['value'] / 1e6:.1f} | {st['part']['value'] / 1e6:.1f} | "
                f"{st['tpl']['value'] / 1e6:.1f} | {a.get('value', 0) / 1e6:.1f} ({a.get('chose')}) | "
                f"{x['e2e']['value'] / 1e6:.1f} | {ph['ms_sort']:.3f} | {ph['ms_rank']:.3f} ({g['rank_passes']}) | "
                f"{ph['ms_group']:.3f} | {ph['ms_exec']:.3f} ({g['depth'] + 1}, {cp.get('us_per_round', 0):.2f}) | "
                f"`{rf['kernel']}` {rf['achieved']:.0f} GB/s = {100 * rf['frac']:.2f}%; {tr} |")
print("\n".join(rows))
print()
here = os.path.dirname(os.path.abspath(__file__))
print(subprocess.run([sys.executable, os.path.join(here, "summarize_ncu.py"), "launches",
                      os.path.join(d, "launches_tm1.csv")], capture_output=True, text=True).stdout)
