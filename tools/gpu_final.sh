# round-end style gate: every GPU test, smoke plain and under ncu, the default bench line
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke.log 2>&1; echo "ncu smoke rc=$?"; tail -1 gpurun_out/ncu_smoke.log
START=$(date +%s); timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$? wall $(( $(date +%s) - START )) s"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
def show(x, name):
    r = x.get("roofline") or {}
    print(name, "value %.3g all %.3g e2e %.3g (pcie h2d %.0f d2h %.0f GB/s, floor %.3f ms) parity %s ms %.3f" % (
        x["value"], x["all_txn_per_s"], x["e2e"]["value"], x["e2e"]["pcie"]["h2d_gbs"], x["e2e"]["pcie"]["d2h_gbs"],
        x["e2e"]["pcie"]["transfer_floor_ms"], x["parity"], x["ms_per_step"]),
          "roof", r.get("kernel"), "%.4f" % (r.get("frac") or 0), "cpu", x["cpu_baseline"] and "%.3g" % x["cpu_baseline"]["value"])
    print("   phases", {k: round(v, 3) for k, v in x["phases_ms"].items()}, "strategies", {k: "%.3g" % v["value"] for k, v in x["strategies"].items()})
show(d, "tm1")
for k, v in d.get("workloads", {}).items(): show(v, k)
print("clocks", d["clocks"], "launches", d["gpu_launches"])
PY
