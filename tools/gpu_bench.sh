# default bench line (N=1) + a gloo 2-rank strong-scaling functional run on the same GPU
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
START=$(date +%s); timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench.err | grep -v "^\s" ; echo "wall $(( $(date +%s) - START )) s"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
def show(x, name):
    r = x.get("roofline") or {}
    print(name, "value %.3g all %.3g e2e %.3g parity %s ms %.3f" % (x["value"], x["all_txn_per_s"], x["e2e"]["value"], x["parity"], x["ms_per_step"]),
          "roof", r.get("kernel"), "%.4f" % (r.get("frac") or 0), "cpu", x["cpu_baseline"] and "%.3g" % x["cpu_baseline"]["value"])
    print("   phases", {k: round(v, 3) for k, v in x["phases_ms"].items()}, "strategies", {k: "%.3g" % v["value"] for k, v in x["strategies"].items()})
show(d, "tm1")
for k, v in d.get("workloads", {}).items(): show(v, k)
print("clocks", d["clocks"])
PY
timeout 120 ./tools/handoff > gpurun_out/handoff.txt 2>&1; cat gpurun_out/handoff.txt
