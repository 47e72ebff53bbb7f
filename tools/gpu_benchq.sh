# quick bench: the default line without the CPU baseline legs, summarised
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
timeout 900 python bench.py --no-cpu-baseline "$@" > gpurun_out/benchq.json 2> gpurun_out/benchq.err; echo "bench rc=$?"
tail -3 gpurun_out/benchq.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/benchq.json").read().strip().splitlines()[-1])
def show(x, name):
    r = x.get("roofline") or {}
    print(name, "value %.4g all %.4g e2e %.4g parity %s ms %.3f" % (
        x["value"], x["all_txn_per_s"], x["e2e"]["value"], x["parity"], x["ms_per_step"]),
          "roof", r.get("kernel"), "%.4f" % (r.get("frac") or 0))
    print("   phases", {k: round(v, 3) for k, v in x["phases_ms"].items()}, "strategies", {k: "%.3g" % v["value"] for k, v in x["strategies"].items()})
show(d, "tm1")
for k, v in d.get("workloads", {}).items(): show(v, k)
print("clocks", d["clocks"], "launches", d["gpu_launches"])
PY
