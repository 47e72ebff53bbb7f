# quick GPU check: selected tests + selected bench workloads
# usage: bash tools/gpu_quick.sh "<pytest -k expr>" "<workloads>" [extra bench args]
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
K="$1"; WLS="$2"; shift 2
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
  tail -5 gpurun_out/pytest_quick.log
fi
for w in $WLS; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  tail -c 600 gpurun_out/bench_$w.err
done
