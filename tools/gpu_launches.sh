# per-kernel launch durations (ncu, cold cache, serialised) of one bench workload
# usage: bash tools/gpu_launches.sh <workload> [bench args]
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
W=$1; shift
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv \
  python bench.py --workload $W --steps 1 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/launches_$W.log 2>&1
tail -c 300 gpurun_out/launches_$W.log
