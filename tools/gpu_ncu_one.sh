# ncu --set full of one kernel of one bench workload:  bash tools/gpu_ncu_one.sh <workload> <kernel-regex> <tag> [skip]
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${4:-3} -c 1 -o gpurun_out/full_$3 \
  python bench.py --workload $1 --steps 1 --warmup 3 --others "" --no-cpu-baseline > gpurun_out/ncu_$3.log 2>&1
tail -2 gpurun_out/ncu_$3.log
