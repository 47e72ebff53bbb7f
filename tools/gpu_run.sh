set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
for w in tm1 tm1_uniform tpcb tpcb_add tpcb_hot_add tpcc tpcc_add tpcb_tiny; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
timeout 300 python bench.py --impl reference --workload tm1 --steps 3 --warmup 3 > gpurun_out/ref_tm1.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tm1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kset_exec|rank_kernel|rs_pass" -c 4 -o gpurun_out/full_tm1 python bench.py --steps 1 --warmup 3 --others "" --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
