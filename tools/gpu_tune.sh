cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "tpcc or tm1 or tpcb_tiny or depths or auto" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log; tail -3 gpurun_out/pytest_quick.log
for r in 0 256 512 1024; do GPUTX_KSET_RUNMAX=$r timeout 300 python bench.py --workload tm1 --steps 5 --warmup 3 --no-cpu-baseline --others "" > gpurun_out/bench_tm1_run$r.json 2>/dev/null; done
timeout 600 python bench.py --workload tpcc --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tpcc.json 2> gpurun_out/bench_tpcc.err; tail -c 400 gpurun_out/bench_tpcc.err
GPUTX_RANK_WINDOW=0 timeout 600 python bench.py --workload tpcc --steps 3 --warmup 3 --no-cpu-baseline --others "" > gpurun_out/bench_tpcc_nowin.json 2>/dev/null
GPUTX_RANK_WINDOW=16 timeout 600 python bench.py --workload tpcc --steps 3 --warmup 3 --no-cpu-baseline --others "" > gpurun_out/bench_tpcc_win16.json 2>/dev/null
GPUTX_RANK_WINDOW=12 timeout 600 python bench.py --workload tpcc --steps 3 --warmup 3 --no-cpu-baseline --others "" > gpurun_out/bench_tpcc_win12.json 2>/dev/null
