cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "tpcc or depths or auto" > gpurun_out/pytest_q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.log; tail -3 gpurun_out/pytest_q.log
GPUTX_RANK_WCLUSTER=0 timeout 300 python -m pytest tests -m gpu -x -q -k "tpcc or depths" > gpurun_out/pytest_c0.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_c0.log; tail -3 gpurun_out/pytest_c0.log
run() { env $1 timeout 90 python bench.py --workload tpcc --steps 3 --warmup 3 --no-cpu-baseline --others "" > gpurun_out/tune_$2.json 2>gpurun_out/tune_$2.err; echo "$2 rc=$?"; }
run "GPUTX_RANK_WINDOW=14 GPUTX_RANK_WCLUSTER=0" w14c0
run "GPUTX_RANK_WINDOW=16 GPUTX_RANK_WCLUSTER=0" w16c0
run "GPUTX_RANK_WINDOW=17 GPUTX_RANK_WCLUSTER=0" w17c0
run "GPUTX_RANK_WINDOW=12" w12
run "GPUTX_RANK_WINDOW=13" w13
run "GPUTX_RANK_WINDOW=14" w14
