cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "tpcb_multibranch or tm1 or depths" > gpurun_out/pytest_q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.log; tail -2 gpurun_out/pytest_q.log
run() { env $1 timeout 120 python bench.py --workload $3 --steps 5 --warmup 3 --no-cpu-baseline --others "" > gpurun_out/tune_$2.json 2>gpurun_out/tune_$2.err; echo "$2 rc=$?"; }
for it in 8 12 16; do
run "GPUTX_SORT_ITEMS=$it" tm1_i$it tm1
run "GPUTX_SORT_ITEMS=$it" tpcbadd_i$it tpcb_add
done
