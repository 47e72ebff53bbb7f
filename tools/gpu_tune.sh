cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "tpcb or add_rule or smoke" > gpurun_out/pytest_q.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_q.log; tail -2 gpurun_out/pytest_q.log
run() { env $1 timeout 200 python bench.py --workload $3 --strategy $4 --steps 3 --warmup 3 --no-cpu-baseline --others "" > gpurun_out/tune_$2.json 2>gpurun_out/tune_$2.err; echo "$2 rc=$?"; }
run "X=1" tpcb tpcb kset
run "GPUTX_KSET_Q=16" tpcb_q16 tpcb kset
run "X=1" tpcbadd tpcb_add kset
run "X=1" tpcbhotadd tpcb_hot_add kset
