cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
run() { env $1 timeout 200 python bench.py --workload $3 --strategy $4 --steps 3 --warmup 3 --no-cpu-baseline --others "" > gpurun_out/tune_$2.json 2>gpurun_out/tune_$2.err; echo "$2 rc=$?"; }
run "GPUTX_KSET_Q=64" tm1_q64 tm1 kset
run "GPUTX_KSET_Q=256" tm1_q256 tm1 kset
run "GPUTX_KSET_CLUSTER=16" tm1_c16 tm1 kset
run "GPUTX_KSET_Q=4" tpcc_q4 tpcc kset
run "GPUTX_KSET_Q=16" tpcc_q16 tpcc kset
run "GPUTX_KSET_CLUSTER=16" tpcc_c16 tpcc kset
run "GPUTX_KSET_CLUSTER=8" tpcb_c8 tpcb kset
