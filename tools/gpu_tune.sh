cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
run() { env $1 timeout 200 python bench.py --workload $3 --strategy $4 --steps 3 --warmup 3 --no-cpu-baseline --others "" > gpurun_out/tune_$2.json 2>gpurun_out/tune_$2.err; echo "$2 rc=$?"; }
run "GPUTX_KSET_Q=24" tpcb_q24 tpcb kset
run "GPUTX_KSET_Q=48" tpcb_q48 tpcb kset
run "GPUTX_KSET_Q=32 GPUTX_KSET_CLUSTER=0" tpcb_q32c0 tpcb kset
run "GPUTX_KSET_Q=16 GPUTX_KSET_CLUSTER=0" tpcb_q16c0 tpcb kset
run "GPUTX_KSET_Q=8 GPUTX_KSET_CLUSTER=0" tpcb_q8c0 tpcb kset
