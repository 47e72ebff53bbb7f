cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
for wb in 15 16 17 18; do for lm in 1 4; do
GPUTX_RANK_WINDOW=$wb GPUTX_RANK_LOCAL=$lm timeout 600 python bench.py --workload tpcc --steps 3 --warmup 3 --no-cpu-baseline --others "" > gpurun_out/bench_tpcc_w${wb}_l${lm}.json 2>/dev/null
done; done
