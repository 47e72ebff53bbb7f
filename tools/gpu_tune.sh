cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out/final2
O=gpurun_out/final2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rank_kernel" -s 1 -c 1 -o $O/full_tpcb_add_rank_kernel \
    python bench.py --workload tpcb_add --steps 1 --warmup 3 --others "" --no-cpu-baseline > $O/ncu_tpcb_add.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rank_window" -s 1 -c 1 -o $O/full_tpcc_add_rank_window \
    python bench.py --workload tpcc_add --steps 1 --warmup 3 --others "" --no-cpu-baseline > $O/ncu_tpcc_add.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"kset_exec" -s 1 -c 1 -o $O/full_tpcb_kset_exec \
    python bench.py --workload tpcb --steps 1 --warmup 3 --others "" --no-cpu-baseline > $O/ncu_tpcb.log 2>&1
timeout 900 python bench.py --workload tpcb_add --steps 5 --warmup 3 > $O/bench_tpcb_add.json 2> $O/bench_tpcb_add.err
ls $O
