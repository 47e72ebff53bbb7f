cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "auto" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log; tail -3 gpurun_out/pytest_quick.log
timeout 300 python tools/probe_rank.py tm1 > gpurun_out/probe_rank_tm1.txt 2>&1
timeout 300 python tools/probe_rounds.py > gpurun_out/probe_rounds_tm1.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"kset_exec" -s 3 -c 1 -o gpurun_out/full_kset_tm1 python bench.py --steps 1 --warmup 3 --others "" --no-cpu-baseline > gpurun_out/ncu_full1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rank_root" -s 3 -c 1 -o gpurun_out/full_rank_tm1 python bench.py --steps 1 --warmup 3 --others "" --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"rs_pass" -s 12 -c 1 -o gpurun_out/full_sort_tm1 python bench.py --steps 1 --warmup 3 --others "" --no-cpu-baseline > gpurun_out/ncu_full3.log 2>&1
ls gpurun_out
