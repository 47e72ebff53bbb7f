cd "${GRAFT_REPO_ROOT:-.}"
bash tools/gpu_rank_tm1.sh
bash tools/gpu_ncu_one.sh tm1 rank_stream rstream 2 > /dev/null 2>&1
ncu -i gpurun_out/full_rstream.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
for n in ('gpu__time_duration.sum','sm__cycles_active.avg','sm__cycles_active.max','sm__cycles_active.min','smsp__inst_executed.sum'): print(n, v[h.index(n)])
"
