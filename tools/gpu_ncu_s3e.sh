# session-3 closing ncu evidence: launch lists of the three bench workloads and --set full of
# the dominant kernels (TM-1 owner executor, TPC-B chain executor, TPC-C K-SET dataflow)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/s3e
export PYTHONUNBUFFERED=1
for w in tm1 tpcb tpcc; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3e/launches_$w.csv \
    python tools/one_bulk.py $w kset > gpurun_out/s3e/launches_$w.log 2>&1; echo "launches $w rc=$?"
done
full() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${4:-1} -c 1 -o gpurun_out/s3e/full_$3 python tools/one_bulk.py $1 kset > gpurun_out/s3e/ncu_$3.log 2>&1; echo "full $3 rc=$?"; }
full tm1 kset_own_pipe tm1_kset_own_pipe
full tpcb kset_chain_exec tpcb_kset_chain_exec
full tpcc tpl_exec_warp tpcc_df_exec
for r in gpurun_out/s3e/full_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
done
rm -f gpurun_out/s3e/*.ncu-rep
