# session-3 ncu evidence: launch lists of the three bench workloads (owner-local K-SET for
# TM-1 / TPC-B, packed outputs) and --set full captures of the new dominant kernels
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r3b
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for w in tm1 tpcb tpcc; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3b/launches_$w.csv \
    python tools/one_bulk.py $w kset > gpurun_out/r3b/launches_$w.log 2>&1; echo "launches $w rc=$?"; tail -1 gpurun_out/r3b/launches_$w.log
done
full() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${4:-1} -c 1 -o gpurun_out/r3b/full_$3 python tools/one_bulk.py $1 kset > gpurun_out/r3b/ncu_$3.log 2>&1; echo "full $3 rc=$?"; }
full tpcb kset_chain_exec tpcb_kset_chain_exec
full tpcb sp_walk tpcb_sp_walk
full tpcc sp_walk tpcc_sp_walk
full tpcc tpl_exec_warp tpcc_df_exec
for r in gpurun_out/r3b/full_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
done
ncu -i gpurun_out/r3b/full_tpcb_kset_chain_exec.ncu-rep --page source --csv --print-source sass > gpurun_out/r3b/full_tpcb_kset_chain_exec.source.csv 2>/dev/null
rm -f gpurun_out/r3b/*.ncu-rep
du -sh gpurun_out/r3b
