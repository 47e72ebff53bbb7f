# round-2 ncu evidence: launch lists of the three bench workloads and --set full captures of
# their dominant kernels (read back here with tools/ncu_traffic.py / summarize_ncu.py)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for w in tm1 tpcb tpcc; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_$w.csv \
    python tools/one_bulk.py $w kset > gpurun_out/r2_launches_$w.log 2>&1; echo "launches $w rc=$?"; tail -1 gpurun_out/r2_launches_$w.log
done
full() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${4:-1} -c 1 -o gpurun_out/r2_full_$3 python tools/one_bulk.py $1 kset > gpurun_out/r2_ncu_$3.log 2>&1; echo "full $3 rc=$?"; }
full tm1 kset_exec tm1_kset_exec
full tpcb kset_exec tpcb_kset_exec
full tpcc tpl_exec_warp tpcc_df_exec
full tpcc rank_window tpcc_rank_window
full tpcb rank_root tpcb_rank_root
full tm1 rank_stream tm1_rank_stream
ls -la gpurun_out/*.ncu-rep
# summaries only travel back (gpurun_out is capped at 64 MiB)
for r in gpurun_out/r2_full_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
done
ncu -i gpurun_out/r2_full_tm1_kset_exec.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_full_tm1_kset_exec.source.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
