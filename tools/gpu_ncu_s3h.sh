# ncu evidence after the TPC-B deposit runs: launch list and --set full of the chain executor and
# the spine walk (now TPC-B's dominant kernel)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/s3h
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3h/launches_tpcb.csv \
  python tools/one_bulk.py tpcb kset > gpurun_out/s3h/launches_tpcb.log 2>&1; echo "launches rc=$?"
full() { timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s ${4:-1} -c 1 -o gpurun_out/s3h/full_$3 python tools/one_bulk.py $1 kset > gpurun_out/s3h/ncu_$3.log 2>&1; echo "full $3 rc=$?"; }
full tpcb kset_chain_exec tpcb_kset_chain_exec
full tpcb sp_walk tpcb_sp_walk
for r in gpurun_out/s3h/full_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
done
rm -f gpurun_out/s3h/*.ncu-rep
