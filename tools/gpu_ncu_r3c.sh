# session-3 final ncu evidence: launch list and --set full of the TM-1 owner-local executor (pipe)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r3c
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3c/launches_tm1.csv \
  python tools/one_bulk.py tm1 kset > gpurun_out/r3c/launches_tm1.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kset_own_pipe -s 1 -c 1 -o gpurun_out/r3c/full_tm1_kset_own_pipe python tools/one_bulk.py tm1 kset > gpurun_out/r3c/ncu.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/r3c/full_tm1_kset_own_pipe.ncu-rep --page raw --csv > gpurun_out/r3c/full_tm1_kset_own_pipe.raw.csv 2>/dev/null
ncu -i gpurun_out/r3c/full_tm1_kset_own_pipe.ncu-rep --page details --csv > gpurun_out/r3c/full_tm1_kset_own_pipe.details.csv 2>/dev/null
rm -f gpurun_out/r3c/*.ncu-rep
