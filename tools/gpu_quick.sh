# quick GPU loop: build, the owner / pipe / packed / parity tests, TM-1 phases and the launch list
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/q
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "own or pipe or packed or parity or deferred or spine" > gpurun_out/q/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/q/pytest.log
for w in ${QW:-tm1}; do timeout 300 python tools/probe_phases.py $w 2>&1 | tail -1; timeout 300 python tools/probe_hostgap.py $w 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/q/launches_tm1.csv \
  python tools/one_bulk.py tm1 kset > gpurun_out/q/launches.log 2>&1; echo "launches rc=$?"
