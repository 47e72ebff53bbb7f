# round 2: reproduce the driver's ncu-wrapped smoke() K-SET mismatch and bisect it
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
echo "== plain smoke"; timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
echo "== GPUTX_DEBUG ncu smoke"
GPUTX_DEBUG=1 timeout 600 ncu --metrics gpu__time_duration.sum -c 1000 --csv --log-file gpurun_out/ncu_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke.log 2>&1; echo "rc=$?"; grep -v "^==PROF" gpurun_out/ncu_smoke.log | tail -8
echo "== cluster 0, full grid"
GPUTX_KSET_CLUSTER=0 GPUTX_DEBUG=1 timeout 300 python tools/repro_kset.py 10 tm1 2>&1 | tail -12
GPUTX_KSET_CLUSTER=0 timeout 300 python tools/repro_kset.py 5 tpcb 2>&1 | tail -4
GPUTX_KSET_CLUSTER=0 timeout 300 python tools/repro_kset.py 5 tpcc 2>&1 | tail -4
echo "== cluster 0, diag 256 (no tail runs)"
GPUTX_KSET_CLUSTER=0 GPUTX_KSET_DIAG=256 timeout 300 python tools/repro_kset.py 5 tm1 2>&1 | tail -4
echo "== default cluster"
timeout 300 python tools/repro_kset.py 10 tm1 2>&1 | tail -4
echo "== racecheck (cluster 0)"
GPUTX_KSET_CLUSTER=0 timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/repro_kset.py 1 tm1 > gpurun_out/racecheck.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/racecheck.log
echo "== memcheck"
timeout 900 compute-sanitizer --tool memcheck python tools/repro_kset.py 1 tm1 > gpurun_out/memcheck.log 2>&1; echo "rc=$?"; tail -6 gpurun_out/memcheck.log
echo "== synccheck"
timeout 900 compute-sanitizer --tool synccheck python tools/repro_kset.py 1 tm1 > gpurun_out/synccheck.log 2>&1; echo "rc=$?"; tail -6 gpurun_out/synccheck.log
