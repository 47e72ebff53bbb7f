cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for w in ${WLS:-tm1 tpcb tpcc}; do timeout 300 python tools/probe_rounds.py $w > gpurun_out/rounds_$w.txt 2>&1; echo "== $w"; head -40 gpurun_out/rounds_$w.txt; done
