cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "tpcc or TPCC or fullsize or stress or shard or fuzz" 2>&1 | tail -2
for s in tpl kset; do timeout 300 python tools/probe_exec.py tpcc $s; done
