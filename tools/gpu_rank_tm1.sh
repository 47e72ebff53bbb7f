# TM-1 stream-rank change: parity tests touching TM-1 + rank time
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "tm1 or TM1 or fullsize or stress or depth" 2>&1 | tail -3 | tee gpurun_out/pytest_tail.txt
timeout 300 python tools/probe_rank_tm1.py
