# TPC-B chain executor check: chain / spine / own / parity / stress tests, phases
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/q
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "tpcb or chain or spine or stress or deferred or packed" > gpurun_out/q/pytest_chain.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/q/pytest_chain.log
timeout 300 python tools/probe_phases.py tpcb 2>&1 | tail -1
