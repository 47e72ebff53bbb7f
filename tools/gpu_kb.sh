cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 8 16; do for q in 64 128; do echo "== KB 256 cluster $c Q $q"; GPUTX_KSET_CLUSTER=$c GPUTX_KSET_Q=$q timeout 300 python tools/probe_rounds.py tm1 2>&1 | grep "exec_ms\|size \["; done; done
timeout 600 python -m pytest tests/test_gpu_stress.py tests/test_gpu_parity.py -q -x -k "tm1" 2>&1 | tail -2
