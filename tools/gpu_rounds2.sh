cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_stress.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_stress.log 2>&1; echo "stress rc=$?"; tail -3 gpurun_out/pytest_stress.log
for w in tm1 tpcb tpcc; do timeout 300 python tools/probe_rounds.py $w > gpurun_out/rounds_$w.txt 2>&1; echo "== $w"; head -1 gpurun_out/rounds_$w.txt; grep "mean us\|size \[" gpurun_out/rounds_$w.txt; done
for q in 64 128; do for c in 16 8; do echo "== tpcb Q=$q C=$c"; GPUTX_KSET_Q=$q GPUTX_KSET_CLUSTER=$c timeout 300 python tools/probe_rounds.py tpcb 2>&1 | grep "exec_ms\|mean us"; done; done
for q in 4 16; do echo "== tpcc Q=$q"; GPUTX_KSET_Q=$q timeout 300 python tools/probe_rounds.py tpcc 2>&1 | grep "exec_ms\|mean us"; done
