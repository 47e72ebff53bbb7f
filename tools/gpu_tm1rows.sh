cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_rounds.py tm1 2>&1 | head -1
timeout 300 python tools/probe_rounds.py tm1 2>&1 | grep "size \["
timeout 600 python bench.py --workload tm1 --also none --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['phases_ms'], {k:'%.3g'%v['value'] for k,v in d['strategies'].items()})"
