cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }

timeout 1500 python tools/pool_bench.py resp,skew --out gpurun_out/pool_bench.json 2>&1 | tail -40
