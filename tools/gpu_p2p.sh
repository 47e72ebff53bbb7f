cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
GPUTX_WATCHDOG_MS=20000 timeout 900 python -m pytest tests/test_gpu_shard.py -q -x -k "fused or cli" > gpurun_out/pytest_p2p.log 2>&1; echo "shard tests rc=$?"; tail -15 gpurun_out/pytest_p2p.log
echo "== 2 ranks gloo on one GPU, strong TPC-C, fused P2P exchange"
GPUTX_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --workload tpcc --scaling strong --steps 3 --warmup 3 --also none --others "" > gpurun_out/n2.json 2> gpurun_out/n2.err; echo "rc=$?"; tail -c 1500 gpurun_out/n2.json; tail -5 gpurun_out/n2.err
