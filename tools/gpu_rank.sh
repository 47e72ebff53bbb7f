cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_pool.py -q -x -k "tm1" 2>&1 | tail -2
for L in 0 16 32 48 96 192; do echo "== rank_long $L"; GPUTX_RANK_LONG=$L timeout 300 python tools/probe_rounds.py tm1 2>&1 | head -1; done
