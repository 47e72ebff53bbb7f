cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -x -k "tpcc or TPCC or fullsize or shard or fuzz or relaxed or chooser or auto" 2>&1 | tail -2
timeout 300 python tools/probe_exec.py tpcc part
