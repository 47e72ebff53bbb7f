cd "${GRAFT_REPO_ROOT:-.}"
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rm in 0 256 512 1024; do echo "== runmax $rm"; GPUTX_KSET_RUNMAX=$rm timeout 300 python tools/probe_rounds.py tm1 2>&1 | grep "exec_ms\|size \["; done
for q in 64 256; do echo "== Q $q"; GPUTX_KSET_Q=$q timeout 300 python tools/probe_rounds.py tm1 2>&1 | grep "exec_ms\|size \["; done
for c in 16 4; do echo "== cluster $c"; GPUTX_KSET_CLUSTER=$c timeout 300 python tools/probe_rounds.py tm1 2>&1 | grep "exec_ms\|size \["; done
