# owner-local executor timing diagnostics: exec phase with bodies skipped (diag 1), without
# cross-warp waits / publishes (diag 64, results invalid), both
cd "${GRAFT_REPO_ROOT:-.}"
python -c "from paper_1103_3105_b200 import build; build.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for w in ${1:-tpcb tm1}; do for d in ${2:-0 1 64 65}; do echo -n "diag $d: "; GPUTX_KSET_DIAG=$d timeout 300 python tools/probe_phases.py $w 2>&1 | tail -1; done; done
