cd "${GRAFT_REPO_ROOT:-.}"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for q in 32 64; do for c in 16 8; do GPUTX_KSET_Q=$q GPUTX_KSET_CLUSTER=$c timeout 200 python tools/probe_exec.py tpcb; done; done
sed -i 's/return S == S_TPCC || S == S_TM1 ? 256 : KX_THREADS;/return S == S_TPCC || S == S_TM1 || S == S_TPCB ? 256 : KX_THREADS;/' paper_1103_3105_b200/csrc/engine.cu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo KB256
for q in 32 64 128; do for c in 16 8; do GPUTX_KSET_Q=$q GPUTX_KSET_CLUSTER=$c timeout 200 python tools/probe_exec.py tpcb; done; done
