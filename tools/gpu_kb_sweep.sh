# K-SET executor CTA size sweep: bash tools/gpu_kb_sweep.sh "<kb list>" <workload> "<Q list>" "<cluster list>"
cd "${GRAFT_REPO_ROOT:-.}"
ORIG=$(grep -n "constexpr int kset_block()" paper_1103_3105_b200/csrc/engine.cu | cut -d: -f1)
for kb in $1; do
  sed -i "${ORIG}s/.*/template <int S> constexpr int kset_block() { return S == S_TPCC ? 256 : $kb; }/" paper_1103_3105_b200/csrc/engine.cu
  python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
  echo "KB $kb"
  for q in $3; do for c in $4; do GPUTX_KSET_Q=$q GPUTX_KSET_CLUSTER=$c timeout 200 python tools/probe_exec.py $2; done; done
done
