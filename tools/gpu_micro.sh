cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }

timeout 1500 python tools/micro_sweep.py ${FIGS:-fig3,calib,fig4,fig5,fig6,fig13,fig14} --out gpurun_out/micro_sweep.json 2>&1 | tail -80
