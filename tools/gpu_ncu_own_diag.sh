# source-level ncu of the owner-local executor skeleton (TPC-B, bodies skipped: diag 1) and the full executor
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/r3d
python -c "from paper_1103_3105_b200 import build; build.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
for d in ${1:-1 0}; do
  GPUTX_KSET_DIAG=$d timeout 900 ncu --set full --clock-control none --import-source on -k regex:kset_own_exec -s 1 -c 1 -o gpurun_out/r3d/tpcb_diag$d python tools/one_bulk.py tpcb kset > gpurun_out/r3d/log$d 2>&1; echo "rc=$?"
  ncu -i gpurun_out/r3d/tpcb_diag$d.ncu-rep --page source --csv --print-source sass > gpurun_out/r3d/tpcb_diag$d.source.csv 2>/dev/null
  ncu -i gpurun_out/r3d/tpcb_diag$d.ncu-rep --page details --csv > gpurun_out/r3d/tpcb_diag$d.details.csv 2>/dev/null
done
rm -f gpurun_out/r3d/*.ncu-rep
