# sort look-back window sweep: TM-1 / TPC-B phases for RS_LB in $1
cd "${GRAFT_REPO_ROOT:-.}"
cp paper_1103_3105_b200/csrc/sort.cuh /tmp/sort.cuh.orig
for lb in $1; do
  sed -i "s/^constexpr int RS_LB = [0-9]*;/constexpr int RS_LB = $lb;/" paper_1103_3105_b200/csrc/sort.cuh
  python -c "from paper_1103_3105_b200 import build; build.build()" > /dev/null 2>&1 || { echo build failed; exit 1; }
  echo "RS_LB $lb"
  for w in tm1 tpcb; do timeout 300 python tools/probe_phases.py $w 2>&1 | tail -1; done
done
cp /tmp/sort.cuh.orig paper_1103_3105_b200/csrc/sort.cuh
