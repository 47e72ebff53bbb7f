cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
N() { ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/ncu_$RANDOM.log "$@"; }
echo "== ncu default"; timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n1.log python tools/repro_kset.py 2 tm1 2>&1 | tail -14
echo "== ncu cluster 0"; GPUTX_KSET_CLUSTER=0 timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n2.log python tools/repro_kset.py 2 tm1 2>&1 | tail -5
echo "== ncu diag 256"; GPUTX_KSET_DIAG=256 timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n3.log python tools/repro_kset.py 2 tm1 2>&1 | tail -5
echo "== ncu cache none clock none"; timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --cache-control none --clock-control none --log-file /tmp/n4.log python tools/repro_kset.py 2 tm1 2>&1 | tail -5
echo "== ncu tpl"; timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n5.log python tools/repro_kset.py 2 tm1 tpl 2>&1 | tail -5
echo "== ncu part"; timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n6.log python tools/repro_kset.py 2 tm1 part 2>&1 | tail -5
echo "== ncu tpcb kset"; timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n7.log python tools/repro_kset.py 2 tpcb 2>&1 | tail -5
echo "== GPUTX_SYNC ncu"; GPUTX_SYNC=1 timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n8.log python tools/repro_kset.py 2 tm1 2>&1 | tail -5
