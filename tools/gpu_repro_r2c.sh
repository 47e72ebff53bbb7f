cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
export PYTHONUNBUFFERED=1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
echo "== ncu default"; GPUTX_DEBUG=1 timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n1.log python tools/repro_kset.py 1 tm1 2>&1 | tail -14
echo "== ncu KSET_Q=4096 (all rounds narrow)"; GPUTX_KSET_Q=4096 timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n2.log python tools/repro_kset.py 1 tm1 2>&1 | tail -3
echo "== ncu KSET_Q=32"; GPUTX_KSET_Q=32 timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n2.log python tools/repro_kset.py 1 tm1 2>&1 | tail -3
echo "== ncu cluster 2"; GPUTX_KSET_CLUSTER=2 timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n3.log python tools/repro_kset.py 1 tm1 2>&1 | tail -3
echo "== ncu cluster 16"; GPUTX_KSET_CLUSTER=16 GPUTX_DEBUG=1 timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n4.log python tools/repro_kset.py 1 tm1 2>&1 | tail -3
echo "== ncu grid 8"; GPUTX_KSET_GRID=8 timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n5.log python tools/repro_kset.py 1 tm1 2>&1 | tail -3
echo "== ncu grid 16"; GPUTX_KSET_GRID=16 timeout 300 ncu --metrics gpu__time_duration.sum -c 2000 --log-file /tmp/n6.log python tools/repro_kset.py 1 tm1 2>&1 | tail -3
