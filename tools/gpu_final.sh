# round-end evidence: full GPU tests, smoke, bench lines for every workload, reference
# arm, ncu launch list of the default bench, ncu --set full of the headline kernels
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/final
O=gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/nvsmi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in tm1 tm1_uniform tpcb tpcb_add tpcb_hot_add tpcb_tiny tpcc tpcc_add; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_tm1.json 2>&1
# the sharded N=2 path end to end (two ranks on this one GPU, gloo all-to-all: a functional
# check only -- the numbers of two ranks sharing one GPU mean nothing)
for w in tpcc tpcb; do
GPUTX_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --workload $w --no-cpu-baseline > $O/bench_n2_$w.json 2> $O/bench_n2_$w.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_tm1.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launches_tm1.log 2>&1
for k in kset_exec rank_stream rs_pass group_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 -o $O/full_tm1_$k \
    python bench.py --steps 1 --warmup 3 --others "" --no-cpu-baseline > $O/ncu_tm1_$k.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rank_kernel" -s 1 -c 1 -o $O/full_tpcb_add_rank_kernel \
    python bench.py --workload tpcb_add --steps 1 --warmup 3 --others "" --no-cpu-baseline > $O/ncu_tpcb_add.log 2>&1
ls $O
