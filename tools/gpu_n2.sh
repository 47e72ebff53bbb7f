# sharded bench path with 2 ranks on one GPU (gloo exchange): functional check
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
i=0
for o in "" part tpl auto; do
  i=$((i+1))
  GPUTX_DIST_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29600+i)) bench.py --gpus 2 --steps 2 --warmup 3 --workload ${1:-tpcc} --no-cpu-baseline --others "$o" > gpurun_out/n2_$i.json 2> gpurun_out/n2_$i.err
  echo "others=[$o] rc=$? $(grep -o 'GputxError.*' gpurun_out/n2_$i.err | head -1)"
done
