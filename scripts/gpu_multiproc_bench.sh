# Dry run of the driver's N-GPU bench path on a one-GPU box: torchrun with 2 ranks
# sharing the GPU over gloo (DP_MESH_BACKEND=gloo-cuda).  Timings are meaningless;
# this checks the multi-process orchestration end to end (no crash / deadlock, JSON).
export DP_MESH_BACKEND=gloo-cuda
for c in cfg2 cfg3 cfg4 cfg5 cfg1; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29611 bench.py --gpus 2 --steps 2 --warmup 3 --config $c --no-cpu-baseline \
      > gpurun_out/mp_$c.json 2> gpurun_out/mp_$c.err
  echo "$c rc=$?"; tail -c 300 gpurun_out/mp_$c.json; echo
done
