timeout 600 python -m pytest tests/test_gpu_comm.py -q -x > gpurun_out/r2d_comm.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_comm.log
NCCL_DEBUG=WARN timeout 200 python scripts/nccl_dup_probe.py > gpurun_out/r2d_dup.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_dup.log
tail -30 gpurun_out/r2d_comm.log; tail -20 gpurun_out/r2d_dup.log
