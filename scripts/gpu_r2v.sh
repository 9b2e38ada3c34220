# host overhead of the per-rank step at 8-GPU strong-scaling size (D = 32 of 256), thread mesh and one-rank NCCL
timeout 300 python scripts/host_overhead.py 32 > gpurun_out/r2v_host_thread.txt 2>&1
BACKEND=nccl timeout 300 python scripts/host_overhead.py 32 > gpurun_out/r2v_host_nccl.txt 2>&1
timeout 300 python scripts/host_overhead.py 256 > gpurun_out/r2v_host_256.txt 2>&1
head -45 gpurun_out/r2v_host_thread.txt; head -3 gpurun_out/r2v_host_nccl.txt; head -45 gpurun_out/r2v_host_nccl.txt | tail -30; head -2 gpurun_out/r2v_host_256.txt
