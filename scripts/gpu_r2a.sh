# round 2 step A: sharded conv on tcgen05 (layout fix) + the existing gpu suite
timeout 900 python -m pytest tests/test_gpu_tc_sharded.py -x -q > gpurun_out/r2a_tc.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_tc.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r2a_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r2a_smoke.log
tail -5 gpurun_out/r2a_tc.log; tail -5 gpurun_out/r2a_gpu.log; tail -3 gpurun_out/r2a_smoke.log
