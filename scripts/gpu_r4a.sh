# session-4 entry check: GPU suite, smoke and cfg1/cfg2 bench lines at HEAD
T=${1:-r4a}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${T}_cfg2.json 2> gpurun_out/${T}_cfg2.err
timeout 600 python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_cfg1.json 2> gpurun_out/${T}_cfg1.err
tail -3 gpurun_out/${T}_tests.log; tail -1 gpurun_out/${T}_smoke.log
