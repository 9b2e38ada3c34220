# final numbers: default bench (cfg2) + every config + reference arm + smoke + tests
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final_cfg2.json 2> /dev/null
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 5 > gpurun_out/final_$c.json 2> /dev/null
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref_cfg2.json 2> /dev/null
tail -1 gpurun_out/final_pytest.log; tail -1 gpurun_out/final_smoke.log
