# closing check at HEAD: full GPU suite, smoke, default bench line, cfg1 line
T=${1:-r4q}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
timeout 600 python bench.py > gpurun_out/${T}_cfg2.json 2> gpurun_out/${T}_cfg2.err
timeout 600 python bench.py --config cfg1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_cfg1.json 2> gpurun_out/${T}_cfg1.err
tail -2 gpurun_out/${T}_tests.log; tail -2 gpurun_out/${T}_smoke.log
for c in cfg2 cfg1; do python -c "
import json; d=json.loads(open('gpurun_out/${T}_$c.json').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['value'], d['e2e']['value'], d['roofline']['frac'], d['simt_calls'], {k: (round(v['avg_ms'],4), round(v['frac'],3)) for k,v in d['kernels'].items()})"; done
