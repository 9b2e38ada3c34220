# round-2 measurement set: full GPU suite, smoke, every config's bench line, the reference arm,
# launch lists and ncu --set full captures (profiles/ + traffic.json keyed by the bench names)
T=r3a
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${T}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${T}_cfg2.json 2> gpurun_out/${T}_cfg2.err
for c in cfg1 cfg3 cfg4 cfg5; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_$c.json 2> gpurun_out/${T}_$c.err; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
# launch lists (cold, serialised)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/${T}_cfg2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/${T}_cfg1_launches.csv python bench.py --config cfg1 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/${T}_cfg4_launches.csv python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv --log-file gpurun_out/${T}_cfg3_launches.csv python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# full captures
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'conv_tc_kernel|conv_wgrad_t' -s 12 -c 6 -o gpurun_out/${T}_cfg2_conv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:'conv_tc_kernel|conv_wgrad_tc_kernel' -s 24 -c 12 -o gpurun_out/${T}_cfg4_conv python bench.py --config cfg4 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:'x3_split_act|conv_tc_kernel|conv_wgrad_ts' -s 15 -c 5 -o gpurun_out/${T}_cfg1_conv python bench.py --config cfg1 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
S=65536 timeout 900 ncu --set full --clock-control none -k regex:attn_.*_tc -c 2 -o gpurun_out/${T}_cfg3_attn python scripts/attn_prof.py > /dev/null 2>&1
grep -E "passed|failed" gpurun_out/${T}_tests.log | tail -2; tail -1 gpurun_out/${T}_smoke.log
python - <<'PY'
import json
for f in ("cfg2", "cfg1", "cfg3", "cfg4", "cfg5", "ref"):
    try:
        d = json.loads(open(f"gpurun_out/r3a_{f}.json").read().strip().splitlines()[-1])
        print(f, d.get("ms_per_step"), d.get("value"), d.get("clocks"), d.get("roofline", {}) and d["roofline"].get("frac"),
              {k: (round(v["avg_ms"], 4), round(v["frac"], 3)) for k, v in d.get("kernels", {}).items()})
    except Exception as e:
        print(f, "ERR", e)
PY
ls -la gpurun_out | grep r3a
