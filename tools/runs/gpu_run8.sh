timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_r2h.log 2>&1; echo "tests rc $?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests_r2h.log | tail -12
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_r2h.json 2> gpurun_out/bench_c4_r2h.err; echo "c4 rc $?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c5_r2h.json 2> gpurun_out/bench_c5_r2h.err; echo "c5 rc $?"
python - <<'PY'
import json
for f in ['gpurun_out/bench_c4_r2h.json','gpurun_out/bench_c5_r2h.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d['ms_per_step'], d['value'], d['roofline']['frac'], d['policy']['ms'] if d.get('policy') else None)
        for k,v in d['stages'].items(): print('  ',k,v['ms'],v['GBps'])
    except Exception as e: print(f, e)
PY
