timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "binning_paths or staged or c4 or 64bit" > gpurun_out/gpu_tests_r2k.log 2>&1; echo "tests rc $?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests_r2k.log | tail -12
for k in 1 2; do for m in 1 2 0; do
VG_RB_STAGED=$m timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-policy --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('mode $m', d['ms_per_step'], {k:v['ms'] for k,v in d['stages'].items()})"
done; done
