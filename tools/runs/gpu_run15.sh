timeout 900 python -m pytest tests/test_slab.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "slab or sense_columns or c5_full" > gpurun_out/gpu_tests_r2l.log 2>&1; echo "tests rc $?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests_r2l.log | tail -12
timeout 300 python tools/slab_timing.py > gpurun_out/slab_timing_r2l.txt 2>&1; tail -3 gpurun_out/slab_timing_r2l.txt
