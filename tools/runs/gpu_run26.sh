VG_LIB_VARIANT=fsc timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_slab.py -m gpu -q -p no:cacheprovider -x > gpurun_out/gpu_tests_fsc.log 2>&1; echo "tests rc $?"
grep -E "passed|failed|FAILED|Error" gpurun_out/gpu_tests_fsc.log | tail -5
VARS="- fsc" CFGS="c5 c4" timeout 1200 bash tools/ab.sh 2>&1
