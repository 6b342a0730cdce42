VG_LIB_VARIANT=q4 timeout 600 python -m pytest tests/test_policy.py tests/test_gpu_rollout.py -m gpu -q -p no:cacheprovider > gpurun_out/q4_tests.log 2>&1; echo "q4 tests rc $?"; tail -2 gpurun_out/q4_tests.log
VARS="- q4" timeout 900 bash tools/policy_bench.sh 2>&1
