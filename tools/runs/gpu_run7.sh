bash tools/policy_bench.sh 2>&1 | tee gpurun_out/policy_ab_r2g.txt
for v in tanh1 tanh2; do VG_LIB_VARIANT=$v timeout 600 python -m pytest tests/test_policy.py tests/test_gpu_rollout.py -m gpu -q -p no:cacheprovider 2>&1 | tail -4; done
