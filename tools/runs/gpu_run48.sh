# K4: both queries' last partial batches in one pass (MIXTAIL) + three-limb reward reduction,
# vs without MIXTAIL (mt0) vs the previous commit (prev2)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t48.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t48.log
VARS="- mt0 prev2" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
