# K4: the first 2 (in-tree) / 1 / 3 candidate halves of a chunk without the skip test
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t73.log 2>&1; echo "tests rc $?"; tail -n1 gpurun_out/t73.log
VARS="- hf1 hf3" CFGS="c5 c4" timeout 1500 bash tools/ab.sh 2>&1
