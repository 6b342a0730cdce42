# K4: run windows of two warp-iterations in one pass (W2) vs one per iteration (w20)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t55.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t55.log
VARS="- w20" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
