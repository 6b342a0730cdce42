# K4: the self pair excluded at the candidate test (slot != own index) instead of in the
# pair pass / emit (SCANSELF)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t44.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t44.log
VARS="- ss0" CFGS="c5 c4 c3" timeout 2400 bash tools/ab.sh 2>&1
