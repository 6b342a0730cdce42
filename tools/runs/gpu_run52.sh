# K4: ring drain two batches per iteration (DRAIN2) vs one (dr0)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t52.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t52.log
VARS="- dr0" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
