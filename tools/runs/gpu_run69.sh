# K4 emit: the four occupancy words as one vector store by lane 0 (OCC_V4) vs per-lane stores
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t69.log 2>&1; echo "tests rc $?"; tail -n1 gpurun_out/t69.log
VARS="- ov0" CFGS="c5 c4" timeout 1500 bash tools/ab.sh 2>&1
