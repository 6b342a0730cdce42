# K4: run windows of four warp-iterations per pass (w4) vs two (in-tree)
VG_LIB_VARIANT=w4 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t56.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t56.log
VARS="- w4" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
