# K4: run windows per pass WN = 4 (in-tree, compare-count lane offsets) vs 5 vs 2
VG_LIB_VARIANT=w5 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "c5 or edge or c2 or c3 or rim" > gpurun_out/t57.log 2>&1; echo "w5 tests rc $?"; tail -1 gpurun_out/t57.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t57b.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t57b.log
VARS="- w5 w2" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
