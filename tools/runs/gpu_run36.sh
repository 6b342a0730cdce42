# staged bin: pass-1 cell totals (CNT, one barrier fewer) / actions preloaded (APRE)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "binning or staged or c4 or determin" > gpurun_out/t36.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/t36.log
VARS="- cnt0 base" CFGS="c4" timeout 1500 bash tools/ab.sh 2>&1
