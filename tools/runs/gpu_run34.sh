# staged bin: actions preloaded (APRE) / dynamic pass-3 items (DYN3) — parity, then A/B on c4
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "binning or staged or c4 or determin" > gpurun_out/t34.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/t34.log
VARS="- base apre dyn3" CFGS="c4" timeout 1500 bash tools/ab.sh 2>&1
