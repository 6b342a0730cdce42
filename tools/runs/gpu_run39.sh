# K4 E8: four halves with the second warp sync the ring bound requires (carried + 2 x 32 HV
# > 256) vs three / two halves (no second sync) vs 16-byte entries
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "c5 or coincident or edge or dyadic or rim" > gpurun_out/t39.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t39.log
VARS="- e8h3 e8h2 e8off" CFGS="c5 c4" timeout 2000 bash tools/ab.sh 2>&1
