# staged bin: pass 1 split into integrate-all-rounds then match/rank rounds (SPLIT1)
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "binning or staged or c4 or determin" > gpurun_out/t43.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t43.log
VARS="- sp0" CFGS="c4" timeout 1500 bash tools/ab.sh 2>&1
