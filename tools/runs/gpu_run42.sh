# K4: LDPRED on; 8-byte entries for single worlds (c5, slab), 16-byte for replica worlds (c4)
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t42.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t42.log
VARS="- e8off" CFGS="c5 c4 c2" timeout 2400 bash tools/ab.sh 2>&1
timeout 300 python tools/slab_timing.py 2>&1 | tail -3
