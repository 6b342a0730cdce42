# K4: the second warp sync per chunk taken only when the chunk's pushes could wrap onto
# entries the drain read (warp-uniform check) — E8 four halves vs two / three vs 16-byte
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t40.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t40.log
VARS="- e8h2 e8h3 e8off" CFGS="c5 c4 c3" timeout 2400 bash tools/ab.sh 2>&1
