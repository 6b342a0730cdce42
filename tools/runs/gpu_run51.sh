# K4: degree-5 atan polynomial (1.7e-6 rad) vs degree 6, on the current kernel
VG_LIB_VARIANT=atan5 timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t51.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/t51.log
VARS="- atan5" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
