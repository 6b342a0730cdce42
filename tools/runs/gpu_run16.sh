VARS="- mb9 mb8c100" CFGS="c5 c4" timeout 1200 bash tools/ab.sh > gpurun_out/ab_r2m.txt 2>&1
cat gpurun_out/ab_r2m.txt
