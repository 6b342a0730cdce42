VARS="p0s0 p0s1 p1s0 - p1s1m7 p0s1m7" CFGS="c5" timeout 1200 bash tools/ab.sh > gpurun_out/ab_r2c.txt 2>&1
cat gpurun_out/ab_r2c.txt
