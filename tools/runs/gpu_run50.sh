# c5 K2: one-CTA scan (18,496 counts staged in 74 KB of shared memory) vs the two-kernel scan
VARS="- scan1" CFGS="c5" timeout 1200 bash tools/ab.sh 2>&1
