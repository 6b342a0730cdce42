# K4 work-item cap for one large world: 64 (in-tree) vs 96 / 56 / 48
VARS="- cs96 cs56 cs48" CFGS="c5" timeout 1500 bash tools/ab.sh 2>&1
