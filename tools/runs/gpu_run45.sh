# K4 with SCANSELF: 8-byte entries for replica worlds too (re8) / 16-byte everywhere (e8off)
VARS="- re8 e8off" CFGS="c5 c4" timeout 2400 bash tools/ab.sh 2>&1
