# K4 drain batches addressed as lane offset + (head mod ring) (rb: VG_SENSE_RINGB=1) vs in-tree
python paper_2207_03945_b200/_build.py --force > gpurun_out/build_93.log 2>&1
VARS="rb -" CFGS="c5 c4" bash tools/ab.sh > gpurun_out/ab_93.txt 2>&1; cat gpurun_out/ab_93.txt
