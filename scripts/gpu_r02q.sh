#!/bin/bash
# round 2, pass q: the reference's tracking run over all 30 snapshots on the
# box's host cores next to the B200; final-build GPU times of the smaller shapes
O=gpurun_out/q
mkdir -p $O
timeout 300 python scripts/converge_time.py case9241pegase 300:3000 2 > $O/conv_9241_gpu.json 2>&1
timeout 300 python scripts/converge_time.py case13659pegase 1000:10000 2 > $O/conv_13659_gpu.json 2>&1
timeout 300 python scripts/converge_time.py case2868rte 1000:10000 2 > $O/conv_2868_gpu.json 2>&1
timeout 3000 python scripts/track_vs_reference.py case_ACTIVSg25k 30 case_ACTIVSg25k 30 $O/r02_track_25k_vs_reference_30.json > $O/tvr25k_30.log 2>&1
echo done
