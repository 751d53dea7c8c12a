#!/bin/bash
# round 2, pass g: the reference's full solves of the pegase-shaped grids on
# the box's host cores next to the B200 (best-quality penalties of the sweep),
# and GPU-side refreshes of the 2868 solve and the 25k tracking run
O=gpurun_out/g
mkdir -p $O
timeout 300 python scripts/converge_time.py case2868rte 1000:10000 3 > $O/conv_2868_gpu.json 2>&1
timeout 1500 python scripts/converge_vs_reference.py case9241pegase 300:3000 1e-4 $O/r02_converge_vs_reference_case9241pegase.json > $O/cvr_9241.log 2>&1
timeout 1500 python scripts/converge_vs_reference.py case13659pegase 1000:10000 1e-4 $O/r02_converge_vs_reference_case13659pegase.json > $O/cvr_13659.log 2>&1
echo done
