#!/bin/bash
# The reference solver's own full runs on the GPU box's host cores next to the
# B200 (profiles/r02_*vs_reference*.json).  Each step is long on the CPU
# (the 70k solve ~45 min, the 25k tracking ~20-30 min): run them one per call.
# usage: O=gpurun_out/vs bash scripts/gpu_vs_reference.sh <70k|25k|2868|9241|13659>
O=${O:-gpurun_out/vs}
mkdir -p $O
case "$1" in
  70k)   timeout 3300 python scripts/converge_vs_reference.py case_ACTIVSg70k case_ACTIVSg70k 1e-4 $O/r02_converge_vs_reference_70k.json ;;
  25k)   timeout 3300 python scripts/track_vs_reference.py case_ACTIVSg25k 30 case_ACTIVSg25k 30 $O/r02_track_25k_vs_reference.json ;;
  2868)  timeout 1500 python scripts/converge_vs_reference.py case2868rte 1000:10000 1e-4 $O/r02_converge_vs_reference_case2868rte.json ;;
  9241)  timeout 1500 python scripts/converge_vs_reference.py case9241pegase 300:3000 1e-4 $O/r02_converge_vs_reference_case9241pegase.json ;;
  13659) timeout 1500 python scripts/converge_vs_reference.py case13659pegase 1000:10000 1e-4 $O/r02_converge_vs_reference_case13659pegase.json ;;
esac > $O/vs_$1.log 2>&1
