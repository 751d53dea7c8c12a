#!/bin/bash
# round 2: the reference's own full solves on the box's host cores next to the
# B200 runs of the same cases (time-to-converge, warm-start tracking)
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt
timeout 600 python scripts/synth_explore.py '[{"shape":"case2868rte","rho":[50,5000]},{"shape":"case2868rte","rho":[100,10000]},{"shape":"case2868rte","rho":[300,3000]},{"shape":"case2868rte","rho":[1000,10000]},{"shape":"case9241pegase","rho":[50,5000]},{"shape":"case13659pegase","rho":[50,5000]},{"shape":"case_ACTIVSg25k","rho":[3000,30000]},{"shape":"case_ACTIVSg70k","rho":[30000,300000]}]' > gpurun_out/explore.jsonl 2> gpurun_out/explore.err
timeout 3000 python scripts/converge_vs_reference.py case_ACTIVSg70k case_ACTIVSg70k 1e-4 gpurun_out/r02_converge_vs_reference_70k.json > gpurun_out/cvr70k.log 2>&1
timeout 2400 python scripts/track_vs_reference.py case_ACTIVSg25k 30 case_ACTIVSg25k 30 gpurun_out/r02_track_25k_vs_reference.json > gpurun_out/tvr25k.log 2>&1
timeout 1500 python scripts/converge_vs_reference.py case2868rte 50:5000 1e-4 gpurun_out/r02_converge_vs_reference_case2868rte.json > gpurun_out/cvr_case2868rte.log 2>&1
for s in case9241pegase case13659pegase; do
  timeout 1500 python scripts/converge_vs_reference.py $s $s 1e-4 gpurun_out/r02_converge_vs_reference_$s.json > gpurun_out/cvr_$s.log 2>&1
done
echo done
