#!/bin/bash
# round 2, pass d: rho sweep for the pegase-shaped grids (GPU only, seconds
# each), then the reference's own runs on the box's host cores: 25k warm-start
# tracking (first 10 of the 30 snapshots on the CPU; all 30 on the GPU) and
# the 2868-shaped full solve
O=gpurun_out/d
mkdir -p $O
for v in noskip default; do
  L=paper_2110_06879_b200/libgridadmm_$v.so; [ $v = default ] && L=paper_2110_06879_b200/libgridadmm.so
  GRIDADMM_LIB=$L timeout 300 python scripts/converge_time.py > $O/conv_$v.json 2>&1
  GRIDADMM_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge --no-track > $O/bench_$v.json 2>&1
done
GRIDADMM_LIB=paper_2110_06879_b200/libgridadmm_stats.so timeout 600 python scripts/probe_path_stats.py case_ACTIVSg70k case_ACTIVSg70k 5 20 > $O/stats_70k_5.json 2>&1
GRIDADMM_LIB=paper_2110_06879_b200/libgridadmm_stats.so timeout 600 python scripts/probe_path_stats.py case_ACTIVSg70k case_ACTIVSg70k 3000 20 > $O/stats_70k_3000.json 2>&1
timeout 900 python scripts/synth_explore.py '[{"shape":"case9241pegase","rho":[100,10000]},{"shape":"case9241pegase","rho":[300,3000]},{"shape":"case9241pegase","rho":[1000,10000]},{"shape":"case9241pegase","rho":[3000,30000]},{"shape":"case13659pegase","rho":[100,10000]},{"shape":"case13659pegase","rho":[1000,10000]},{"shape":"case13659pegase","rho":[3000,30000]}]' > $O/explore_pegase.jsonl 2> $O/explore.err
timeout 600 python scripts/converge_vs_reference.py case2868rte 1000:10000 1e-4 $O/r02_converge_vs_reference_case2868rte.json > $O/cvr_2868.log 2>&1
timeout 2900 python scripts/track_vs_reference.py case_ACTIVSg25k 30 case_ACTIVSg25k 10 $O/r02_track_25k_vs_reference.json > $O/tvr25k.log 2>&1
echo done
