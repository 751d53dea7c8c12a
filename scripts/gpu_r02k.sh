#!/bin/bash
# round 2, pass k: segment-wise Cauchy pre-screen (lane phase) vs none
O=gpurun_out/k
mkdir -p $O
for v in noskip default; do
  L=paper_2110_06879_b200/libgridadmm_$v.so; [ $v = default ] && L=paper_2110_06879_b200/libgridadmm.so
  GRIDADMM_LIB=$L timeout 300 python scripts/converge_time.py > $O/conv_$v.json 2>&1
  GRIDADMM_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge --no-track > $O/bench_$v.json 2>&1
done
GRIDADMM_LIB=paper_2110_06879_b200/libgridadmm_stats.so timeout 600 python scripts/probe_path_stats.py case_ACTIVSg70k case_ACTIVSg70k 5 20 > $O/stats_70k_5.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lane_kernel -s 10 -c 1 -o $O/lane_kernel -f python scripts/ncu_target.py case_ACTIVSg70k 12 > $O/ncu_lane.log 2>&1
echo done
