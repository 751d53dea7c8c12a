#!/bin/bash
# bus kernel threads-per-bus A/B: 70k bench window + 2868 full-solve phase profile
O=${O:-gpurun_out/tpb}; mkdir -p $O
for v in "$@"; do
  L=paper_2110_06879_b200/libgridadmm_$v.so; [ $v = default ] && L=paper_2110_06879_b200/libgridadmm.so
  GRIDADMM_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge --no-track > $O/bench_$v.json 2>&1
  GRIDADMM_LIB=$L timeout 300 python scripts/probe_solve_profile.py case2868rte 1000:10000 $O/prof2868_$v.json > $O/prof2868_$v.log 2>&1
done
