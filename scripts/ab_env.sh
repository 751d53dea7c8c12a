#!/bin/bash
# A/B of a runtime switch on one build: O=<dir> L=<lib> VAR=<env var> bash scripts/ab_env.sh v1 v2 ...
# (bench window + full 70k solve per value, alternating)
O=${O:-gpurun_out/abe}; mkdir -p $O
L=${L:-paper_2110_06879_b200/libgridadmm.so}
for v in "$@"; do
  env GRIDADMM_LIB=$L $VAR=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge --no-track > $O/bench_$v.json 2>&1
done
for v in "$@" "$@"; do
  env GRIDADMM_LIB=$L $VAR=$v timeout 400 python scripts/converge_time.py ${SHAPE:-case_ACTIVSg70k} ${PRESET:-case_ACTIVSg70k} 1 >> $O/conv_$v.json 2>&1
done
