#!/bin/bash
# A/B of build variants on the bench window (device value + kernel split):
# O=<out dir> bash scripts/ab_bench.sh v1 v2 ...   ("default" = libgridadmm.so)
O=${O:-gpurun_out/abb}
mkdir -p $O
for v in "$@"; do
  L=paper_2110_06879_b200/libgridadmm_$v.so; [ $v = default ] && L=paper_2110_06879_b200/libgridadmm.so
  GRIDADMM_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge --no-track > $O/bench_$v.json 2>&1
done
