#!/bin/bash
# A/B of build variants on the full 70k-shaped solve: O=<out dir> bash scripts/ab_converge.sh v1 v2 ...
# (variant v = paper_2110_06879_b200/libgridadmm_v.so; "default" = libgridadmm.so)
O=${O:-gpurun_out/ab}
mkdir -p $O
for v in "$@"; do
  L=paper_2110_06879_b200/libgridadmm_$v.so; [ $v = default ] && L=paper_2110_06879_b200/libgridadmm.so
  GRIDADMM_LIB=$L timeout 400 python scripts/converge_time.py ${SHAPE:-case_ACTIVSg70k} ${PRESET:-case_ACTIVSg70k} 1 >> $O/conv_$v.json 2>&1
done
echo done
