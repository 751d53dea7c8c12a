#!/bin/bash
O=gpurun_out/s
mkdir -p $O
for v in lb64 lb256 default; do
  L=paper_2110_06879_b200/libgridadmm_$v.so; [ $v = default ] && L=paper_2110_06879_b200/libgridadmm.so
  GRIDADMM_LIB=$L timeout 300 python scripts/converge_time.py > $O/conv_$v.json 2>&1
done
echo done
