#!/bin/bash
# round 2, pass j: fused generator projection with hoisted loads (default) vs
# the separate generator kernel, tile widths 2 / 4 / 8; gpu tests on the
# default build
O=gpurun_out/j
mkdir -p $O
for v in genk tile2 tile4 default; do
  L=paper_2110_06879_b200/libgridadmm_$v.so; [ $v = default ] && L=paper_2110_06879_b200/libgridadmm.so
  GRIDADMM_LIB=$L timeout 300 python scripts/converge_time.py > $O/conv_$v.json 2>&1
  GRIDADMM_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge --no-track > $O/bench_$v.json 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
echo done
