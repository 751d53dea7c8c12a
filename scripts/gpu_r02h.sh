#!/bin/bash
# round 2, pass h: bus-kernel occupancy A/B (staging rows x min blocks per SM)
# and the 2868-shaped full-solve parity test
O=gpurun_out/h
mkdir -p $O
for v in b12m6 b8m8 b10m7; do
  GRIDADMM_LIB=paper_2110_06879_b200/libgridadmm_$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge --no-track > $O/bench_$v.json 2>&1
done
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge --no-track > $O/bench_default.json 2>&1
timeout 900 python -m pytest tests/test_gpu_acceptance.py -m gpu -q -k 2868 > $O/pytest_2868.log 2>&1; echo "rc=$?" >> $O/pytest_2868.log
echo done
