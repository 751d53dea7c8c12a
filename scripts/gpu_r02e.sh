#!/bin/bash
# round 2, pass e: gpu tests on the current build, pre-screen A/B on the full
# 70k solve, bench, path statistics, launch list + ncu captures, sanitizers
O=gpurun_out/e
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for v in noskip default; do
  L=paper_2110_06879_b200/libgridadmm_$v.so; [ $v = default ] && L=paper_2110_06879_b200/libgridadmm.so
  GRIDADMM_LIB=$L timeout 300 python scripts/converge_time.py > $O/conv_$v.json 2>&1
  GRIDADMM_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge --no-track > $O/bench_$v.json 2>&1
done
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
GRIDADMM_LIB=paper_2110_06879_b200/libgridadmm_stats.so timeout 600 python scripts/probe_path_stats.py case_ACTIVSg70k case_ACTIVSg70k 5 20 > $O/stats_70k_5.json 2>&1
timeout 600 python scripts/probe_solve_profile.py case_ACTIVSg70k case_ACTIVSg70k $O/solve_profile_70k.json > $O/solve_profile.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-converge --no-track > $O/launches.log 2>&1
O=gpurun_out/e/ncu bash scripts/gpu_ncu.sh > gpurun_out/e/ncu.log 2>&1
O=gpurun_out/e/san SAN_TIMEOUT=600 bash scripts/gpu_sanitize.sh
echo done
