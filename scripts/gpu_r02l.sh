#!/bin/bash
# round 2, pass l (final build): gpu tests, bench, solve profile, launch list,
# ncu captures + FP64 counts, sanitizers
O=gpurun_out/p
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python scripts/probe_solve_profile.py case_ACTIVSg70k case_ACTIVSg70k $O/solve_profile_70k.json > $O/solve_profile.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-converge --no-track > $O/launches.log 2>&1
O=gpurun_out/p/ncu bash scripts/gpu_ncu.sh > gpurun_out/p/ncu.log 2>&1
O=gpurun_out/p/san SAN_TIMEOUT=600 bash scripts/gpu_sanitize.sh
echo done
