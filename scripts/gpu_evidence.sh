#!/bin/bash
# The evidence pass of a build (one GPU): gpu tests, bench (both arms), solve
# profile, launch list, ncu captures + FP64 counts, compute-sanitizer.
# usage (on the GPU box): O=gpurun_out/ev bash scripts/gpu_evidence.sh
O=${O:-gpurun_out/ev}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 600 python scripts/probe_solve_profile.py case_ACTIVSg70k case_ACTIVSg70k $O/solve_profile_70k.json > $O/solve_profile.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-converge --no-track > $O/launches.log 2>&1
O=$O/ncu bash scripts/gpu_ncu.sh > $O/ncu.log 2>&1
O=$O/san SAN_TIMEOUT=600 bash scripts/gpu_sanitize.sh
echo done
