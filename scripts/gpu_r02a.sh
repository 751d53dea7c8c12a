#!/bin/bash
# round-2 first GPU pass: gpu tests, bench (device window + e2e + converge), 25k tracking probe
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-track --cpu-steps 5 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
timeout 1200 python scripts/track_bench.py case_ACTIVSg25k 6 > gpurun_out/track25k_6.json 2> gpurun_out/track25k_6.err
echo done
