#!/bin/bash
# round 2, pass m: bus-major row storage — gpu tests, bench window, full solve
O=gpurun_out/m
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=900 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python scripts/converge_time.py > $O/conv_default.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge --no-track > $O/bench_default.json 2>&1
echo done
