# parity tests + a bench line + launch list
set -x
mkdir -p gpurun_out/q
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/q/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q/pytest_gpu.log
timeout 600 python bench.py ${BENCH_ARGS:---no-cpu-baseline} > gpurun_out/q/bench.jsonl 2> gpurun_out/q/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/q/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q/bench_ncu.log 2>&1
