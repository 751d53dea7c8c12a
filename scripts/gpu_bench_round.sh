# Round-end style evidence: full bench line, reference arm, launch list with dram bytes.
set -x
mkdir -p gpurun_out/r
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r/nvsmi.txt 2>&1
timeout 900 python bench.py > gpurun_out/r/bench.jsonl 2> gpurun_out/r/bench.err
timeout 600 python bench.py --impl reference >> gpurun_out/r/bench.jsonl 2>> gpurun_out/r/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-converge > gpurun_out/r/bench_ncu.log 2>&1
