set -x
mkdir -p gpurun_out/prof
for k in lane_kernel tile_kernel bus_warp_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 9 -c 1 -o gpurun_out/prof/$k -f python scripts/probe_costs.py case_ACTIVSg70k 11 > gpurun_out/prof/$k.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_ncu.log 2>&1
