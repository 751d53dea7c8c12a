# ncu --set full of the per-iteration kernels at inner iteration 10 (70k-shaped).
set -x
mkdir -p gpurun_out/ncu
for k in ${KERNELS:-lane_kernel tile_kernel bus_warp_kernel}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 10 -c 1 \
      -o gpurun_out/ncu/$k -f python scripts/ncu_target.py case_ACTIVSg70k 12 > gpurun_out/ncu/$k.log 2>&1
done
