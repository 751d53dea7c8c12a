# ncu --set full of the per-iteration kernels at inner iteration 10 of the
# 70k-shaped cold start, plus executed FP64 instruction counts of the branch
# kernels over iterations 1-12 (the roofline cross-check of the census).
set -x
O=${O:-gpurun_out/ncu}
mkdir -p $O
# (the bus kernel unsplit, GRIDADMM_BUS_OVERLAP=0: one launch per iteration)
for k in ${KERNELS:-lane_kernel tile_kernel bus_block_kernel}; do
  ov=1; [ $k = bus_block_kernel ] && ov=0
  GRIDADMM_BUS_OVERLAP=$ov timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 10 -c 1 \
      -o $O/$k -f python scripts/ncu_target.py case_ACTIVSg70k 12 > $O/$k.log 2>&1
done
timeout 900 ncu --clock-control none --csv -k regex:"lane_kernel|tile_kernel|solo_kernel" \
    --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    python scripts/ncu_target.py case_ACTIVSg70k 12 > $O/fp64_counts.csv 2> $O/fp64_counts.err
