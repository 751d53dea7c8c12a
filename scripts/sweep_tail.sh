mkdir -p gpurun_out/tail2
for t in 0 1 4 8 1000; do
  GRIDADMM_TAIL_NUM=$t timeout 300 python scripts/converge_time.py case_ACTIVSg70k case_ACTIVSg70k 1 | sed "s/^{/{\"tail_num\": $t, /" >> gpurun_out/tail2/sweep.jsonl 2>&1
done
GRIDADMM_TAIL_NUM=1000 GRIDADMM_TILE_BUDGET=0 timeout 300 python scripts/converge_time.py case_ACTIVSg70k case_ACTIVSg70k 1 | sed 's/^{/{"tail_num": 1000, "tile_budget": 0, /' >> gpurun_out/tail2/sweep.jsonl 2>&1
