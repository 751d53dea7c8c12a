#!/bin/bash
# schedule knobs on a small grid (2868-shaped), env-only knobs per process
O=${O:-gpurun_out/small2}; mkdir -p $O
C='[{}, {"lane_budget": 1, "lane_cap": 1}]'
for t in 2 8 32 1000; do
  GRIDADMM_TAIL_NUM=$t timeout 300 python scripts/sched_sweep.py case2868rte 1000:10000 "$C" | sed "s/^{/{\"tail_num\": $t, /" >> $O/sweep.jsonl 2>&1
done
