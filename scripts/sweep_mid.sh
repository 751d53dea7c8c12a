#!/bin/bash
# lane-phase hand-off knobs across grid sizes (full solves)
O=${O:-gpurun_out/mid}; mkdir -p $O
C='[{}, {"lane_budget": 1, "lane_cap": 1}, {"lane_budget": 1}, {"lane_cap": 4}]'
timeout 400 python scripts/sched_sweep.py case9241pegase 300:3000 "$C" > $O/sweep_9241.jsonl 2>&1
timeout 400 python scripts/sched_sweep.py case13659pegase 1000:10000 "$C" > $O/sweep_13659.jsonl 2>&1
timeout 600 python scripts/sched_sweep.py case_ACTIVSg25k case_ACTIVSg25k "$C" > $O/sweep_25k.jsonl 2>&1
