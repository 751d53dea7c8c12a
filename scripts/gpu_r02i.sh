#!/bin/bash
# round 2, pass i: branch-schedule sweeps on the full 70k solve (runtime knobs
# and the tile width), results never depend on them
O=gpurun_out/i
mkdir -p $O
timeout 1500 python scripts/sched_sweep.py case_ACTIVSg70k case_ACTIVSg70k '[{}, {"lane_budget": 2}, {"lane_budget": 8}, {"lane_cap": 8}, {"lane_cap": 32}, {"tile_budget": 24}, {"tile_budget": 96}, {"tile_budget": 0}]' > $O/sched_70k.jsonl 2>&1
for v in tile4 tile16 order; do GRIDADMM_LIB=paper_2110_06879_b200/libgridadmm_$v.so timeout 300 python scripts/converge_time.py > $O/conv_$v.json 2>&1; done
timeout 300 python scripts/converge_time.py > $O/conv_default.json 2>&1
timeout 900 python scripts/sched_sweep.py case_ACTIVSg25k case_ACTIVSg25k '[{}, {"lane_budget": 2}, {"lane_cap": 8}, {"lane_cap": 32}, {"tile_budget": 24}, {"tile_budget": 96}]' > $O/sched_25k.jsonl 2>&1
echo done
