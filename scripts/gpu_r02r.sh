#!/bin/bash
O=gpurun_out/r
mkdir -p $O
timeout 900 python -m pytest tests/test_cli_reference.py tests/test_capi_reference.py -m gpu -q > $O/pytest_cli.log 2>&1; echo "rc=$?" >> $O/pytest_cli.log
GRIDADMM_LIB=paper_2110_06879_b200/libgridadmm_stats.so timeout 600 python scripts/probe_path_stats.py case_ACTIVSg70k case_ACTIVSg70k 5 20 > $O/stats_70k_5.json 2>&1
GRIDADMM_LIB=paper_2110_06879_b200/libgridadmm_stats.so timeout 600 python scripts/probe_path_stats.py case_ACTIVSg70k case_ACTIVSg70k 3000 20 > $O/stats_70k_3000.json 2>&1
timeout 1500 python scripts/sched_sweep.py case_ACTIVSg70k case_ACTIVSg70k '[{}, {"lane_budget": 2}, {"lane_budget": 6}, {"lane_cap": 12}, {"lane_cap": 24}, {"tile_budget": 24}, {"tile_budget": 96}, {"tile_budget": 0}]' > $O/sched_70k.jsonl 2>&1
echo done
