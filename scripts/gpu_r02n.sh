#!/bin/bash
O=gpurun_out/n
mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bus_block_kernel -s 10 -c 1 -o $O/bus_block_kernel -f python scripts/ncu_target.py case_ACTIVSg70k 12 > $O/ncu_bus.log 2>&1
echo done
