#!/bin/bash
# compute-sanitizer memcheck / racecheck / initcheck of the branch, bus and
# extraction kernels on the 2868-shaped grid with every hand-off forced
# (scripts/sanitize_target.py)
O=${O:-gpurun_out/san}
mkdir -p $O
for tool in memcheck racecheck initcheck; do
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_target.py 2 > $O/sanitize_$tool.log 2>&1; echo "rc=$?" >> $O/sanitize_$tool.log
done
