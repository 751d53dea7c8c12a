set -x
mkdir -p gpurun_out/tail
GRIDADMM_LIB=$PWD/paper_2110_06879_b200/libgridadmm_stats.so timeout 600 python scripts/probe_tail.py case_ACTIVSg70k 31 > gpurun_out/tail/probe.txt 2>&1
for T in 8 16 32; do
  GRIDADMM_LIB=$PWD/paper_2110_06879_b200/libgridadmm_t$T.so timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/tail/bench_t$T.jsonl 2>&1
done
