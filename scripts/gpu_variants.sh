# time library variants on the bench workload: VARIANTS="L3T3 L4T4 ..."
mkdir -p gpurun_out/var
for v in base $VARIANTS; do
  lib=$PWD/paper_2110_06879_b200/libgridadmm_$v.so; [ $v = base ] && lib=$PWD/paper_2110_06879_b200/libgridadmm.so
  GRIDADMM_LIB=$lib timeout 600 python bench.py --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/var/$v.jsonl 2>&1
done
