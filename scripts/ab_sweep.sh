# A/B of library variants: bench window + full 70k solve. VARIANTS="base nosb"
mkdir -p gpurun_out/ab
for v in ${VARIANTS:-base}; do
  lib=$PWD/paper_2110_06879_b200/libgridadmm_$v.so; [ $v = base ] && lib=$PWD/paper_2110_06879_b200/libgridadmm.so
  GRIDADMM_LIB=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v bench', round(d['value'],1), {k: round(v['ms_total']/30*1e3,1) for k,v in d['kernels'].items()})" > gpurun_out/ab/bench_$v.txt 2>&1
  [ -n "$SOLVE" ] && GRIDADMM_LIB=$lib timeout 600 python scripts/probe_solve_profile.py case_ACTIVSg70k 100 1e4 1000 20 /tmp/p.csv > gpurun_out/ab/solve_$v.txt 2>&1
done
