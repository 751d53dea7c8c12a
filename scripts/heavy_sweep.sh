mkdir -p gpurun_out/heavy
for hs in ${HS:-0 400}; do
  GRIDADMM_HEAVY_STEPS=$hs timeout 600 python scripts/probe_solve_profile.py case_ACTIVSg70k 100 1e4 1000 20 /tmp/p.csv > gpurun_out/heavy/solve_$hs.txt 2>&1
  GRIDADMM_HEAVY_STEPS=$hs timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hs=$hs bench', round(d['value'],1), {k: round(v['ms_total']/30*1e3,1) for k,v in d['kernels'].items()})" > gpurun_out/heavy/bench_$hs.txt 2>&1
done
