mkdir -p gpurun_out/tb
for tb in ${TBS:-8 16 48}; do
  GRIDADMM_TILE_BUDGET=$tb timeout 300 python scripts/probe_solve_profile.py case_ACTIVSg70k 100 1e4 1000 20 /tmp/p.csv 2>&1 | sed -n 1,2p | sed "s/^/tb=$tb /" >> gpurun_out/tb/sweep.txt
  GRIDADMM_TILE_BUDGET=$tb timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tb=$tb bench', round(d['value'],1), {k: round(v['ms_total']/30*1e3,1) for k,v in d['kernels'].items()})" >> gpurun_out/tb/sweep.txt
done
