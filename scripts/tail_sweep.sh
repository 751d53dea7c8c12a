mkdir -p gpurun_out/tail2
for tn in ${TNS:-2 4 8}; do
  GRIDADMM_TAIL_NUM=$tn timeout 300 python scripts/probe_solve_profile.py case_ACTIVSg70k 100 1e4 1000 4 /tmp/p.csv 2>&1 | sed -n 2p | sed "s/^/tn=$tn /" >> gpurun_out/tail2/sweep.txt
  GRIDADMM_TAIL_NUM=$tn timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tn=$tn bench', round(d['value'],1), {k: round(v['ms_total']/30*1e3,1) for k,v in d['kernels'].items()})" >> gpurun_out/tail2/sweep.txt
done
