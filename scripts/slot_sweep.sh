mkdir -p gpurun_out/slot
for sm in ${SMS:-1 2 4}; do
  GRIDADMM_SLOT_MULT=$sm timeout 300 python scripts/probe_solve_profile.py case_ACTIVSg70k 100 1e4 1000 4 /tmp/p.csv 2>&1 | sed -n 2p | sed "s/^/sm=$sm /" >> gpurun_out/slot/sweep.txt
  GRIDADMM_SLOT_MULT=$sm timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sm=$sm bench', round(d['value'],1), {k: round(v['ms_total']/30*1e3,1) for k,v in d['kernels'].items()})" >> gpurun_out/slot/sweep.txt
done
