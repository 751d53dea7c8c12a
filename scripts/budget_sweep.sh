# lane cap sweep on a truncated 70k-shaped solve (rho 100/1e4, 4 outer x 1000 inner)
# plus the bench window (preset rho)
mkdir -p gpurun_out/budget
for lc in ${LCS:-4 16 32 64}; do
  GRIDADMM_LANE_CAP=$lc timeout 300 python scripts/probe_solve_profile.py case_ACTIVSg70k 100 1e4 1000 4 /tmp/p.csv 2>&1 | sed -n 2p | sed "s/^/lc=$lc /" >> gpurun_out/budget/sweep.txt
  GRIDADMM_LANE_CAP=$lc timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lc=$lc bench', round(d['value'],1), {k: round(v['ms_total']/30*1e3,1) for k,v in d['kernels'].items()})" >> gpurun_out/budget/sweep.txt
done
