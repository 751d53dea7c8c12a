O=gpurun_out/bb; mkdir -p $O
for v in default bb96 bb160 bb64 default; do
  L=paper_2110_06879_b200/libgridadmm_$v.so; [ $v = default ] && L=paper_2110_06879_b200/libgridadmm.so
  GRIDADMM_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-converge --no-track > $O/bench_$v.json 2>&1
done
O=gpurun_out/bb bash scripts/ab_converge.sh bb96 bb160 default
