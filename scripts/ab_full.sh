#!/bin/bash
# A/B of a build variant: bench window, full 70k solve, and the GPU parity suite on the variant
# usage: O=<dir> bash scripts/ab_full.sh <variant>
O=${O:-gpurun_out/abf}; mkdir -p $O; v=$1
O=$O bash scripts/ab_bench.sh default $v
O=$O bash scripts/ab_converge.sh $v default
GRIDADMM_LIB=paper_2110_06879_b200/libgridadmm_$v.so timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_$v.log 2>&1
