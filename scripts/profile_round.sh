#!/bin/bash
# Evidence pass for one round (run under gpurun, ONE GPU): launch list of the
# bench command, full ncu captures of the 1-GPU layer kernels and the EP8 hot
# rank's kernels, summarised into profiles/$1/. Usage: scripts/profile_round.sh r01
set -u
R=${1:-r01}
mkdir -p gpurun_out profiles/$R
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-virtual-ep > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'router_kernel|align_kernel|permute_kernel|gather_rows_kernel|grouped_gemm|combine_kernel' -c 7 \
    -o gpurun_out/prof_layer python scripts/profile_kernels.py layer > gpurun_out/prof_layer.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'grouped_gemm|quant' -c 8 \
    -o gpurun_out/prof_ep8hot python scripts/profile_kernels.py ep8hot > gpurun_out/prof_ep8hot.log 2>&1
ls -la gpurun_out/
