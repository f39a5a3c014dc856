#!/usr/bin/env bash
# One GPU session's evidence for profiles/<round>/ (run through gpurun from the
# repo root): GPU tests, the bench line, the reference arm, the ncu launch list of
# a short bench run, and full ncu captures of the dominant kernels.
#   gpurun --timeout 3000 -- 'bash scripts/round_profile.sh r02'
set -u
R=${1:-r02}
O=gpurun_out/$R
mkdir -p "$O"
rm -f gpurun_out/parity_log.jsonl
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > "$O/smoke.log" 2>&1; tail -2 "$O/smoke.log"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > "$O/gputest.log" 2>&1; tail -3 "$O/gputest.log"
cp gpurun_out/parity_log.jsonl "$O/parity_log.jsonl" 2>/dev/null
timeout 600 python bench.py --steps 20 --warmup 5 > "$O/bench.json" 2> "$O/bench.err"; tail -c 300 "$O/bench.json"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > "$O/reference.json" 2> "$O/reference.err"
# launch list (cold cache, serialised): kernel shares of the step
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file "$O/launches.csv" python bench.py --steps 2 --warmup 1 --no-virtual-ep --no-cpu-baseline \
  --sustained-steps 0 \
  > "$O/launches_bench.log" 2>&1
# full captures: the bench layer's K5 gate_up (the roofline kernel) and down, router, dispatch, combine
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"grouped_gemm_bf16|router|combine|gather|permute" \
  -c 6 -o "$O/layer_full" python bench.py --steps 1 --warmup 1 --no-virtual-ep --no-cpu-baseline --sustained-steps 0 \
  > "$O/layer_full.log" 2>&1
echo done
