O=gpurun_out/k6v2prof; mkdir -p $O
for d in 0 23 31; do
  REALB_K6_VERSION=2 REALB_DBG_FP4=$d timeout 300 ncu --set full --import-source on --clock-control none --profile-from-start off \
      -o $O/v2_dbg$d python scripts/prof_k6.py k6_down > $O/v2_dbg$d.log 2>&1
  ncu -i $O/v2_dbg$d.ncu-rep --page raw --csv > $O/v2_dbg$d.raw.csv 2>/dev/null
done
K6_WAIT=0 K6_DBG=23,31,1 timeout 300 python scripts/bench_k6_v2.py 2>&1 | grep -E "^down|Error|error"
ls $O
