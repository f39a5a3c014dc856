# ncu --set full of K6 (1-CTA, 2-CTA pair) and cuBLASLt on the EP8 hot-rank shapes
O=gpurun_out/k6prof; mkdir -p $O
for v in k6_down k6_gate_up cublaslt_down cublaslt_gate_up; do
  for cl in 1 2; do
    case $v in cublas*) [ $cl = 2 ] && continue;; esac
    REALB_GEMM_CLUSTER=$cl timeout 300 ncu --set full --import-source on --clock-control none --profile-from-start off \
      -o $O/${v}_cl$cl python scripts/prof_k6.py $v > $O/${v}_cl$cl.log 2>&1
    ncu -i $O/${v}_cl$cl.ncu-rep --page details --csv > $O/${v}_cl$cl.details.csv 2>/dev/null
    ncu -i $O/${v}_cl$cl.ncu-rep --page raw --csv > $O/${v}_cl$cl.raw.csv 2>/dev/null
  done
done
ls -la $O
