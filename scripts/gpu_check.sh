set -u
O=gpurun_out/${1:-r02c}; mkdir -p $O
rm -f gpurun_out/parity_log.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/gputest.log 2>&1; tail -3 $O/gputest.log
cp gpurun_out/parity_log.jsonl $O/ 2>/dev/null
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; tail -c 400 $O/bench.json
