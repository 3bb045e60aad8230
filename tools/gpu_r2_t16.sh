mkdir -p gpurun_out/r2u
timeout -s KILL 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "silu or gate_up or stream_k or small_m or long_k" > gpurun_out/r2u/pytest_sel.txt 2>&1
tail -3 gpurun_out/r2u/pytest_sel.txt
for w in 0 1050 1100 1150 1200; do
  rm -f gpurun_out/sweep.jsonl
  QUICK_SK_WEIGHT=$w timeout -s KILL 300 python tools/sweep.py big 1,16 pdl > gpurun_out/r2u/sweep_w$w.txt 2>&1
  QUICK_SK_WEIGHT=$w timeout -s KILL 300 python tools/sweep.py mistral 1,16 pdl >> gpurun_out/r2u/sweep_w$w.txt 2>&1
done
QUICK_SK_WEIGHT=1100 timeout -s KILL 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "stream_k or small_m or long_k or silu" > gpurun_out/r2u/pytest_w1100.txt 2>&1
tail -3 gpurun_out/r2u/pytest_w1100.txt
timeout -s KILL 300 python bench.py --workload mistral7b_stack --no-cpu-baseline --steps 200 > gpurun_out/r2u/bench_mistral.json 2>/dev/null
