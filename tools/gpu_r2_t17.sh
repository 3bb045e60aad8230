mkdir -p gpurun_out/r2v
for w in 0 1100 0 1100 1200 1050 1150; do
  rm -f gpurun_out/sweep.jsonl
  QUICK_SK_WEIGHT=$w timeout -s KILL 300 python tools/sweep.py big 1,16 pdl >> gpurun_out/r2v/sweep_w$w.txt 2>&1
  QUICK_SK_WEIGHT=$w timeout -s KILL 300 python tools/sweep.py mistral 1,16 pdl >> gpurun_out/r2v/sweep_w$w.txt 2>&1
done
QUICK_SK_WEIGHT=1150 timeout -s KILL 120 python tools/trace_gemm.py 16 28672 8192 > gpurun_out/r2v/trace_w1150.txt 2>&1
QUICK_SK_WEIGHT=1150 timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "stream_k or small_m or long_k or silu" > gpurun_out/r2v/pytest_w1150.txt 2>&1
tail -3 gpurun_out/r2v/pytest_w1150.txt
