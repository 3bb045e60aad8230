mkdir -p gpurun_out/r2e
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "silu or gate_up" > gpurun_out/r2e/pytest_silu.txt 2>&1
tail -5 gpurun_out/r2e/pytest_silu.txt
for c in "16 28672 8192" "1 4096 4096" "1 13824 5120"; do
  timeout -s KILL 120 python tools/trace_gemm.py $c > "gpurun_out/r2e/trace_${c// /_}.txt" 2>&1
done
