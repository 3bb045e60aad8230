# round-2 (session 3) baseline on a fresh box: GPU tests, default bench, small-M sweep
mkdir -p gpurun_out/r2c
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2c/pytest_gpu.txt 2>&1
tail -3 gpurun_out/r2c/pytest_gpu.txt
timeout -s KILL 600 python bench.py > gpurun_out/r2c/bench.json 2> gpurun_out/r2c/bench.err
timeout -s KILL 600 python bench.py --workload llama2_7b_attn --no-cpu-baseline > gpurun_out/r2c/bench_attn.json 2> gpurun_out/r2c/bench_attn.err
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 300 python tools/sweep.py all 1,4,16,64 pdl > gpurun_out/r2c/sweep_small.txt 2>&1
cat gpurun_out/r2c/sweep_small.txt | tail -30
