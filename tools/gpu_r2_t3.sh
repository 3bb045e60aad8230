mkdir -p gpurun_out/r2f
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2f/pytest_gpu.txt 2>&1
tail -5 gpurun_out/r2f/pytest_gpu.txt
timeout -s KILL 600 python bench.py --workload mistral7b_stack --no-cpu-baseline > gpurun_out/r2f/bench_mistral.json 2> gpurun_out/r2f/bench_mistral.err
tail -c 400 gpurun_out/r2f/bench_mistral.err
