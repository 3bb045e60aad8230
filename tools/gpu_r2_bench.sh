# round-2 bench runs: default workload (configs[3]) + configs[1]; sweep of the small-M PDL trigger modes
mkdir -p gpurun_out/r2c
timeout -s KILL 600 python bench.py > gpurun_out/r2c/bench_default.json 2> gpurun_out/r2c/bench_default.err
tail -c 600 gpurun_out/r2c/bench_default.err
timeout -s KILL 600 python bench.py --workload llama2_7b_attn --no-cpu-baseline > gpurun_out/r2c/bench_7b.json 2> gpurun_out/r2c/bench_7b.err
tail -c 600 gpurun_out/r2c/bench_7b.err
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 400 python tools/sweep.py all 1,16 pdl,pdlearly > gpurun_out/r2c/sweep_pdlearly.txt 2>&1
