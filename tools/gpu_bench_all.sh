# every bench.py workload + the reference arm + the ncu launch list of the default bench command
mkdir -p gpurun_out/b
for w in llama2_7b_attn llama2_70b_mlp llama2_13b_mlp mistral7b_stack tiny; do
  timeout -s KILL 400 python bench.py --workload $w > gpurun_out/b/bench_$w.json 2> gpurun_out/b/bench_$w.err
done
timeout -s KILL 400 python bench.py --impl reference > gpurun_out/b/bench_reference.json 2> gpurun_out/b/bench_reference.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/b/launches.csv python bench.py --steps 32 --warmup 3 --no-cpu-baseline > gpurun_out/b/ncu_bench.log 2>&1
