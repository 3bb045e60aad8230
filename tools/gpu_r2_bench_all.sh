# round-2 bench lines for every workload + the reference arm + the 32-layer Mistral chain
mkdir -p gpurun_out/r2t
timeout -s KILL 600 python bench.py > gpurun_out/r2t/bench.json 2> gpurun_out/r2t/bench.err
for w in llama2_7b_attn llama2_13b_mlp mistral7b_stack tiny paper_fig7; do
  timeout -s KILL 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r2t/bench_$w.json 2> gpurun_out/r2t/bench_$w.err
done
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2t/bench_reference.json 2> gpurun_out/r2t/bench_reference.err
rm -f gpurun_out/layer_chain.jsonl
timeout -s KILL 300 python tools/layer_chain.py 1,16,64,256 > gpurun_out/r2t/layer_chain.txt 2>&1
ls -la gpurun_out/r2t
