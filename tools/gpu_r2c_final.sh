# round-2 session-3 final verification on a fresh box: GPU tests, smoke(), bench lines for every workload,
# the reference arm, the 32-layer Mistral chain, small-M sweep
mkdir -p gpurun_out/r2cf
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/r2cf/pytest_gpu.txt 2>&1
tail -3 gpurun_out/r2cf/pytest_gpu.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2cf/smoke.txt 2>&1
tail -1 gpurun_out/r2cf/smoke.txt
timeout -s KILL 600 python bench.py > gpurun_out/r2cf/bench.json 2> gpurun_out/r2cf/bench.err
for w in llama2_7b_attn llama2_13b_mlp mistral7b_stack tiny paper_fig7; do
  timeout -s KILL 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/r2cf/bench_$w.json 2> gpurun_out/r2cf/bench_$w.err
done
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2cf/bench_reference.json 2> gpurun_out/r2cf/bench_reference.err
rm -f gpurun_out/layer_chain.jsonl
timeout -s KILL 300 python tools/layer_chain.py 1,16,64,256 > gpurun_out/r2cf/layer_chain.txt 2>&1
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 400 python tools/sweep.py all 1,4,16,64,128,256,512,1024 pdl > gpurun_out/r2cf/sweep.txt 2>&1
ls -la gpurun_out/r2cf
