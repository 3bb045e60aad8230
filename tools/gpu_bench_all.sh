set -x
mkdir -p gpurun_out/b
for w in llama2_7b_attn llama2_70b_mlp llama2_13b_mlp mistral7b_stack tiny; do
  timeout -s KILL 400 python bench.py --workload $w > gpurun_out/b/bench_$w.json 2> gpurun_out/b/bench_$w.err
done
timeout -s KILL 400 python bench.py --impl reference > gpurun_out/b/bench_reference.json 2> gpurun_out/b/bench_reference.err
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:quick_w4a16 --launch-skip 1 -c 1 -o gpurun_out/b/pair_70b_m1024 python tools/prof_gemm.py --M 1024 --N 28672 --K 8192 --reps 3 > gpurun_out/b/ncu1.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:quick_w4a16 --launch-skip 1 -c 1 -o gpurun_out/b/pair_13b_m256 python tools/prof_gemm.py --M 256 --N 13824 --K 5120 --reps 3 > gpurun_out/b/ncu2.log 2>&1
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 600 python tools/sweep.py all 1,4,16,32,64,128,256,512,1024 auto,pdl,nosk > gpurun_out/b/sweep.txt 2>&1
