# exercise bench.py's N > 1 code paths with 2 ranks sharing the one GPU (gloo process group; not a measurement)
mkdir -p gpurun_out/r2w
timeout -s KILL 600 python bench.py --gpus 2 --dist-backend gloo --steps 40 --warmup 3 > gpurun_out/r2w/bench_n2_gloo.json 2> gpurun_out/r2w/bench_n2_gloo.err
tail -c 400 gpurun_out/r2w/bench_n2_gloo.err
timeout -s KILL 600 python bench.py --gpus 2 --dist-backend gloo --comm peer --steps 40 --warmup 3 > gpurun_out/r2w/bench_n2_peer.json 2> gpurun_out/r2w/bench_n2_peer.err
tail -c 400 gpurun_out/r2w/bench_n2_peer.err
timeout -s KILL 600 python bench.py --gpus 2 --dist-backend gloo --comm peer --workload mistral7b_stack --steps 40 --warmup 3 > gpurun_out/r2w/bench_n2_peer_mistral.json 2> gpurun_out/r2w/bench_n2_peer_mistral.err
tail -c 400 gpurun_out/r2w/bench_n2_peer_mistral.err
timeout -s KILL 600 python bench.py --gpus 2 --dist-backend gloo --workload mistral7b_stack --steps 40 --warmup 3 > gpurun_out/r2w/bench_n2_gloo_mistral.json 2> gpurun_out/r2w/bench_n2_gloo_mistral.err
tail -c 400 gpurun_out/r2w/bench_n2_gloo_mistral.err
