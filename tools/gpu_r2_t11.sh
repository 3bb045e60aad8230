mkdir -p gpurun_out/r2n
rm -f gpurun_out/layer_chain.jsonl
timeout -s KILL 600 python tools/layer_chain.py 1,16,64,256 24 > gpurun_out/r2n/layer_chain.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2n/pytest_gpu.txt 2>&1
tail -5 gpurun_out/r2n/pytest_gpu.txt
