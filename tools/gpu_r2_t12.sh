mkdir -p gpurun_out/r2o
rm -f gpurun_out/layer_chain.jsonl
timeout -s KILL 300 python tools/layer_chain.py 1,64 2 > gpurun_out/r2o/layer_chain_pf2.txt 2>&1
timeout -s KILL 300 python tools/layer_chain.py 1 0.25 > gpurun_out/r2o/layer_chain_pf025.txt 2>&1
