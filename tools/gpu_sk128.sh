# stream-K for the 128-token tile (forced) vs the automatic plans at M = 128..1024; parity of the forced plan
mkdir -p gpurun_out/sk128
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/sk128/pytest.txt 2>&1; tail -1 gpurun_out/sk128/pytest.txt
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 900 python tools/sweep.py all 128,256,512,1024 pdl,t128s0k > gpurun_out/sk128/sweep.txt 2>&1
timeout -s KILL 300 python tools/sweep.py mistral 128,256 pdl,t128s0k >> gpurun_out/sk128/sweep.txt 2>&1
cat gpurun_out/sk128/sweep.txt
