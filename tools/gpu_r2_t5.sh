mkdir -p gpurun_out/r2h
timeout -s KILL 600 python -m pytest tests/test_gpu_tp.py -x -q -p no:cacheprovider -k "fused" > gpurun_out/r2h/pytest_fused.txt 2>&1
tail -30 gpurun_out/r2h/pytest_fused.txt
