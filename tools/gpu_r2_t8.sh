mkdir -p gpurun_out/r2k
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "bf16" > gpurun_out/r2k/pytest_bf16.txt 2>&1
tail -15 gpurun_out/r2k/pytest_bf16.txt
