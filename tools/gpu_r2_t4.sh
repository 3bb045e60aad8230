mkdir -p gpurun_out/r2g
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "repack or gptq" > gpurun_out/r2g/pytest_f3.txt 2>&1
tail -5 gpurun_out/r2g/pytest_f3.txt
