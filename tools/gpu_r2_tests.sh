set -x
mkdir -p gpurun_out/r2b
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2b/pytest_gpu.txt 2>&1
tail -30 gpurun_out/r2b/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b/smoke.txt 2>&1; tail -3 gpurun_out/r2b/smoke.txt
