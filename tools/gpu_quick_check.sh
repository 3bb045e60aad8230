# quick GPU check after a kernel change: parity tests + small-M sweep (PDL) of the BJ shapes
# usage: bash tools/gpu_quick_check.sh <tag> [Ms] [shapes]
tag=${1:-x}; Ms=${2:-1,16,64}; shapes=${3:-all}
mkdir -p gpurun_out/qc
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/qc/${tag}_pytest.txt 2>&1
tail -2 gpurun_out/qc/${tag}_pytest.txt
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 300 python tools/sweep.py $shapes $Ms pdl > gpurun_out/qc/${tag}_sweep.txt 2>&1
cat gpurun_out/qc/${tag}_sweep.txt
