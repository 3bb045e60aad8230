# mma.sync decode ablation: parity tests + PDL-chain sweep beside the automatic (tcgen05) plan
mkdir -p gpurun_out/mms
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mmasync or bias or stream_k" > gpurun_out/mms/pytest.txt 2>&1; tail -1 gpurun_out/mms/pytest.txt
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 600 python tools/sweep.py all 1,4,8,16 pdl,mmasync > gpurun_out/mms/sweep.txt 2>&1
timeout -s KILL 300 python tools/sweep.py mistral 1,8,16 pdl,mmasync >> gpurun_out/mms/sweep.txt 2>&1
cat gpurun_out/mms/sweep.txt
