# cluster split-K push reduce: GPU parity tests, then push vs pull (flag 1<<15) on the cluster-split shapes
mkdir -p gpurun_out/push
timeout -s KILL 1200 python -m pytest tests -m gpu -x -q > gpurun_out/push/pytest.txt 2>&1
tail -3 gpurun_out/push/pytest.txt
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 600 python tools/sweep.py all 1,16,64,128,256,512,1024 pdl,pull > gpurun_out/push/sweep.txt 2>&1
cat gpurun_out/push/sweep.txt | awk '{print $1,$2,$3,$4,$5,$6,$7,$8,$9,$10,$11,$12,$13,$14,$15,$16,$17,$18,$19,$20}'
