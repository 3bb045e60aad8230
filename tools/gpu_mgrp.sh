# m-tile groups for long-K cluster grids: tests, DRAM traffic and timing of 8192x28672 at M = 512 / 1024
mkdir -p gpurun_out/mgrp
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pair or full_size or tails or llama7b" > gpurun_out/mgrp/pytest.txt 2>&1; tail -1 gpurun_out/mgrp/pytest.txt
for M in 512 1024; do
  timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:quick_w4a16 --launch-skip 1 -c 1 --csv python tools/prof_gemm.py --M $M --N 8192 --K 28672 --reps 3 \
    > gpurun_out/mgrp/traffic_down70_m$M.csv 2>&1
  grep -E "dram__bytes|gpu__time" gpurun_out/mgrp/traffic_down70_m$M.csv | awk -F'","' '{print $(NF-2), $NF}'
done
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 300 python tools/sweep.py big 512,1024 pdl | sed 's/hbm [0-9.]* //'
