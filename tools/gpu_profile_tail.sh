# launch list of the default bench command + the auto-plan sweep (PDL and plain) over the BJ shapes
mkdir -p gpurun_out/b
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/b/launches.csv python bench.py --steps 32 --warmup 3 --no-cpu-baseline > gpurun_out/b/ncu_bench.log 2>&1
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 600 python tools/sweep.py all 1,4,16,32,64,128,256,512,1024 auto,pdl,nosk > gpurun_out/b/sweep.txt 2>&1
