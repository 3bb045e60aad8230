# final round-1 evidence: every bench workload + reference arm, the launch list of the default bench
# command, ncu --set full of the roofline kernels, the auto-plan sweep
bash tools/gpu_bench_all.sh
bash tools/ncu_capture_r01.sh
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 600 python tools/sweep.py all 1,4,16,32,64,128,256,512,1024 auto,pdl,nosk > gpurun_out/b/sweep.txt 2>&1
