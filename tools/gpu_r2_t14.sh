mkdir -p gpurun_out/r2r
for v in new alt new alt; do
  if [ $v = alt ]; then export QUICK_LIB=$PWD/paper_2402_10076_b200/libquick_alt.so; else unset QUICK_LIB; fi
  rm -f gpurun_out/sweep.jsonl
  timeout -s KILL 300 python tools/sweep.py big 128,256,512,1024 pdl > gpurun_out/r2r/sweep_$v.txt 2>&1
  cat gpurun_out/r2r/sweep_$v.txt >> gpurun_out/r2r/sweep_all_$v.txt
  timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:quick_w4a16 --launch-skip 1 -c 1 --csv python tools/prof_gemm.py --M 1024 --N 8192 --K 28672 --reps 3 \
    > gpurun_out/r2r/traffic_down70_m1024_$v.csv 2>&1
done
unset QUICK_LIB
