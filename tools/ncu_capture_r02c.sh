# round-2 (session 3, final build) ncu evidence for profiles/: the launch list of the default bench command, --set full captures of
# the dominant kernel group (8192x28672 down-projection, tile-128 CTA pairs, split 4) and of the small-M
# stream-K kernel (summarised on the box: raw + source CSV pages, reports deleted to stay under gpurun's
# 64 MiB return limit), and per-launch DRAM traffic of the dominant group's launches
mkdir -p gpurun_out/r2cq
timeout -s KILL 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/r2cq/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2cq/launches_bench.log 2>&1
tail -c 300 gpurun_out/r2cq/launches_bench.log
cap() {  # name M N K
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:quick_w4a16 --launch-skip 1 -c 1 \
    -o /tmp/$1 -f python tools/prof_gemm.py --M $2 --N $3 --K $4 --reps 3 > gpurun_out/r2cq/$1.log 2>&1
  ncu -i /tmp/$1.ncu-rep --page raw --csv > gpurun_out/r2cq/$1_raw.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page details --csv > gpurun_out/r2cq/$1_details.csv 2>&1
  ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/r2cq/$1_source.csv 2>&1
  gzip -f gpurun_out/r2cq/$1_source.csv
  rm -f /tmp/$1.ncu-rep
}
cap down70_m512 512 8192 28672
cap down70_m1024 1024 8192 28672
cap up70_m16 16 28672 8192
cap attn_m1 1 4096 4096
for M in 128 256 512 1024; do
  timeout -s KILL 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:quick_w4a16 --launch-skip 1 -c 1 --csv python tools/prof_gemm.py --M $M --N 8192 --K 28672 --reps 3 \
    > gpurun_out/r2cq/traffic_down70_m$M.csv 2>&1
done
du -sh gpurun_out
