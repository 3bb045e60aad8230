# M = 64 limiter probe: L2 / DRAM / issue counters of the automatic plan's launch (70B up and down, 13B)
mkdir -p gpurun_out/m64
for shp in "28672 8192" "8192 28672" "13824 5120"; do
  set -- $shp
  timeout -s KILL 300 ncu --clock-control none -k regex:quick_w4a16 --launch-skip 1 -c 1 \
    --metrics gpu__time_duration.sum,lts__t_sectors.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,dram__bytes_read.sum,launch__grid_size,launch__cluster_dim_x \
    --csv python tools/prof_gemm.py --M 64 --N $1 --K $2 --reps 3 > gpurun_out/m64/m64_$1x$2.csv 2>&1
  echo "== $1 x $2"; grep -E '"(gpu__|lts__|dram__|l1tex__|smsp__|sm__|launch__)' gpurun_out/m64/m64_$1x$2.csv | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"'
done
