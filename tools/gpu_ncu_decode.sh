# ncu --set full of the decode kernel (70B M = 1), summarised on the box
mkdir -p gpurun_out/dec
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:quick_decode --launch-skip 1 -c 1 \
  -o /tmp/dec1 -f python tools/prof_gemm.py --M 1 --N 28672 --K 8192 --reps 3 > gpurun_out/dec/dec1.log 2>&1
ncu -i /tmp/dec1.ncu-rep --page raw --csv > gpurun_out/dec/dec1_raw.csv 2>&1
ncu -i /tmp/dec1.ncu-rep --page details --csv > gpurun_out/dec/dec1_details.csv 2>&1
ncu -i /tmp/dec1.ncu-rep --page source --csv --print-source sass > gpurun_out/dec/dec1_source.csv 2>&1
gzip -f gpurun_out/dec/dec1_source.csv
tail -3 gpurun_out/dec/dec1.log
