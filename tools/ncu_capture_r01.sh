# ncu --set full captures of the roofline kernels named by the bench lines (one launch each,
# after one warm-up launch), for profiles/ (tools/ncu_summary.py)
mkdir -p gpurun_out/ncu
cap() {  # name M N K
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:quick_w4a16 --launch-skip 1 -c 1 \
    -o gpurun_out/ncu/$1 -f python tools/prof_gemm.py --M $2 --N $3 --K $4 --reps 3 > gpurun_out/ncu/$1.log 2>&1
}
cap attn_m256 256 4096 4096
cap mlp70_m1024 1024 28672 8192
cap mlp70_m128 128 28672 8192
cap mlp13_m512 512 5120 13824
cap mistral_m256 256 28672 4096
