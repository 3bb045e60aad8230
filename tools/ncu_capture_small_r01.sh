# ncu --set full of the small-M (HBM-bound) kernels on the final round-1 code
mkdir -p gpurun_out/ncu
cap() {  # name M N K
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:quick_w4a16 --launch-skip 1 -c 1 \
    -o gpurun_out/ncu/$1 -f python tools/prof_gemm.py --M $2 --N $3 --K $4 --reps 3 > gpurun_out/ncu/$1.log 2>&1
}
cap attn_m1 1 4096 4096
cap attn_m16 16 4096 4096
cap mlp70_m16 16 28672 8192
cap mlp13_m16 16 13824 5120
