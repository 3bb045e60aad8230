# round 2: the paper's Fig. 7 shape (8192x8192) M-sweep beside cuBLAS fp16 dense,
# and the Fig. 3 question (shared-memory bank conflicts of a write-back design) at 64x8192x8192
mkdir -p gpurun_out/r2d
rm -f gpurun_out/cublas_context.jsonl gpurun_out/ablation.jsonl
timeout -s KILL 600 python tools/cublas_context.py 8192x8192 1,16,64,128,256,512,1024 > gpurun_out/r2d/fig7_sweep.txt 2>&1
timeout -s KILL 600 python tools/ablation_smem_a.py 64x8192x8192x16x2,64x8192x8192x128x4 > gpurun_out/r2d/ablation_64x8192.txt 2>&1
M="l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_shared_ld.sum,gpu__time_duration.sum,dram__bytes_read.sum"
for v in "16 2 0x4 tmemA" "16 2 0x200004 smemA" "128 4 0x4 tmemA" "128 4 0x200004 smemA"; do
  set -- $v
  timeout -s KILL 300 ncu --metrics $M --clock-control none -k regex:quick_w4a16 --launch-skip 1 -c 1 --csv \
    python tools/prof_gemm.py --M 64 --N 8192 --K 8192 --tile_n $1 --split_k $2 --flags $3 --reps 3 > gpurun_out/r2d/ncu_fig3_t$1_$4.csv 2>&1
done
timeout -s KILL 600 python bench.py > gpurun_out/r2d/bench_default.json 2> gpurun_out/r2d/bench_default.err
tail -3 gpurun_out/r2d/bench_default.err
