# per-SMSP issue balance of the small-M stream-K kernel (70B up-projection, M = 16): ncu min/avg/max over
# the SM sub-partitions of issued instructions, FMA-pipe activity and active warps
mkdir -p gpurun_out/smsp
M=${1:-16}; N=${2:-28672}; K=${3:-8192}
timeout -s KILL 400 ncu --clock-control none -k regex:quick_w4a16 --launch-skip 1 -c 1 \
  --metrics smsp__inst_issued.sum,smsp__inst_issued.max,smsp__inst_issued.min,smsp__inst_issued.avg,smsp__pipe_fma_cycles_active.max,smsp__pipe_fma_cycles_active.min,smsp__pipe_fma_cycles_active.avg,smsp__warps_active.max,smsp__warps_active.min,smsp__warps_active.avg,smsp__cycles_active.avg,sm__cycles_elapsed.avg,smsp__issue_active.max,smsp__issue_active.min,smsp__issue_active.avg \
  --csv python tools/prof_gemm.py --M $M --N $N --K $K --reps 3 > gpurun_out/smsp/m${M}_${N}x${K}.csv 2>&1
grep -E "smsp__|sm__" gpurun_out/smsp/m${M}_${N}x${K}.csv | awk -F'","' '{print $(NF-2), $NF}'
