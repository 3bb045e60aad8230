# small-M probes: load-path ceiling (debug modes), per-stage trace, plain vs PDL at 70B M=1/16
mkdir -p gpurun_out/r2b
timeout -s KILL 300 python tools/loadpath_bench.py > gpurun_out/r2b/loadpath.txt 2>&1
timeout -s KILL 120 python tools/trace_gemm.py 1 28672 8192 > gpurun_out/r2b/trace_70b_m1.txt 2>&1
timeout -s KILL 120 python tools/trace_gemm.py 1 4096 4096 > gpurun_out/r2b/trace_4096_m1.txt 2>&1
cat gpurun_out/r2b/loadpath.txt
