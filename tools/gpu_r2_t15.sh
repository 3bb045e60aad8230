mkdir -p gpurun_out/r2t
timeout -s KILL 120 python tools/trace_gemm.py 16 28672 8192 > gpurun_out/r2t/trace_plain.txt 2>&1
TRACE_FLAGS=0x10000 timeout -s KILL 120 python tools/trace_gemm.py 16 28672 8192 > gpurun_out/r2t/trace_reversed.txt 2>&1
timeout -s KILL 120 python tools/trace_gemm.py 16 13824 5120 > gpurun_out/r2t/trace13_plain.txt 2>&1
TRACE_FLAGS=0x10000 timeout -s KILL 120 python tools/trace_gemm.py 16 13824 5120 > gpurun_out/r2t/trace13_reversed.txt 2>&1
head -2 gpurun_out/r2t/*.txt
