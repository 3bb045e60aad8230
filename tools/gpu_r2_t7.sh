mkdir -p gpurun_out/r2j
timeout -s KILL 600 python tools/diag_split_margin.py 128:1p,128:2p,128:4p,16:1,16:2,16:4 256 > gpurun_out/r2j/split_margin.txt 2>&1
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 600 python tools/sweep.py big 256,512,1024 pdl,t128s1p,t128s2p,t128s4p,t256s1p,t256s2p > gpurun_out/r2j/sweep_forced.txt 2>&1
