mkdir -p gpurun_out/r2m
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 900 python tools/sweep.py mistral 128,256,512 pdl,t128s1,t128s2,t128s4,t128s8,t128s1p,t128s2p,t128s4p,t256s1,t256s2,t256s4,t256s1p,t256s2p,t256s4p > gpurun_out/r2m/sweep_forced_small_n.txt 2>&1
