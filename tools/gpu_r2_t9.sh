mkdir -p gpurun_out/r2l
timeout -s KILL 900 python tools/diag_split_margin.py 128:1p,128:2p,256:2p,128:4p,16:1,16:2,16:4 256 > gpurun_out/r2l/split_margin_m256.txt 2>&1
timeout -s KILL 900 python tools/diag_split_margin.py 128:1p,128:2p,256:2p,128:4p 1024 > gpurun_out/r2l/split_margin_m1024.txt 2>&1
