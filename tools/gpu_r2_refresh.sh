# round-2 refresh after the small-M kernel changes: every bench line, then the ncu evidence
bash tools/gpu_r2_bench_all.sh
bash tools/ncu_capture_r02.sh
