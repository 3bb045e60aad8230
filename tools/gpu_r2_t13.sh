mkdir -p gpurun_out/r2q
for v in new alt new alt; do
  if [ $v = alt ]; then export QUICK_LIB=$PWD/paper_2402_10076_b200/libquick_alt.so; else unset QUICK_LIB; fi
  rm -f gpurun_out/sweep.jsonl
  timeout -s KILL 300 python tools/sweep.py all 1,16,64 pdl > gpurun_out/r2q/sweep_$v.txt 2>&1
  cat gpurun_out/r2q/sweep_$v.txt >> gpurun_out/r2q/sweep_all_$v.txt
done
unset QUICK_LIB
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2q/pytest_gpu.txt 2>&1
tail -3 gpurun_out/r2q/pytest_gpu.txt
