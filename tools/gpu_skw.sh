# stream-K placement weights (QUICK_SK_WEIGHT_PROBE build): CTAs [0, P/2) weighted w/1000
export QUICK_LIB=$PWD/paper_2402_10076_b200/libquick_alt.so
for w in 0 900 950 1000 1050 1100 1150; do
  rm -f gpurun_out/sweep.jsonl
  echo "== weight $w"; QUICK_SK_WEIGHT=$w timeout -s KILL 200 python tools/sweep.py big 1,16 pdl 2>&1 | sed 's/hbm.*//'
done
