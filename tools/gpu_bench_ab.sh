# A/B of a build variant (libquick_alt.so) in the default bench (power-capped long run), alternating
# separate processes; prints value, the 8192x28672 M=1024 point and the clocks of each run
mkdir -p gpurun_out/benchab
for rep in 1 2 3; do
  for v in new alt; do
    if [ $v = new ]; then unset QUICK_LIB; else export QUICK_LIB=$PWD/paper_2402_10076_b200/libquick_alt.so; fi
    timeout -s KILL 600 python bench.py --no-cpu-baseline > gpurun_out/benchab/${v}_$rep.json 2>/dev/null
    python - $v gpurun_out/benchab/${v}_$rep.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
pt = {(s["N"], s["K"], s["M"]): s["us"] for s in d["sweep"]}
print(sys.argv[1], d["value"], "down1024 %.1f up1024 %.1f" % (pt[(8192, 28672, 1024)], pt[(28672, 8192, 1024)]), d["clocks"]["sm_mhz"])
PY
  done
done
