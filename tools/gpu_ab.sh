# A/B of a build variant (paper_2402_10076_b200/libquick_alt.so) against the default build:
# parity tests on the variant, then alternating small-M sweeps.  usage: bash tools/gpu_ab.sh tag [Ms] [shapes] [tests]
tag=${1:-ab}; Ms=${2:-1,16,64}; shapes=${3:-all}; tests=${4:-1}
mkdir -p gpurun_out/ab
if [ "$tests" = 1 ]; then
  QUICK_LIB=$PWD/paper_2402_10076_b200/libquick_alt.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/ab/${tag}_pytest_alt.txt 2>&1
  tail -2 gpurun_out/ab/${tag}_pytest_alt.txt
fi
for v in new alt new alt; do
  if [ $v = alt ]; then export QUICK_LIB=$PWD/paper_2402_10076_b200/libquick_alt.so; else unset QUICK_LIB; fi
  rm -f gpurun_out/sweep.jsonl
  echo "== $v" >> gpurun_out/ab/${tag}.txt
  timeout -s KILL 300 python tools/sweep.py $shapes $Ms pdl >> gpurun_out/ab/${tag}.txt 2>&1
done
unset QUICK_LIB
python - <<PY
import re,collections
d=collections.defaultdict(list); v=None
for line in open("gpurun_out/ab/${tag}.txt"):
    if line.startswith("=="): v=line.split()[1]; continue
    m=re.match(r"(\d+) (\d+) (\d+) .* pdl ([\d.]+)us",line)
    if m: d[(m[1],m[2],m[3])].append((v,float(m[4])))
for k,vals in d.items():
    a=[t for vv,t in vals if vv=="new"]; b=[t for vv,t in vals if vv=="alt"]
    print(*k, "new %.2f alt %.2f  alt/new %.3f"%(min(a),min(b),min(b)/min(a)))
PY
