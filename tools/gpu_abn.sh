# A/B/n of build variants (paper_2402_10076_b200/libquick_<v>.so) against the default build: alternating
# small-M PDL sweeps, min time per point.  usage: bash tools/gpu_abn.sh tag "v1 v2" [Ms] [shapes]
tag=${1:-abn}; vars=${2:-alt}; Ms=${3:-1,16,64}; shapes=${4:-all}
mkdir -p gpurun_out/ab
out=gpurun_out/ab/${tag}.txt
for rep in 1 2; do
  for v in new $vars; do
    if [ $v = new ]; then unset QUICK_LIB; else export QUICK_LIB=$PWD/paper_2402_10076_b200/libquick_$v.so; fi
    rm -f gpurun_out/sweep.jsonl
    echo "== $v" >> $out
    timeout -s KILL 300 python tools/sweep.py $shapes $Ms pdl >> $out 2>&1
  done
done
unset QUICK_LIB
python - "$out" <<'PY'
import re, collections, sys
d = collections.defaultdict(lambda: collections.defaultdict(list)); v = None; order = []
for line in open(sys.argv[1]):
    if line.startswith("=="):
        v = line.split()[1]; order.append(v) if v not in order else None; continue
    m = re.match(r"(\d+) (\d+) (\d+) .* pdl ([\d.]+)us", line)
    if m: d[(m[1], m[2], m[3])][v].append(float(m[4]))
for k, vals in d.items():
    base = min(vals["new"])
    print(*k, " ".join("%s %.2f (%.3f)" % (vv, min(vals[vv]), min(vals[vv]) / base) for vv in order if vals[vv]))
PY
