# PDL-wave rule A/B with alternating builds in separate processes (controls the power/thermal drift that
# biased back-to-back mode comparisons): new = no PDL for grids > 5 waves, oldpdl = PDL everywhere
mkdir -p gpurun_out/ab
out=gpurun_out/ab/pdlwave.txt; rm -f $out
for rep in 1 2 3; do
  for v in new oldpdl; do
    if [ $v = new ]; then unset QUICK_LIB; else export QUICK_LIB=$PWD/paper_2402_10076_b200/libquick_oldpdl.so; fi
    rm -f gpurun_out/sweep.jsonl
    echo "== $v" >> $out
    timeout -s KILL 300 python tools/sweep.py big 512,1024 pdl >> $out 2>&1
  done
done
unset QUICK_LIB
python - "$out" <<'PY'
import re, collections, sys
d = collections.defaultdict(lambda: collections.defaultdict(list)); v = None
for line in open(sys.argv[1]):
    if line.startswith("=="): v = line.split()[1]; continue
    m = re.match(r"(\d+) (\d+) (\d+) .* pdl ([\d.]+)us", line)
    if m: d[(m[1], m[2], m[3])][v].append(float(m[4]))
for k, vals in d.items():
    print(*k, "new", vals["new"], "oldpdl", vals["oldpdl"], "min ratio %.3f" % (min(vals["new"]) / min(vals["oldpdl"])))
PY
