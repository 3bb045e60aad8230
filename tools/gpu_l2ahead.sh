# in-kernel L2 prefetch of the weights STAGES load stages ahead (flag 1<<15) vs the default, PDL chains, 2 reps
mkdir -p gpurun_out/l2a
for rep in 1 2; do
  rm -f gpurun_out/sweep.jsonl
  timeout -s KILL 600 python tools/sweep.py all ${1:-1,16,64,128,512,1024} pdl,l2ahead > gpurun_out/l2a/sweep_$rep.txt 2>&1
done
python - <<'PY'
import re, collections
d = collections.defaultdict(lambda: collections.defaultdict(list))
for rep in (1, 2):
    for l in open(f"gpurun_out/l2a/sweep_{rep}.txt"):
        m = re.match(r"(\d+) (\d+) (\d+) .* pdl ([\d.]+)us .* l2ahead ([\d.]+)us", l)
        if m:
            d[(m[1], m[2], m[3])]["pdl"].append(float(m[4])); d[(m[1], m[2], m[3])]["l2"].append(float(m[5]))
for k, v in d.items():
    print(*k, "pdl %.2f l2ahead %.2f (%.3f)" % (min(v["pdl"]), min(v["l2"]), min(v["l2"]) / min(v["pdl"])))
PY
