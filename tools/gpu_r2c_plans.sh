# session 3: relaxed final cluster arrive (libquick_relax.so) A/B on the cluster split-K shapes, then forced
# small-M plans on 4096^2 and the 13B shapes (PDL chains)
mkdir -p gpurun_out/r2c
bash tools/gpu_abn.sh relax "relax" 1,16,128,256 small > /dev/null 2>&1
python - <<'PY' > gpurun_out/r2c/relax_ab.txt
import re, collections
d = collections.defaultdict(lambda: collections.defaultdict(list)); v = None
for line in open("gpurun_out/ab/relax.txt"):
    if line.startswith("=="): v = line.split()[1]; continue
    m = re.match(r"(\d+) (\d+) (\d+) .* pdl ([\d.]+)us", line)
    if m: d[(m[1], m[2], m[3])][v].append(float(m[4]))
for k, vals in d.items():
    print(*k, "new %.2f relax %.2f (%.3f)" % (min(vals["new"]), min(vals["relax"]), min(vals["relax"]) / min(vals["new"])))
PY
cat gpurun_out/r2c/relax_ab.txt
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 600 python tools/sweep.py small 1,16 pdl,t16s2,t16s4,t16s8,t16s0k,t32s4,t32s8 > gpurun_out/r2c/forced_4096.txt 2>&1
cat gpurun_out/r2c/forced_4096.txt | tail -4
timeout -s KILL 600 python tools/sweep.py all 1,16 pdl,t16s0k,t16s2,t16s4,t16s6,t16s8 > gpurun_out/r2c/forced_all.txt 2>&1
cat gpurun_out/r2c/forced_all.txt | tail -12
