# forced plans at M = 64 / 128 on the 70B and 13B shapes (PDL chains)
mkdir -p gpurun_out/r2c
rm -f gpurun_out/sweep.jsonl
timeout -s KILL 600 python tools/sweep.py big 64,128 pdl,t64s0k,t64s1,t64s2,t64s4,t128s1p,t128s2p,t128s4p,t128s1,t128s2,t128s4 > gpurun_out/r2c/forced_m128.txt 2>&1
timeout -s KILL 600 python tools/sweep.py all 64,128 pdl,t64s0k,t64s2,t128s1p,t128s2p,t128s2 >> gpurun_out/r2c/forced_m128.txt 2>&1
python - <<'PY'
import re
for l in open("gpurun_out/r2c/forced_m128.txt"):
    m = re.match(r"(\d+) (\d+) (\d+) (\{.*?\}) (.*)", l)
    if not m: continue
    modes = re.findall(r"(\S+) ([\d.]+)us", m[5])
    best = min(modes, key=lambda t: float(t[1]))
    print(m[1], m[2], m[3], " ".join(f"{a} {b}" for a, b in modes), "| best", best[0], best[1])
PY
