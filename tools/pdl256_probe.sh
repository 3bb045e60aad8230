# tile-256 PDL prefetch-depth probe: fresh processes, pair and one-CTA tile-256 plans
for i in $(seq 1 ${PROBE_N:-6}); do
  timeout -s KILL 60 python tools/pdl_repro.py 1024 13824 5120 20 2 3 2>&1 | tail -1
  timeout -s KILL 60 python tools/pdl_repro.py 1024 13824 5120 20 0x80002 3 2>&1 | tail -1
  timeout -s KILL 60 python tools/pdl_repro.py 512 28672 8192 20 0x80002 3 2>&1 | tail -1
  timeout -s KILL 60 python tools/pdl_repro.py 768 4096 4096 40 0x80002 3 2>&1 | tail -1
done
