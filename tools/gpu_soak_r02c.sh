# soak of the final build: the GPU test suite twice more, then back-to-back PDL launches of the automatic
# plan (the bench's launch mode) in fresh processes over the BJ shapes and M points, checked against a
# non-PDL launch (tools/pdl_repro.py prints OK / FAIL)
mkdir -p gpurun_out/soak
for r in 1 2; do
  timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/soak/pytest_$r.txt 2>&1
  tail -1 gpurun_out/soak/pytest_$r.txt
done
n=0; bad=0
for shp in "4096 4096" "13824 5120" "5120 13824" "28672 8192" "8192 28672" "8192 8192"; do
  set -- $shp
  for M in 1 16 64 128 256 512 1024; do
    out=$(timeout -s KILL 90 python tools/pdl_repro.py $M $1 $2 40 2>&1 | tail -1)
    n=$((n+1)); case "$out" in *"bit-equal to a non-PDL launch: True"*) ;; *) bad=$((bad+1)); echo "FAIL $M $1 $2: $out";; esac
  done
done
echo "pdl chains: $n fresh processes, $bad failures"
