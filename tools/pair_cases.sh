#!/bin/bash
# CTA-pair plan cases, one process each, each under its own timeout
cases="${PAIR_CASES:-256,512,512,256,1 200,256,1024,128,1 256,4096,4096,256,1 256,4096,4096,256,2 256,4096,4096,256,4 256,4096,4096,128,1 256,4096,4096,128,2 512,4096,4096,256,2 512,4096,4096,128,2 1024,28672,8192,256,1 1024,28672,8192,128,1 256,13824,5120,256,1}"
for c in $cases; do
  IFS=, read M N K T S <<< "$c"
  timeout -s KILL 90 python tools/pair_check.py $M $N $K $T $S $PAIR_PDL || echo "$c: exit $?"
done
