# A/B of the automatic plan with and without CTA pairs under sustained load (bench.py's timing,
# clocks sampled during the timed region): alternating runs on one box
for i in 1 2; do
  for f in 0 0x80000; do
    QUICK_BENCH_EXTRA_FLAGS=$f timeout -s KILL 300 python bench.py --workload ${AB_WORKLOAD:-llama2_70b_mlp} --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('flags $f', d['value'], d['unit'], 'clocks', d['clocks']['sm_mhz'], d['clocks']['reasons'], ' '.join('M%d:%.1f' % (r['M'], r['us']) for r in d['sweep']))"
  done
done
