# Round-2 A/B experiments run on the B200 (results in profiles/r02_*.txt); each is a function,
# run one with e.g.  bash tools/gpu_r2_experiments.sh warp_roles
# Build variants for A/B: python -c "from paper_2402_10076_b200 import build as b; \
#   b.build(out=b.LIB.replace('libquick.so','libquick_alt.so'), defines=['QUICK_ROLES_FIRST'])"
# and select one with QUICK_LIB=<path> (tools only).
set -u
mkdir -p gpurun_out/r2x
ab_sweep() {  # $1 = tag, $2 = shapes, $3 = Ms: alternate the default build and libquick_alt.so twice
  for v in new alt new alt; do
    if [ $v = alt ]; then export QUICK_LIB=$PWD/paper_2402_10076_b200/libquick_alt.so; else unset QUICK_LIB; fi
    rm -f gpurun_out/sweep.jsonl
    timeout -s KILL 300 python tools/sweep.py $2 $3 pdl >> gpurun_out/r2x/$1_$v.txt 2>&1
  done
  unset QUICK_LIB
}
warp_roles() { ab_sweep warp_roles all 1,16,64,256,1024; }          # r02_warp_roles_ab.txt
dequant_addressing() { ab_sweep dequant_addr all 1,16,64; }          # r02_dequant_addressing_ab.txt
l2_policy() { ab_sweep l2_policy big 128,256,512,1024; }            # r02_l2_policy_ab.txt
split_margin() {                                                     # r02_split_margin.txt
  timeout -s KILL 900 python tools/diag_split_margin.py 128:1p,128:2p,256:2p,128:4p,16:1,16:2,16:4 256 > gpurun_out/r2x/split_margin_m256.txt 2>&1
  timeout -s KILL 900 python tools/diag_split_margin.py 128:1p,128:2p,256:2p,128:4p 1024 > gpurun_out/r2x/split_margin_m1024.txt 2>&1
}
forced_plans() {                                                     # r02_sweep_forced_70b.txt
  timeout -s KILL 600 python tools/sweep.py big 256,512,1024 pdl,t128s1p,t128s2p,t128s4p,t256s1p,t256s2p > gpurun_out/r2x/forced_70b.txt 2>&1
  timeout -s KILL 900 python tools/sweep.py mistral 128,256,512 pdl,t128s1,t128s2,t128s4,t128s8,t128s1p,t128s2p,t128s4p,t256s1,t256s2,t256s4,t256s1p,t256s2p,t256s4p > gpurun_out/r2x/forced_small_n.txt 2>&1
}
sk_placement() {                                                     # r02_sk_placement.txt
  timeout -s KILL 120 python tools/trace_gemm.py 16 28672 8192 > gpurun_out/r2x/trace_plain.txt 2>&1
  TRACE_FLAGS=0x10000 timeout -s KILL 120 python tools/trace_gemm.py 16 28672 8192 > gpurun_out/r2x/trace_reversed.txt 2>&1
}
layer_chain() { timeout -s KILL 300 python tools/layer_chain.py 1,16,64,256 > gpurun_out/r2x/layer_chain.txt 2>&1; }   # r02_mistral_layer_chain.txt
n2_one_gpu() {                                                       # r02_n2_one_gpu/
  for c in nccl peer; do
    timeout -s KILL 600 python bench.py --gpus 2 --dist-backend gloo --comm $c --steps 40 --warmup 3 > gpurun_out/r2x/bench_n2_$c.json 2>&1
  done
}
"$@"
