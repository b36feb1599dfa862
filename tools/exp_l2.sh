# L2 residency experiments at 7B: persisting set-aside sizes (runtime), then build variants.
cd $GRAFT_REPO_ROOT
B="--steps 30 --warmup 3 --no-cpu-baseline --no-e2e"
for mb in 0 48 96 200; do
  SONIC_L2_PERSIST_MB=$mb timeout 300 python bench.py $B --breakdown gpurun_out/l2_$mb.json > /dev/null 2> gpurun_out/l2_$mb.err
  echo "=== persist $mb MB: $(grep 'l2 persist' gpurun_out/l2_$mb.err)"; python tools/show_bench.py gpurun_out/l2_$mb.json | grep -vE "^(tokens|layer|gpu_l|roofline|pct)"
done
EXPS="${EXPS:--DSONIC_L2PF=2;-DSONIC_L2_HINTS=0}" bash tools/exp_build.sh
