# interleaved A/B of libsonic variants at 7B: LIBS="a b c" REPS=3 bash tools/ab.sh  (exp_libs/<v>.so)
cd $GRAFT_REPO_ROOT
for r in $(seq 1 ${REPS:-3}); do
  for v in $LIBS; do
    SONIC_LIB=$PWD/exp_libs/$v.so timeout 300 python bench.py --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e \
      ${BENCH_ARGS} --breakdown gpurun_out/ab_${v}_$r.json > /dev/null 2> gpurun_out/ab_${v}_$r.err || echo "FAIL $v"
    echo "=== $v rep $r"; python tools/show_bench.py gpurun_out/ab_${v}_$r.json | grep -E "${SHOW:-^value|^ms_per|^clocks|^up|^down|^dH|^dXt|^dW}"
  done
done
