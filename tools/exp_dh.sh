set -e
cd $GRAFT_REPO_ROOT
for v in ${EXPS:-1 0}; do
  if [ $v = 0 ]; then unset SONIC_NVCC_EXTRA; else export SONIC_NVCC_EXTRA="-DSONIC_EXPERIMENT_DH_EPI=$v"; fi
  python paper_2512_14080_b200/build.py --force > /dev/null 2>&1
  timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e --breakdown gpurun_out/exp_$v.json > /dev/null 2>&1
  python tools/show_bench.py gpurun_out/exp_$v.json | grep -E "^dH|^up"
done
