# usage: EXPS="flagsA;flagsB;..." bash tools/exp_build.sh   -- builds + benches each flag set (7B), prints kernel table
cd $GRAFT_REPO_ROOT
IFS=';' read -ra SETS <<< "$EXPS"
i=0
for f in "${SETS[@]}"; do
  export SONIC_NVCC_EXTRA="$f"
  python paper_2512_14080_b200/build.py --force > /dev/null 2>&1 || echo "BUILD FAILED: $f"
  timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} --breakdown gpurun_out/exp_$i.json > /dev/null 2>&1
  echo "=== [$f]"; python tools/show_bench.py gpurun_out/exp_$i.json | grep -E "${SHOW:-.}"
  i=$((i+1))
done
unset SONIC_NVCC_EXTRA
python paper_2512_14080_b200/build.py --force > /dev/null 2>&1
