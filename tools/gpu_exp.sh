# fused vs two-kernel up/down A/B + cycle counters of the fused kernel
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
SONIC_LIB=$PWD/exp_libs/timing.so timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-l2-flush 2>&1 | grep "TIMING" | sort | uniq -c | sort -rn | head -20
LIBS="base" REPS=2 STEPS=20 SHOW="^value|^ms_per|^clocks|^updown|^up |^down" bash tools/ab.sh
BENCH_ARGS="--fuse" LIBS="base" REPS=2 STEPS=20 SHOW="^value|^ms_per|^clocks|^updown|^up |^down" bash tools/ab.sh
