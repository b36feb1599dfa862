set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "fused or tiny or multi or n256 or 7b_dims" 2>&1 | tail -3
SONIC_LIB=$PWD/exp_libs/timing.so timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep "TIMING updown" | tail -2
LIBS="epw4 nopf base" REPS=2 STEPS=30 SHOW="^value|^updown|^up |^down" bash tools/ab.sh
BENCH_ARGS="--fuse" LIBS="base" REPS=2 STEPS=30 SHOW="^value|^updown|^up |^down" bash tools/ab.sh
