cd $GRAFT_REPO_ROOT
for v in tbase tnp8; do SONIC_LIB=$PWD/exp_libs/$v.so timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | grep "TIMING kind=[45]" | tail -2 | sed "s/^/$v /"; done
LIBS="base np8 np2" REPS=2 STEPS=30 SHOW="^value|^clocks|^up |^dH|^dW" bash tools/ab.sh
