cd $GRAFT_REPO_ROOT
SONIC_LIB=$PWD/exp_libs/direct.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
LIBS="base direct" REPS=3 STEPS=20 SHOW="^value|^down|^dXt|^agg" bash tools/ab.sh
