cd $GRAFT_REPO_ROOT
SONIC_LIB=$PWD/exp_libs/aggA.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -E "passed|failed|Error|assert" | tail -4 | sed "s/^/aggA parity: /"
LIBS="base aggA aggB aggD" REPS=2 STEPS=30 SHOW="^value|^ms_per|^dW|^agg_dX" bash tools/ab.sh
