cd $GRAFT_REPO_ROOT
SONIC_LIB=$PWD/exp_libs/ord1.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "7b or n256 or multi" 2>&1 | tail -1
LIBS="base ord1" REPS=3 STEPS=20 SHOW="^value|^ms_per|^dXt|^dW|^agg_dX" bash tools/ab.sh
