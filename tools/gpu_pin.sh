cd $GRAFT_REPO_ROOT
SONIC_LIB=$PWD/exp_libs/pin16.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
LIBS="base pin8 pin12 pin16 pin24" REPS=2 STEPS=20 SHOW="^value|^ms_per|^dW|^agg_dX" bash tools/ab.sh
