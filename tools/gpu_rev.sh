cd $GRAFT_REPO_ROOT
SONIC_LIB=$PWD/exp_libs/rev.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "7b or multi or n256 or tiny" 2>&1 | tail -1
LIBS="base rev revnh nh" REPS=3 STEPS=20 SHOW="^value|^ms_per|^dH|^dXt|^dW" bash tools/ab.sh
