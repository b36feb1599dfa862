cd $GRAFT_REPO_ROOT
SONIC_LIB=$PWD/exp_libs/x1.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "7b or multi or n256" 2>&1 | tail -1
LIBS="base x1 d1" REPS=3 STEPS=20 SHOW="^value|^ms_per|^down|^dXt" bash tools/ab.sh
