cd $GRAFT_REPO_ROOT
SONIC_LIB=$PWD/exp_libs/g4.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -E "passed|failed|Error|assert" | tail -4 | sed "s/^/g4 parity: /"
LIBS="base g4" REPS=3 STEPS=30 SHOW="^value|^ms_per|^dW" bash tools/ab.sh
