cd $GRAFT_REPO_ROOT
for v in d2 x2; do SONIC_LIB=$PWD/exp_libs/$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -E "passed|failed|Error|assert" | tail -4 | sed "s/^/$v parity: /"; done
LIBS="base d2 d2s2 x2" REPS=3 STEPS=30 SHOW="^value|^down|^dXt" bash tools/ab.sh
