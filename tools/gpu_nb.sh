cd $GRAFT_REPO_ROOT
LIBS="base nb1 nb4" REPS=3 STEPS=20 SHOW="^value|^dW" bash tools/ab.sh
