cd $GRAFT_REPO_ROOT
LIBS="base e1 e2 e3 noepi" REPS=2 STEPS=20 SHOW="^value|^down|^dXt|^up |^dW1" bash tools/ab.sh
