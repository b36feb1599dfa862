cd $GRAFT_REPO_ROOT
LIBS="base e2 e4" REPS=2 STEPS=20 SHOW="^value|^down|^dXt|^up " bash tools/ab.sh
