cd $GRAFT_REPO_ROOT
LIBS="base nopdl" REPS=2 STEPS=20 BENCH_ARGS="--fp8-up --fp8-dxt --fp8-w1-cached" SHOW="^value|^ms_per|^quant|^dXt|^agg|^route" bash tools/ab.sh
