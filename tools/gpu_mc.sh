# MC4 check: L2 feed microbenchmark, parity tests, A/B mc vs nomc
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 120 ./tools/l2feed_bin | tee gpurun_out/l2feed.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
LIBS="mc nomc" REPS=2 STEPS=20 SHOW="^value|^ms_per|^clocks|^down|^dXt|^dW|^dH|^up" bash tools/ab.sh
