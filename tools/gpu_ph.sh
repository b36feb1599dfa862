cd $GRAFT_REPO_ROOT
SONIC_LIB=$PWD/exp_libs/ph3.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "n256 or 2048 or 7b" 2>&1 | grep -E "passed|failed|Error|assert" | tail -3 | sed "s/^/ph3 parity: /"
LIBS="base ph1 ph2 ph3" REPS=2 STEPS=30 SHOW="^value|^ms_per|^dW1" bash tools/ab.sh
timeout 300 python tools/cublas_shapes.py > gpurun_out/cublas_shapes_r2.txt 2>&1; cat gpurun_out/cublas_shapes_r2.txt
