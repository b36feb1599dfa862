cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
for a in "--fp8-up --fp8-w1-cached" "--fp8-up --fp8-dxt --fp8-w1-cached"; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e $a > gpurun_out/f8.json 2>gpurun_out/f8.err; echo "[$a] rc=$?"
  python tools/show_bench.py gpurun_out/f8.json | grep -E "^value|^ms_per|^quant|^up |^dXt"
done
