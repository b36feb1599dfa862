cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fp8_dxt" 2>&1 | tail -1
for a in "--fp8-up --fp8-w1-cached" "--fp8-up --fp8-dxt --fp8-w1-cached" "--fp8-up --fp8-w1-cached" "--fp8-up --fp8-dxt --fp8-w1-cached"; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e $a > gpurun_out/f8.json 2>gpurun_out/f8.err; echo "[$a] rc=$?"
  python tools/show_bench.py gpurun_out/f8.json | grep -E "^value|^ms_per|^dXt|^quant_dh"
done
