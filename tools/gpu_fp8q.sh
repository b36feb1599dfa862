cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fp8_dxt" 2>&1 | tail -2
for a in "--fp8-up --fp8-w1-cached" "--fp8-up --fp8-dxt --fp8-w1-cached"; do
  timeout 300 python bench.py --config qwen3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $a > gpurun_out/f8q.json 2>gpurun_out/f8q.err; echo "qwen3 [$a] rc=$?"
  python tools/show_bench.py gpurun_out/f8q.json | grep -E "^value|^ms_per|^dXt|^quant"
done
