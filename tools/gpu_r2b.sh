cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "not qwen3 and not kimi and not dsv3" 2>&1 | tail -3
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --breakdown gpurun_out/bench_r2b.json > gpurun_out/bench_r2b.line 2>&1; python tools/show_bench.py gpurun_out/bench_r2b.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"sonic_gemm_kernel<(1|3)," -c 2 -o gpurun_out/prof_down_dxt -f \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-l2-flush > /dev/null 2>&1; echo "ncu rc=$?"
