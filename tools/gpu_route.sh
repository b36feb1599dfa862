cd ${GRAFT_REPO_ROOT:-.}
for v in topk_old topk_new; do for c in 7b qwen3 kimi; do SONIC_LIB=$PWD/exp_libs/$v.so python tools/route_time.py $c tc | sed "s/^/$v /"; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q -k "not qwen3_full" 2>&1 | tail -3
