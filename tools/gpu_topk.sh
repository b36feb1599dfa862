cd $GRAFT_REPO_ROOT
for r in 1 2; do for v in base m6 m8; do for m in tc tr; do SONIC_LIB=$PWD/exp_libs/$v.so timeout 120 python tools/route_time.py 7b $m 2>&1 | tail -1 | sed "s/^/$v /"; done; done; done
SONIC_LIB=$PWD/exp_libs/m8.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "route or tiny or multi or variants" 2>&1 | tail -1
