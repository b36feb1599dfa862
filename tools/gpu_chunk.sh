cd $GRAFT_REPO_ROOT
for r in 1 2; do for c in "" "--chunked"; do timeout 300 python bench.py --ep --steps 20 --warmup 5 --no-cpu-baseline --no-e2e $c > gpurun_out/ep_${c:-plain}.json 2>gpurun_out/ep_${c:-plain}.err; echo "ep $c rc=$?"; python tools/show_bench.py gpurun_out/ep_${c:-plain}.json | grep -E "^value|^ms_per"; done; done
tail -3 gpurun_out/ep_--chunked.err
