cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ep1.csv python bench.py --ep --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
