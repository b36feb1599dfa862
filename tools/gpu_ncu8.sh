cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
A="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --fp8-up --fp8-dxt --fp8-w1-cached"
timeout 600 ncu --set full --clock-control none --import-source on -k sonic_gemm_kernel -s 9 -c 1 -o gpurun_out/prof_dxt8 python bench.py $A > gpurun_out/ncu8.log 2>&1; echo dxt8=$?
timeout 600 ncu --set full --clock-control none -k sonic_gemm_kernel -s 6 -c 1 -o gpurun_out/prof_up8 python bench.py $A >> gpurun_out/ncu8.log 2>&1; echo up8=$?
