cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
A="--config qwen3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none -k sonic_gemm_kernel -s 8 -c 1 -o gpurun_out/prof_q_dh python bench.py $A > gpurun_out/ncuq.log 2>&1; echo dh=$?
timeout 600 ncu --set full --clock-control none -k sonic_gemm_kernel -s 6 -c 1 -o gpurun_out/prof_q_up python bench.py $A >> gpurun_out/ncuq.log 2>&1; echo up=$?
