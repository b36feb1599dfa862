# Captures the round's ncu evidence on the GPU box (1 GPU).
#  1) launch list of one step (all kernels, gpu__time_duration) -> gpurun_out/launches.csv
#  2) ncu --set full of the dominant GEMM launch(es)             -> gpurun_out/prof_<name>.ncu-rep
# usage: bash tools/profile_round.sh "<kernel-skip list: name:skip ...>"
export PATH=/usr/local/cuda/bin:$PATH
cd $GRAFT_REPO_ROOT
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo launches=$?
for spec in ${PROFS:-dW1:11}; do
  name=${spec%%:*}; skip=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k sonic_gemm_kernel -s $skip -c 1 \
    -o gpurun_out/prof_$name python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo prof_$name=$?
done
