# round-end evidence: default bench line (+ sustained), the config sweep, ncu launch list + full sets
cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python bench.py --steps 20 --warmup 5 --sustain-s 3 > gpurun_out/final_7b.json 2> gpurun_out/final_7b.err; echo final_7b=$?
bash tools/round_bench.sh
PROFS="dW1:11 up:6 dXt:9" bash tools/profile_round.sh
ls -la gpurun_out/*.ncu-rep
