cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 20 --warmup 5 --sustain-s 3 > gpurun_out/final_7b.json 2> gpurun_out/final_7b.err; echo final_7b=$?
bash tools/round_bench.sh
