# Round-end bench lines for the configs (1 GPU), into gpurun_out/r_<tag>.json
cd $GRAFT_REPO_ROOT
run() { tag=$1; shift; timeout 600 python bench.py "$@" > gpurun_out/r_$tag.json 2> gpurun_out/r_$tag.err; echo "$tag rc=$? $(head -c 300 gpurun_out/r_$tag.json)"; }
run 7b_tc --steps 20
run 7b_tc_fp8 --steps 20 --fp8-up --fp8-w1-cached --no-cpu-baseline
run 7b_tc_fp8dxt --steps 20 --fp8-up --fp8-dxt --fp8-w1-cached --no-cpu-baseline
run 7b_tr --steps 20 --mode tr --no-cpu-baseline
run qwen3_tc --config qwen3 --steps 20 --no-cpu-baseline
run qwen3_tr --config qwen3 --steps 20 --mode tr --no-cpu-baseline
run dsv3_tc --config dsv3 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3
run kimi_tr --config kimi --mode tr --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3
run ep1 --ep --steps 20 --no-cpu-baseline
run ref --impl reference --steps 3 --warmup 3
