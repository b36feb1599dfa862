cd $GRAFT_REPO_ROOT
for r in 1 2 3; do
  for g in "" "--graph"; do
    timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e $g > gpurun_out/g_${r}_${g:-eager}.json 2>/dev/null
    python - "$r" "$g" gpurun_out/g_${r}_${g:-eager}.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[3]).read().strip().splitlines()[-1])
print(sys.argv[1], sys.argv[2] or "eager", round(d["ms_per_step"],4), round(d["value"],1), d["clocks"], "warm", round(d["warm"]["ms_per_step"],4))
PY
  done
done
