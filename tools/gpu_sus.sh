cd $GRAFT_REPO_ROOT
for r in 1 2; do for a in "" "--fuse"; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --sustain-s 3 $a > gpurun_out/sus.json 2>gpurun_out/sus.err; echo "[$a] rc=$?"
  python - <<'PY'
import json
d=json.loads(open("gpurun_out/sus.json").read().strip().splitlines()[-1])
print(" 20-step", round(d["ms_per_step"],4), "sustained", round(d["sustained"]["ms_per_step"],4), d["sustained"]["clocks"].get("sm_mhz"), d["sustained"]["clocks"].get("power_w"))
PY
done; done
