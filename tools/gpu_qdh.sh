cd $GRAFT_REPO_ROOT
export PATH=/usr/local/cuda/bin:$PATH
timeout 300 ncu --set full --clock-control none -k regex:k_quant_dh -s 2 -c 1 -o gpurun_out/prof_qdh python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --fp8-dxt > /dev/null 2>&1; echo ncu=$?
ncu -i gpurun_out/prof_qdh.ncu-rep --page details --csv 2>/dev/null | grep -E '"Duration"|"DRAM Throughput"|"Memory Throughput"|"Achieved Occupancy"|"Registers Per|"L2 Hit Rate"|"Theoretical Occupancy"|Elapsed Cycles|"Compute \(SM\) Throughput"' | head -20
ncu -i gpurun_out/prof_qdh.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2] if len(r)>2 else r[1]
for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','smsp__average_warp_latency_issue_stalled_long_scoreboard','smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct','smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct','smsp__warp_issue_stalled_barrier_per_warp_active.pct','smsp__warp_issue_stalled_membar_per_warp_active.pct','launch__grid_size','sm__warps_active.avg.pct_of_peak_sustained_active']:
  if k in h: print(k, v[h.index(k)])
"
