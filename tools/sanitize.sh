# compute-sanitizer over tools/sanitize_cases.py: every libsonic kernel variant on small shapes.
# Logs -> gpurun_out/sanitizer_<tag>_<tool>.log (summaries are copied to profiles/).
#  memcheck   all kernels, all cases (no leak check: torch's caching allocator never frees at exit)
#  synccheck  all kernels, all cases
#  racecheck  the SIMT kernels (route, aggregation, EP, router bwd) on all cases; the tcgen05 GEMM
#             kernels separately per kernel template on two cases (the tool does not model the
#             async-proxy writes of TMA / cp.async.mbarrier or tcgen05.alloc)
#  initcheck  the SIMT kernels (TMA bulk stores are not seen as initialising writes by the tool; the
#             GEMM outputs are covered by tests/test_gpu_parity.py::test_poisoned_buffers instead)
cd ${GRAFT_REPO_ROOT:-.}
TAG=${TAG:-r2}
CS=/usr/local/cuda/bin/compute-sanitizer
EXC="--kernel-name-exclude kns=sonic_gemm_kernel --kernel-name-exclude kns=sonic_updown_kernel"
run() {  # name, timeout, args...
  local name=$1 tmo=$2; shift 2
  timeout $tmo $CS "$@" > gpurun_out/sanitizer_${TAG}_${name}.log 2>&1
  echo "$name rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer_${TAG}_${name}.log | tail -1)"
}
if [ -z "$ONLY" ] || [ "$ONLY" = memcheck ]; then
  run memcheck 1500 --tool memcheck --print-limit 200 python tools/sanitize_cases.py --ep; fi
if [ -z "$ONLY" ] || [ "$ONLY" = synccheck ]; then
  run synccheck 1500 --tool synccheck --print-limit 200 python tools/sanitize_cases.py --ep; fi
if [ -z "$ONLY" ] || [ "$ONLY" = racecheck ]; then
  run racecheck_simt 1500 --tool racecheck --racecheck-report all --print-limit 200 $EXC python tools/sanitize_cases.py --ep
  for k in 0ELi128ELb1 1ELi128ELb1 2ELi64ELb0 3ELi128ELb1 4ELi128ELb1 5ELi128ELb1 0ELi64ELb0 1ELi64ELb0 2ELi32ELb0 \
           3ELi64ELb0 4ELi64ELb0 5ELi64ELb0; do
    run racecheck_gemm_$k 600 --tool racecheck --racecheck-report all --print-limit 30 --kernel-name kns=gemm_kernelILi$k \
      python tools/sanitize_cases.py --only tiny_tc,ragged_tc
  done
  run racecheck_gemm_n256 900 --tool racecheck --racecheck-report all --print-limit 60 --kernel-name kns=sonic_ \
      python tools/sanitize_cases.py --only "n256 fused"
fi
if [ -z "$ONLY" ] || [ "$ONLY" = initcheck ]; then
  # k_aggregate reads Y / dX~, written by the (excluded) GEMMs' TMA stores: excluded too
  run initcheck_simt 2400 --tool initcheck --print-limit 200 $EXC --kernel-name-exclude kns=k_aggregate \
      python tools/sanitize_cases.py --ep; fi
