#!/usr/bin/env bash
# compute-sanitizer sweep over the kernel-level GPU tests (run on the B200 box
# from the repo root). Logs land in gpurun_out/sanitize_<tool>.log; a summary
# line per tool in gpurun_out/sanitize_summary.txt.
#   memcheck  : out-of-bounds / misaligned global + shared accesses, leaks
#   racecheck : shared-memory hazards (mbarrier rings, DSMEM split-K fold)
#   synccheck : illegal __syncthreads / barrier usage
# The full-size C5 gradient test is left to memcheck only (racecheck replays
# every shared-memory access of 8192x4096x4096 GEMMs: hours).
set -u
mkdir -p gpurun_out
TESTS="tests/test_gpu_kernels.py tests/test_gpu_gemm.py tests/test_gpu_coherence.py tests/test_gpu_f32tc.py"
SUM=gpurun_out/sanitize_summary.txt
: > "$SUM"
for tool in memcheck racecheck synccheck; do
  sel=""
  extra=""
  case $tool in
    memcheck) extra="--leak-check no" ;;
    racecheck) sel="not full_size and not many_tiles and not long_k and not 8192 and not 4096 and not trajectory"; extra="--racecheck-report all" ;;
    synccheck) sel="not full_size" ;;
  esac
  log=gpurun_out/sanitize_$tool.log
  start=$(date +%s)
  if [ -n "$sel" ]; then
    timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool $extra --error-exitcode 99 --print-limit 50 \
      python -m pytest $TESTS -m gpu -q -x -p no:cacheprovider -k "$sel" > "$log" 2>&1
  else
    timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool $extra --error-exitcode 99 --print-limit 50 \
      python -m pytest $TESTS -m gpu -q -x -p no:cacheprovider > "$log" 2>&1
  fi
  rc=$?
  end=$(date +%s)
  echo "$tool rc=$rc seconds=$((end - start)) $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' "$log" | tr '\n' ' ')" >> "$SUM"
done
cat "$SUM"
