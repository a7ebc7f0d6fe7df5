#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of the small cases (summary -> gpurun_out/sanitize_*.log)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for mode in single loopback ragged; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py $mode > gpurun_out/sanitize_${tool}_$mode.log 2>&1
    echo "$tool $mode rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok' gpurun_out/sanitize_${tool}_$mode.log | tr '\n' ' ')"
  done
done
