#!/bin/bash
# compute-sanitizer, one tool per pass, on the small end-to-end cases (logs in gpurun_out/)
python tools/sanitize_case.py > gpurun_out/r02_sanitize_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/r02_sanitize_plain.log; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_case.py > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/r02_sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
