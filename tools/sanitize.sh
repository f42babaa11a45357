#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over
# tools/sanitize_smoke.py; logs to gpurun_out/sanitize_<tool>.log.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python tools/sanitize_smoke.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/sanitize_plain.log; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 \
    --target-processes all python tools/sanitize_smoke.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_$tool.log | tail -2 | tr '\n' ' ')"
done
