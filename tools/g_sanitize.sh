#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every kernel class (tools/sanitize.py)
D=gpurun_out/sanitize; mkdir -p $D
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all python tools/sanitize.py > $D/$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a $D/summary.txt
  tail -4 $D/$tool.txt
done
