#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py (every kernel family)
mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize.py > gpurun_out/san/$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/san/$t.log
  tail -3 gpurun_out/san/$t.log
done
