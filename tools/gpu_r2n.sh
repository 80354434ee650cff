#!/bin/bash
for v in "" build_variants/s1b3.so build_variants/s1b2.so; do
  for f in cec2022_f6 rosenbrock; do echo "lib=${v:-default}"; APO_LIB=$v timeout 120 python tools/prof_split.py $f; done
done 2>&1 | grep -v "^$"
