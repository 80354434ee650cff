#!/bin/bash
# run selected GPU tests: bash tools/gpu_tests.sh <pytest args...>
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
timeout 2400 python -m pytest -p no:cacheprovider -q "$@" > gpurun_out/pytest_sel.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_sel.log
tail -30 gpurun_out/pytest_sel.log
