#!/bin/bash
# where lane-per-protozoon groups win: single runs (latency) and the C2 suite (throughput) at small D
for v in "0 32" "1 32"; do
  set -- $v
  export APO_BATCH_LPP=$1 APO_BATCH_LPP_G=$2
  echo "LPP=$1 G=$2"
  for d in 3 5 8; do python tools/prof_c1.py 100 $d 1000 sphere 2>&1 | tail -1; done
  python tools/prof_c1.py 100 5 1000 cec2022_f1 2>&1 | tail -1
  for d in 5 8 10; do echo "C2 D=$d"; C2_DIM=$d python tools/c2_shapes.py "c2:" | tail -1; done
done
