#!/bin/bash
# C2 suite under a minimum batch group size (APO_BATCH_G); not a bench value
python tools/c2_shapes.py 'g0:' 'g8:APO_BATCH_G=8' 'g10:APO_BATCH_G=10' 'g16:APO_BATCH_G=16' 'g0b:'
for g in 0 8 16; do APO_BATCH_G=$g python tools/prof_c1.py 2>&1 | tail -1; done
