#!/bin/bash
# K1 tuning variants on configs[1] (f2 d=5 to tolerance) only: tools/k1_variants.py over $LIBS
mkdir -p gpurun_out
D=5 INIT=0 ITS=40 timeout 1200 python tools/k1_variants.py $LIBS 2>&1 | tee gpurun_out/${TAG:-ab}_d5.txt
