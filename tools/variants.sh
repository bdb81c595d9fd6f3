#!/bin/bash
# time C2/C5 stage 1 for every library variant under build/variants (development aid)
for lib in paper_2506_04165_b200/libatkg.so build/variants/*.so; do
  echo "== $lib"
  ATKG_LIB=$lib python tools/seg_sweep.py C2 ${C2SEGS:-2,4,8,16} 2>&1 | tail -4
  ATKG_LIB=$lib python tools/seg_sweep.py C5 ${C5SEGS:-296,592,1184} 2>&1 | tail -3
done
