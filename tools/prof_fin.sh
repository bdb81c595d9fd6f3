#!/bin/bash
OUT=$1; mkdir -p $OUT
ncu --set full --clock-control none --import-source on -k regex:st_finish -s 2 -c 1 -o $OUT/st_finish -f \
  python tools/prof_one.py C2 3 > $OUT/ncu_fin.log 2>&1
tail -2 $OUT/ncu_fin.log
