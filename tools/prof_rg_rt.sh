#!/bin/bash
OUT=$1; mkdir -p $OUT
ncu --set full --clock-control none --import-source on -k regex:row_reg -s 2 -c 1 -o $OUT/rowreg_rt -f \
  python -c "
import sys, runpy
import paper_2506_04165_b200 as atk
atk._lib.set_option('rowreg_rt', 1)
sys.argv = ['prof_one.py', 'C3', '3']
runpy.run_path('tools/prof_one.py', run_name='__main__')
" > $OUT/ncu_rt.log 2>&1
tail -2 $OUT/ncu_rt.log
