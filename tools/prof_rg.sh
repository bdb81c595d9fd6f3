#!/bin/bash
# ncu --set full of one row_reg_kernel launch on C3 (after the plain run exits 0)
# usage: bash tools/prof_rg.sh <outdir> [warps]
OUT=$1; W=${2:-16}
mkdir -p $OUT
python - <<PY > $OUT/prof_target.log 2>&1 || exit 1
import paper_2506_04165_b200 as atk
atk._lib.set_option("rowreg_warps", $W)
import runpy, sys
sys.argv = ["prof_one.py", "C3", "3"]
runpy.run_path("tools/prof_one.py", run_name="__main__")
PY
ATKG_RG_WARPS=$W ncu --set full --clock-control none --import-source on -k regex:row_reg -s 2 -c 1 -o $OUT/rowreg_w$W -f \
  python -c "
import sys, runpy
import paper_2506_04165_b200 as atk
atk._lib.set_option('rowreg_warps', $W)
sys.argv = ['prof_one.py', 'C3', '3']
runpy.run_path('tools/prof_one.py', run_name='__main__')
" > $OUT/ncu_w$W.log 2>&1
tail -3 $OUT/ncu_w$W.log
