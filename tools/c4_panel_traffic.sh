#!/bin/bash
# DRAM bytes of gemm_tc_kernel per tile-order panel width (ncu, two counters only)
OUT=$1; mkdir -p $OUT
for NP in 1 2 4 8 16 32; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc -s 3 -c 1 --csv \
    python -c "
import sys; sys.path.insert(0, '.')
import paper_2506_04165_b200 as atk
atk._lib.set_option('gemm_n_panel', $NP)
sys.argv = ['prof_c4_target.py', '5']
import runpy; runpy.run_path('tools/prof_c4_target.py', run_name='__main__')
" 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' -v np=$NP '{gsub(/"/,"",$NF); print "n_panel=" np, $(NF-2), $(NF-1), $NF}'
done | tee $OUT/c4_panel_traffic.log
