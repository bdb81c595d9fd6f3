#!/bin/bash
# per-line and headline counters of an ncu capture of one libatkg kernel
# usage: bash tools/ncu_report.sh <file.ncu-rep> <object under build/atkg> <mangled kernel name> [lines]
REP=$1; OBJ=$2; KERN=$3; N=${4:-45}
D=$(mktemp -d)
(cd $D && cuobjdump -xelf all /root/repo/build/atkg/$OBJ >/dev/null 2>&1 && nvdisasm -g *.cubin > all.dis 2>/dev/null)
ncu -i $REP --page source --csv --print-source sass 2>/dev/null > $D/sass.csv
ncu -i $REP --page raw --csv 2>/dev/null > $D/raw.csv
python /root/repo/tools/ncu_lines.py $D/sass.csv $D/all.dis $KERN 2>/dev/null | head -$N
python - <<PY
import csv
rows=list(csv.reader(open('$D/raw.csv')))
h=rows[0]; u=rows[1]; v=rows[2]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct','smsp__inst_executed.sum','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','smsp__thread_inst_executed_per_inst_executed.ratio','launch__registers_per_thread','dram__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio','smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio','smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio','smsp__average_warps_issue_stalled_wait_per_issue_active.ratio','smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio','smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio','smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio','smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio','smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio','smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio']
for i,n in enumerate(h):
    if n in want: print(n,u[i],v[i])
PY
rm -rf $D
