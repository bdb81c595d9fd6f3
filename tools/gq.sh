#!/bin/bash
# build here, then run the given command on the GPU box (stop if the build fails)
set -e
python /root/repo/paper_2506_04165_b200/build.py > /tmp/build.log 2>&1 || { grep -A3 " error" /tmp/build.log | head -20; exit 1; }
/usr/local/graft/bin/gpurun --timeout ${T:-900} -- "$@"
