mkdir -p gpurun_out
timeout 300 python tools/quick_time.py C2 C5 > gpurun_out/q_nw.log 2>&1
for v in n16s3 n16s2 n4s3; do echo "== $v" >> gpurun_out/q_nw.log; ATKG_LIB=build/libatkg_$v.so timeout 300 python tools/quick_time.py C2 C5 >> gpurun_out/q_nw.log 2>&1; done
