mkdir -p gpurun_out; : > gpurun_out/qtv.log
for lib in paper_2506_04165_b200/libatkg.so build/variants/*.so; do
  echo "== $lib" >> gpurun_out/qtv.log
  ATKG_LIB=$lib timeout 120 python tools/quick_time.py C3 >> gpurun_out/qtv.log 2>&1
done
