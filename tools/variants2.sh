#!/bin/bash
for lib in paper_2506_04165_b200/libatkg.so build/variants/*.so; do
  echo "== $lib"
  ATKG_LIB=$lib python tools/quick_time.py C2 C5 C3 2>&1 | tail -3
done
