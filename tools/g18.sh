mkdir -p gpurun_out
ATKG_LIB=build/libatkg_hp.so timeout 300 python tools/cpu_cost.py > gpurun_out/cpu_cost.log 2>&1
env | wc -l >> gpurun_out/cpu_cost.log
