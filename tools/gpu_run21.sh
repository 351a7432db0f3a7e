mkdir -p gpurun_out
OV_ONLY=1 DPRO_WARPS=2 timeout 600 python tools/overlay_bench.py 4 1776 3 > gpurun_out/r02_i_w2_1776.log 2>&1
OV_ONLY=1 DPRO_WARPS=2 timeout 600 python tools/overlay_bench.py 4 1480 3 > gpurun_out/r02_i_w2_1480.log 2>&1
