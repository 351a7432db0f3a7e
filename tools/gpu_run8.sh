mkdir -p gpurun_out
OV_ONLY=1 timeout 600 python tools/overlay_bench.py 4 148 2 > gpurun_out/r02_ab_ov148.log 2>&1
MAT_ONLY=1 DPRO_DEEP_FIRST=0 DPRO_RING=16 timeout 600 python tools/overlay_bench.py 4 148 2 > gpurun_out/r02_ab_mat148.log 2>&1
MAT_ONLY=1 DPRO_DEEP_FIRST=0 DPRO_RING=16 timeout 600 python tools/overlay_bench.py 4 296 2 > gpurun_out/r02_ab_mat296.log 2>&1
MAT_ONLY=1 DPRO_DEEP_FIRST=1 timeout 600 python tools/overlay_bench.py 4 148 2 > gpurun_out/r02_ab_matdeep148.log 2>&1
