mkdir -p gpurun_out
NO_VARIANTS=1 OV_ONLY=1 timeout 600 python tools/overlay_bench.py 4 148 2 > gpurun_out/r02_v_nov148.log 2>&1
NO_VARIANTS=1 OV_ONLY=1 timeout 600 python tools/overlay_bench.py 4 740 2 > gpurun_out/r02_v_nov740.log 2>&1
OV_ONLY=1 timeout 600 python tools/overlay_bench.py 4 740 3 > gpurun_out/r02_v_740.log 2>&1
OV_ONLY=1 timeout 900 python tools/overlay_bench.py 4 1480 3 > gpurun_out/r02_v_1480.log 2>&1
NO_VARIANTS=1 OV_ONLY=1 DPRO_WARPS=2 timeout 600 python tools/overlay_bench.py 4 740 2 > gpurun_out/r02_v_nov740_w2.log 2>&1
NO_VARIANTS=1 OV_ONLY=1 DPRO_WARPS=8 timeout 600 python tools/overlay_bench.py 4 740 2 > gpurun_out/r02_v_nov740_w8.log 2>&1
