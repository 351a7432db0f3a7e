mkdir -p gpurun_out
NO_VARIANTS=1 OV_ONLY=1 DPRO_GRING0=1 timeout 600 python tools/overlay_bench.py 4 1184 2 > gpurun_out/r02_g_w4.log 2>&1
NO_VARIANTS=1 OV_ONLY=1 DPRO_GRING0=1 DPRO_WARPS=2 timeout 600 python tools/overlay_bench.py 4 1776 2 > gpurun_out/r02_g_w2.log 2>&1
timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_ref_c4.log
