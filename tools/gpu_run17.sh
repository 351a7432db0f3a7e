mkdir -p gpurun_out
NO_VARIANTS=1 OV_ONLY=1 DPRO_WARPS=1 timeout 600 python tools/overlay_bench.py 4 740 2 > gpurun_out/r02_x_w1.log 2>&1
timeout 2400 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_ref_c4.log
