mkdir -p gpurun_out
for r in 16 32 64; do OV_ONLY=1 DPRO_RING=$r timeout 600 python tools/overlay_bench.py 4 296 1 > gpurun_out/r02_ring${r}_c4.log 2>&1; done
