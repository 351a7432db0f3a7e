mkdir -p gpurun_out
OV_ONLY=1 timeout 600 python tools/overlay_bench.py 4 1184 3 > gpurun_out/r02_h_1184.log 2>&1
OV_ONLY=1 timeout 600 python tools/overlay_bench.py 4 1480 3 > gpurun_out/r02_h_1480.log 2>&1
OV_ONLY=1 timeout 600 python tools/overlay_bench.py 4 1776 3 > gpurun_out/r02_h_1776.log 2>&1
timeout 900 python -m pytest tests/test_overlay.py -x -q > gpurun_out/r02_h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_h_tests.log
