set -x
mkdir -p gpurun_out
timeout 900 python -X faulthandler -m pytest tests/test_overlay.py -x -q > gpurun_out/r02_ov_tests3.log 2>&1; echo "rc=$?" >> gpurun_out/r02_ov_tests3.log
timeout 600 python tools/overlay_bench.py 4 148 2 > gpurun_out/r02_ov3_c4_148.log 2>&1
timeout 600 python tools/overlay_bench.py 4 592 2 > gpurun_out/r02_ov3_c4_592.log 2>&1
timeout 600 python tools/overlay_bench.py 2 1024 2 > gpurun_out/r02_ov3_c2_1024.log 2>&1
