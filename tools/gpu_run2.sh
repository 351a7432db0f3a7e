set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_overlay.py tests/test_scale_parity.py -k "overlay or ns_" -x -q > gpurun_out/r02_ov_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_ov_tests.log
timeout 600 python tools/overlay_bench.py 4 148 2 > gpurun_out/r02_ov_c4_148.log 2>&1
timeout 600 python tools/overlay_bench.py 4 592 2 > gpurun_out/r02_ov_c4_592.log 2>&1
timeout 600 python tools/overlay_bench.py 4 1184 2 > gpurun_out/r02_ov_c4_1184.log 2>&1
timeout 600 python tools/overlay_bench.py 2 1024 3 > gpurun_out/r02_ov_c2_1024.log 2>&1
timeout 600 python tools/overlay_bench.py 2 4096 2 > gpurun_out/r02_ov_c2_4096.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu2.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pytest_gpu2.log
