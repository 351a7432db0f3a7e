set -x
mkdir -p gpurun_out
timeout 900 python -X faulthandler -m pytest tests/test_overlay.py -x -q > gpurun_out/r02_ov_tests2.log 2>&1; echo "rc=$?" >> gpurun_out/r02_ov_tests2.log
timeout 600 python tools/overlay_bench.py 4 148 2 > gpurun_out/r02_ov2_c4_148.log 2>&1
timeout 600 python tools/overlay_bench.py 4 1184 2 > gpurun_out/r02_ov2_c4_1184.log 2>&1
timeout 900 python -X faulthandler -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu3.log 2>&1; echo "rc=$?" >> gpurun_out/r02_pytest_gpu3.log
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/r02_sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r02_sanitize_memcheck.log
