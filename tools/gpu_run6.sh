mkdir -p gpurun_out
OV_ONLY=1 timeout 600 python tools/overlay_bench.py 4 296 2 > gpurun_out/r02_t_c4_296.log 2>&1
OV_ONLY=1 timeout 900 python tools/overlay_bench.py 4 1184 2 > gpurun_out/r02_t_c4_1184.log 2>&1
timeout 600 python tools/overlay_bench.py 2 1024 2 > gpurun_out/r02_t_c2_1024.log 2>&1
timeout 900 python -X faulthandler -m pytest tests/test_overlay.py tests/test_replay_gpu.py tests/test_delta.py -x -q > gpurun_out/r02_t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_t_tests.log
