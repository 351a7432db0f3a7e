mkdir -p gpurun_out
timeout 900 python -X faulthandler -m pytest tests/test_tsync_gpu.py tests/test_greedy.py tests/test_search.py -x -q > gpurun_out/r02_k2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_k2_tests.log
timeout 600 python tools/tsync_speed.py ring 8 0 256 16 > gpurun_out/r02_tsync_speed.log 2>&1
timeout 600 python tools/tsync_speed.py ps 16 4 64 16 >> gpurun_out/r02_tsync_speed.log 2>&1
timeout 600 python tools/tsync_speed.py ring 64 0 16 16 >> gpurun_out/r02_tsync_speed.log 2>&1
