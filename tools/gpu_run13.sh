mkdir -p gpurun_out
timeout 900 python -X faulthandler -m pytest tests/test_overlay.py tests/test_replay_gpu.py -x -q > gpurun_out/r02_w_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_w_tests.log
NO_VARIANTS=1 OV_ONLY=1 timeout 600 python tools/overlay_bench.py 4 148 2 > gpurun_out/r02_w_nov148.log 2>&1
OV_ONLY=1 timeout 900 python tools/overlay_bench.py 4 1480 3 > gpurun_out/r02_w_1480.log 2>&1
CFG=4 NB=148 OVERLAY=1 DPRO_LIB=exp/prof/libdpro_cuda.so timeout 600 python tools/prof_phases.py > gpurun_out/r02_w_phases_c4_148.log 2>&1
