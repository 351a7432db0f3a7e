mkdir -p gpurun_out
timeout 900 python -X faulthandler -m pytest tests/test_replay_gpu.py tests/test_overlay.py tests/test_delta.py -x -q > gpurun_out/r02_u_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_u_tests.log
timeout 600 python tools/profile_ov.py 4 296 2 > gpurun_out/r02_u_prof_plain.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:replay_ov_kernel --launch-skip 1 --launch-count 1 -o gpurun_out/r02_ov_c4_pass0 python tools/profile_ov.py 4 296 1 > gpurun_out/r02_u_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_ov_c4_launches.csv python tools/profile_ov.py 4 296 1 > gpurun_out/r02_u_ncu2.log 2>&1
