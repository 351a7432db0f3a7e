mkdir -p gpurun_out
CFG=4 NB=148 OVERLAY=1 DPRO_LIB=exp/prof/libdpro_cuda.so timeout 600 python tools/prof_phases.py > gpurun_out/r02_phases_c4_148.log 2>&1
CFG=4 NB=740 OVERLAY=1 DPRO_LIB=exp/prof/libdpro_cuda.so timeout 600 python tools/prof_phases.py > gpurun_out/r02_phases_c4_740.log 2>&1
CFG=2 NB=1024 DPRO_LIB=exp/prof/libdpro_cuda.so timeout 600 python tools/prof_phases.py > gpurun_out/r02_phases_c2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_c4_1480_launches.csv python tools/profile_ov.py 4 1480 1 > gpurun_out/r02_c4_1480_ncu.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:replay_ov_kernel --launch-count 1 -o gpurun_out/r02_c4_1480_pass0 python tools/profile_ov.py 4 1480 1 > gpurun_out/r02_c4_1480_ncu2.log 2>&1
