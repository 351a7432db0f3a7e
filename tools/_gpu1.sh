set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | head -20 > gpurun_out/r02_lscpu.txt; nproc >> gpurun_out/r02_lscpu.txt; free -g >> gpurun_out/r02_lscpu.txt
timeout 600 python tools/scale_check.py 4 148 > gpurun_out/r02_scale4.log 2>&1
timeout 600 python tools/scale_check.py 4 296 > gpurun_out/r02_scale4_296.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv python tools/scale_check.py 4 148 > gpurun_out/r02_c4_ncu1.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"replay_fast|pack_kernel|delta_merge" -c 4 -o gpurun_out/r02_c4_full python tools/scale_check.py 4 148 > gpurun_out/r02_c4_ncu2.log 2>&1
ls -la gpurun_out
