mkdir -p gpurun_out
DPRO_LIB=exp/r1/libdpro_cuda.so timeout 600 python tools/scale_check.py 4 148 > gpurun_out/r02_abr1_old.log 2>&1
timeout 600 python tools/scale_check.py 4 148 > gpurun_out/r02_abr1_new.log 2>&1
DPRO_LIB=exp/r1/libdpro_cuda.so timeout 600 python tools/profile_replay.py --config 2 --batch 1024 --iters 3 > gpurun_out/r02_abr1_old_c2.log 2>&1
timeout 600 python tools/profile_replay.py --config 2 --batch 1024 --iters 3 > gpurun_out/r02_abr1_new_c2.log 2>&1
