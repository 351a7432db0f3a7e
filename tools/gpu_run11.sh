mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r02_bench_c4_v2.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_c4_v2.log
timeout 600 python bench.py --config 2 --cpu-seconds 0 > gpurun_out/r02_bench_c2_v2.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_c2_v2.log
