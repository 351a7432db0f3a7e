mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r02_bench_c4_v3.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_c4_v3.log
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_c4_1776_launches.csv python tools/profile_ov.py 4 1776 1 > gpurun_out/r02_c4_1776_ncu.log 2>&1
