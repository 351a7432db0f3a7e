mkdir -p gpurun_out
timeout 2400 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_bench_ref_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_ref_c4.log
