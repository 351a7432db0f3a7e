# gpurun helper: tests, bench, launch list (each step logged under gpurun_out/)
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r02_bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_c4.log
timeout 600 python bench.py --config 2 --cpu-seconds 0 > gpurun_out/r02_bench_c2.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_c2.log
