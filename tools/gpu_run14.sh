mkdir -p gpurun_out
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r02_bench_c4_n2.log 2>&1; echo "rc=$?" >> gpurun_out/r02_bench_c4_n2.log
