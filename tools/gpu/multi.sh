# N>1 code path of bench.py with 2 ranks sharing the one GPU over gloo (a path check, not a measurement)
B2L_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --n-events 200000 --n-bufs 100000 2>&1 | tail -5 | cut -c1-2500
