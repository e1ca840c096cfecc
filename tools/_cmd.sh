python -m pytest tests -m gpu -q -x -k "graph or peer or shard or dist" 2>&1 | tail -2
BS_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline 2>/tmp/e.log | tail -1 | cut -c1-300 || tail -5 /tmp/e.log
