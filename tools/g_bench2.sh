#!/bin/bash
# bench (N=1, full) + the N>1 code path on one GPU (2 ranks over gloo; host-logic check, timings meaningless)
D=gpurun_out/bench; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout 900 python bench.py ${BENCH_ARGS:-} > $D/bench.json 2> $D/bench.err; tail -c 400 $D/bench.json; tail -3 $D/bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --backend gloo --steps 6 --warmup 3 --no-sweep > $D/multi_gloo.json 2> $D/multi_gloo.err; tail -c 600 $D/multi_gloo.json; tail -5 $D/multi_gloo.err
