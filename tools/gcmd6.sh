#!/bin/bash
export PYTHONUNBUFFERED=1
D=gpurun_out/r33; mkdir -p $D
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; tail -c 2500 $D/bench.json; tail -3 $D/bench.err
timeout 1500 python tools/sweep.py --out $D/sweep.json > $D/sweep.log 2>&1; tail -3 $D/sweep.log
