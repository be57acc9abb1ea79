#!/bin/bash
D=gpurun_out/bench_${1:-x}; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; tail -c 400 $D/bench.err
