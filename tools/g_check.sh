#!/bin/bash
# re-entry check: gpu tests + smoke + bench on a fresh box
D=gpurun_out/chk; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > $D/pytest.txt; cat $D/pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1; tail -2 $D/smoke.txt
timeout 900 python bench.py > $D/bench.json 2> $D/bench.err; tail -c 1500 $D/bench.json
