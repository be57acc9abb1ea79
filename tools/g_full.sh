#!/bin/bash
# full GPU test suite (+ threshold sweep log) and compute-sanitizer runs
D=gpurun_out/full; mkdir -p $D
export PYTHONUNBUFFERED=1 FTGEMM_FP_SWEEP_OUT=$D
timeout 1800 python -m pytest tests -m gpu -q -rf 2>&1 | tail -30 > $D/pytest.txt; cat $D/pytest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
[ -n "$SAN" ] && bash tools/g_sanitize.sh
true
