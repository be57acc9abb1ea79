#!/bin/bash
# GPU test run: pytest -m gpu (optionally a -k expression / file list), log under gpurun_out/tests
D=gpurun_out/tests; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout ${T:-1500} python -m pytest ${@:-tests} -m gpu -q ${X:-} -rf 2>&1 | tail -40 > $D/pytest.txt; cat $D/pytest.txt
