#!/bin/bash
D=gpurun_out/epi_${1:-x}; mkdir -p $D
export PYTHONUNBUFFERED=1
timeout 300 python tools/ft_vs_off.py bf16 8192 8192 8192 bf16 16384 16384 128 bf16 4096 4096 4096 tf32 8192 8192 8192 tf32 16384 16384 128 bf16 128 16384 16384 > $D/t.txt 2>&1; cat $D/t.txt
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > $D/pytest.txt; cat $D/pytest.txt
