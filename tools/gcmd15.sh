#!/bin/bash
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests -m gpu -x -q -k "fused_encode" 2>&1 | tail -2
sed -n '/^timeout 300 python - <<.PY./,/^PY$/p' tools/gcmd14.sh | sed '1d;$d' > /tmp/fe.py
timeout 300 python /tmp/fe.py
