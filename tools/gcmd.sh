mkdir -p gpurun_out/t1
D=gpurun_out/t1
timeout 1200 python -m pytest tests -q -m gpu -x --timeout 600 > $D/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1
echo done
