mkdir -p gpurun_out/r20
D=gpurun_out/r20
timeout 1200 python -m pytest tests -q -m gpu -x > $D/pytest_gpu.log 2>&1
for a in "bf16 8192 8192 8192 2" "bf16 8192 8192 8192 0" "tf32 8192 8192 8192 2" "tf32 8192 8192 8192 0" "bf16 8192 8192 1024 2" "bf16 8192 8192 1024 0" "bf16 16384 16384 128 2" "bf16 16384 16384 128 0"; do timeout 120 python tools/perf_probe.py $a >> $D/perf.log 2>&1; done
echo done
