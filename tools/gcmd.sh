mkdir -p gpurun_out/r6
D=gpurun_out/r6
timeout 200 python tools/gpu_debug.py full_bf16 full_tf32 big > $D/dbg.log 2>&1
for a in "bf16 8192 8192 8192 2" "bf16 8192 8192 8192 0" "tf32 8192 8192 8192 2" "tf32 8192 8192 8192 0" "bf16 8192 8192 1024 2" "bf16 8192 8192 1024 0"; do timeout 60 python tools/perf_probe.py $a >> $D/perf.log 2>&1; done
echo done
