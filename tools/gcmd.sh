mkdir -p gpurun_out/debug6
D=gpurun_out/debug6
timeout 120 python tools/gpu_debug.py full_bf16 > $D/bf16.log 2>&1
timeout 300 compute-sanitizer --tool memcheck --show-backtrace device python tools/gpu_debug.py bf16 > $D/san.log 2>&1
timeout 300 python tools/gpu_debug.py big > $D/big.log 2>&1
echo done
