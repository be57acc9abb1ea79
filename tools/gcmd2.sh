mkdir -p gpurun_out/r19
D=gpurun_out/r19
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/k128_ft python tools/prof_shape.py bf16 16384 16384 128 2 > $D/b.log 2>&1
echo done
