mkdir -p gpurun_out/r28
D=gpurun_out/r28
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/tf32_ft python tools/prof_shape.py tf32 8192 8192 8192 2 > $D/a.log 2>&1
FTGEMM_LIB=paper_2305_01024_b200/libftgemm_nover.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/tf32_nover python tools/prof_shape.py tf32 8192 8192 8192 2 > $D/b.log 2>&1
echo done
