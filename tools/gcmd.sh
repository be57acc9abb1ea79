mkdir -p gpurun_out/r22
D=gpurun_out/r22
timeout 900 python bench.py --steps 50 --warmup 5 > $D/bench.log 2>&1
timeout 900 python tools/sweep.py --out $D/sweep_r1.json > $D/sweep.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $D/launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --cpu-seconds 1 > $D/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_ftgemm -s 1 -c 1 -o $D/fused_ft python tools/prof_run.py bf16 8192 2 3 > $D/ncu_ft.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:tc_ftgemm -s 1 -c 1 -o $D/fused_off python tools/prof_run.py bf16 8192 0 3 > $D/ncu_off.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:encode -s 2 -c 2 -o $D/encode python tools/prof_run.py bf16 8192 2 3 > $D/ncu_enc.log 2>&1
echo done
