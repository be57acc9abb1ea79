mkdir -p gpurun_out/r10
D=gpurun_out/r10
timeout 1200 python -m pytest tests -q -m gpu -x > $D/pytest_gpu.log 2>&1
for a in "bf16 8192 8192 8192 2" "tf32 8192 8192 8192 2" "f32_simt 8192 8192 8192 2"; do timeout 120 python tools/perf_probe.py $a >> $D/perf.log 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 12 --csv --log-file $D/launches.csv python tools/prof_run.py bf16 8192 2 2 > $D/ncu_launch.log 2>&1
echo done
