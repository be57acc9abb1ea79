#!/bin/bash
export PYTHONUNBUFFERED=1
D=gpurun_out/r36; mkdir -p $D
for shape in "128 16384 16384" "16384 128 16384"; do
  for ft in 2 0; do
    n=$(echo $shape | tr ' ' x)_$ft
    timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__grid_size,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:tc_ftgemm -s 1 -c 1 --csv --log-file $D/$n.csv python tools/prof_shape.py bf16 $shape $ft > /dev/null 2>&1
    echo "== $n"; grep -v "^==" $D/$n.csv | python -c "
import csv,sys
for r in csv.reader(sys.stdin):
    if len(r)>14 and r[0]!='ID': print('  ', r[-4], r[-2], r[-1])
"
  done
done
