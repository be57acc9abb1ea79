#!/bin/bash
# schedule-group x L2-hint experiment: interleaved timing + ncu DRAM bytes per variant
D=gpurun_out/l2_${1:-a}; mkdir -p $D
export PYTHONUNBUFFERED=1
V="0:0 4:0 12:0 17:0 33:0 0:2 0:8 0:10 0:16 0:26 0:4 0:20 17:26"
timeout 600 python tools/l2_sweep.py bf16 8192 8192 8192 2 $V > $D/time_ft.jsonl 2>&1; cat $D/time_ft.jsonl
timeout 300 python tools/l2_sweep.py bf16 8192 8192 8192 0 0:0 0:16 0:26 17:0 > $D/time_off.jsonl 2>&1; cat $D/time_off.jsonl
for v in $V; do
  gs=${v%%:*}; h=${v##*:}
  if [ "$gs" != 0 ]; then export FTGEMM_GROUP=$gs; else unset FTGEMM_GROUP; fi
  export FTGEMM_L2HINT=$h
  timeout 120 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:tc_ftgemm -s 1 -c 1 --csv python tools/prof_run.py bf16 8192 2 2 > $D/ncu_${gs}_${h}.csv 2>&1
  echo "$v $(grep -E 'dram__bytes|gpu__time|hit_rate' $D/ncu_${gs}_${h}.csv | awk -F'","' '{print $(NF-2)"="$NF}' | tr '\n' ' ')"
done
echo done
