#!/bin/bash
# cuBLAS BF16 8192^3 vs the fused kernel (FT off / FT): DRAM and L2->SM traffic, cluster shape
D=gpurun_out/cublas_cmp; mkdir -p $D
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex.sum,launch__cluster_dim_x,launch__cluster_dim_y,launch__grid_size,launch__block_size,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"
timeout 200 ncu --metrics $M --clock-control none -k regex:"gemm|sm100|nvjet|cutlass" -s 3 -c 1 --csv python -c "
import torch
a=torch.randn(8192,8192,device='cuda').to(torch.bfloat16);b=torch.randn(8192,8192,device='cuda').to(torch.bfloat16)
for _ in range(6): c=a@b
torch.cuda.synchronize()
" > $D/cublas.csv 2>&1
timeout 200 ncu --metrics $M --clock-control none -k regex:tc_ftgemm -s 1 -c 1 --csv python tools/prof_run.py bf16 8192 0 > $D/off.csv 2>&1
timeout 200 ncu --metrics $M --clock-control none -k regex:tc_ftgemm -s 1 -c 1 --csv python tools/prof_run.py bf16 8192 2 > $D/ft.csv 2>&1
for f in cublas off ft; do echo "== $f"; grep -E '^"[0-9]' $D/$f.csv | awk -F'","' '{print $5" | "$(NF-2)" = "$NF}' | cut -c1-60,100-400 | sed 's/"$//'; done
