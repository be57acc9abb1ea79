#!/bin/bash
D=gpurun_out/r40; mkdir -p $D
timeout 300 ncu --set full --clock-control none -k regex:gemm\|sm100\|nvjet -s 3 -c 1 -o $D/cublas_bf16 python -c "
import torch
a=torch.randn(8192,8192,device='cuda').to(torch.bfloat16);b=torch.randn(8192,8192,device='cuda').to(torch.bfloat16)
for _ in range(6): c=a@b
torch.cuda.synchronize()
" > $D/c.log 2>&1
echo done
