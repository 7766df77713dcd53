#!/bin/bash
# ncu evidence for the current kernels (summaries copied to profiles/ afterwards).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'refresh|internal_merge|combine|partial_simt' -c 2500 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 2 -c 1 -o gpurun_out/k1_b16 python scripts/profile_k1.py --batch 16 --layers 2 --reps 2 > gpurun_out/ncu_k1.log 2>&1; echo "k1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:internal_merge -s 2 -c 1 -o gpurun_out/k2_b16 python scripts/profile_k1.py --batch 16 --layers 2 --reps 2 > gpurun_out/ncu_k2.log 2>&1; echo "k2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -c 1 -o gpurun_out/k1_prefill python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_2602_05305_b200 import kernels as K
g=torch.Generator(device='cuda').manual_seed(1)
r=lambda *s: torch.randn(s, device='cuda', generator=g).to(torch.bfloat16)
q,k,v=r(8,4*32768,128),r(8,32768,128),r(8,32768,128)
K.block_causal_attention(q,k,v,32768,0,32); torch.cuda.synchronize()
" > gpurun_out/ncu_prefill.log 2>&1; echo "prefill rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -c 1 -o gpurun_out/k1_c5 python scripts/prof_c5.py > gpurun_out/ncu_c5.log 2>&1; echo "c5 rc=$?"
timeout 300 ncu --set full --clock-control none -k regex:'row_cosine|pairwise' -c 2 -o gpurun_out/sim python -c "
import sys; sys.path.insert(0,'.')
import torch
from paper_2602_05305_b200 import kernels as K
a=torch.randn(12,4680,128,device='cuda'); b=torch.randn(12,4680,128,device='cuda')
K.row_cosine(a,b); K.pairwise_cosine(a[:, :256].contiguous(), b[:, :256].contiguous()); torch.cuda.synchronize()
" > gpurun_out/ncu_sim.log 2>&1; echo "sim rc=$?"
