#!/bin/bash
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__shared_mem_per_block_dynamic --csv python tools/gemm_case.py 2048 1024 4096 --iters 2 --cublas > gpurun_out/cublas_list_fc2m.csv 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__shared_mem_per_block_dynamic --csv python tools/gemm_case.py 16384 1024 512 --iters 2 --cublas > gpurun_out/cublas_list_fc2k.csv 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__shared_mem_per_block_dynamic --csv python tools/gemm_case.py 8192 8192 8192 --iters 2 --cublas > gpurun_out/cublas_list_sq.csv 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"nvjet|sm100|gemm|Kernel" -c 1 -o gpurun_out/ncu_cublas_fc2m python tools/gemm_case.py 2048 1024 4096 --iters 1 --cublas > gpurun_out/ncu_cb.log 2>&1
echo ALLDONE
