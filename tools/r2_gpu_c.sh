#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_micro tools/mma_micro.cu && timeout 120 /tmp/mma_micro > gpurun_out/r2_mma_micro.txt 2>&1
