#!/bin/bash
# Microbenchmarks: TMEM load / MUFU / F2FP rates and the TMA gather4 swizzle layout.
mkdir -p gpurun_out/mb
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/mb/microbench scripts/microbench.cu
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/mb/g4 scripts/gather4_test.cu -lcuda
timeout 60 gpurun_out/mb/g4 > gpurun_out/mb/g4.txt 2>&1; echo "rc=$?" >> gpurun_out/mb/g4.txt
timeout 120 gpurun_out/mb/microbench > gpurun_out/mb/micro.txt 2>&1; echo "rc=$?" >> gpurun_out/mb/micro.txt
cat gpurun_out/mb/g4.txt gpurun_out/mb/micro.txt
rm -f gpurun_out/mb/microbench gpurun_out/mb/g4
