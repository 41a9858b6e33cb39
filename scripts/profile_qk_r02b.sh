#!/bin/bash
# cfg3 (QK B=4 H=12 T=16384 D=64 drop 0.5) evidence: launch list of three fused steps and ncu
# --set full of one step's attention kernels.
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/qk_launches.csv python scripts/prof_qk.py 3 > gpurun_out/qk_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scfa_attn_kernel -s 3 -c 3 \
    -o gpurun_out/prof_qk -f python scripts/prof_qk.py 2 > gpurun_out/qk_full.log 2>&1
ls -la gpurun_out
