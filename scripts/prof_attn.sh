#!/bin/bash
# Per-tile timestamps + ncu --set full of the three attention kernels of one cfg2 step.
mkdir -p gpurun_out
timeout 300 python scripts/timing.py > gpurun_out/timing.log 2>&1; tail -40 gpurun_out/timing.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scfa_attn -s 9 -c 3 \
    -o gpurun_out/prof_attn -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
