#!/bin/bash
# Round-2 closing evidence: bench line, ncu launch list of a short bench run, ncu --set full of
# one cfg2 step's three attention kernels and of the preparation kernels (prep_ncu.py).
mkdir -p gpurun_out
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cfg3 --no-cudnn --no-cpu-baseline \
    > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scfa_attn_kernel -s 6 -c 3 \
    -o gpurun_out/prof_attn -f python scripts/prof_step.py 3 > gpurun_out/ncu_full.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"hash_prepare|permute_rows|tile_list" -s 4 -c 4 \
    -o gpurun_out/prof_prep -f python scripts/prep_ncu.py > gpurun_out/ncu_prep.log 2>&1
ls -la gpurun_out
