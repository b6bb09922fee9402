#!/bin/bash
# ncu --set full of the first two ResNet-20 stage launches with source attribution (session 3)
set -u
O=gpurun_out/s3
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ks_stage_kernel -s 0 -c 2 -o $O/ncu_stage python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/ncu_stage.log 2>&1; echo "ncu stage rc=$?"
ncu -i $O/ncu_stage.ncu-rep --page source --csv --print-source cuda,sass --launch-skip 1 --launch-count 1 > $O/stage_src.csv 2>/dev/null; echo "src rc=$?"
ls -la $O
