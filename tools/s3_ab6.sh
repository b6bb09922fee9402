#!/bin/bash
# session-3 A/B 6: tiler knobs on the ResNet-18 shape (env only)
set -u
export BENCH_ARGS="--workload resnet18"
bash tools/ab_env.sh "SFHR_MMA_RUN_ROWS=64" "SFHR_MMA_RUN_ROWS=32" "SFHR_MMA_RUN_ROWS=128" "SFHR_CONV_BLOCK=1" "SFHR_CONV_BLOCK=4" "SFHR_MMA_GATHER_CLK=3" "SFHR_MMA_GATHER_CLK=13" "SFHR_MMA_SAME_ROWS=128" "SFHR_MMA_RUN_ROWS=64"
